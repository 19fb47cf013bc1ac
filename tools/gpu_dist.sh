set -x
free -g | head -2; nproc
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -15
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --engine dist --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
timeout 900 python bench.py --config powerlaw_gcn --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
timeout 900 python bench.py --config powerlaw_ggcn --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
