# the bench's multi-rank (torchrun) path on a one-GPU box: N ranks share cuda:0 over gloo
# (SG_DIST_BACKEND test hook; NCCL refuses two ranks on one device).  Validates barriers,
# max-over-ranks timing, e2e, launch counts and the JSON line the driver's scaling run parses.
for n in 2 4; do
SG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dist_gloo_gcn_$n.json 2> gpurun_out/dist_gloo_gcn_$n.err; echo "gcn n=$n rc=$?"
done
SG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --config blogcatalog10 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dist_gloo_ggcn_2.json 2> gpurun_out/dist_gloo_ggcn_2.err; echo "ggcn n=2 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/dist_ref_2.json 2> gpurun_out/dist_ref_2.err; echo "ref n=2 rc=$?"
for f in gpurun_out/dist_gloo_*.json gpurun_out/dist_ref_2.json; do echo "== $f"; head -c 700 $f; echo; done
tail -5 gpurun_out/dist_gloo_gcn_2.err
