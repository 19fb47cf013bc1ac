for p in 1 4; do timeout 900 python tools/stream_bench.py --parts $p --model gcn 2>&1 | tail -1; done
for p in 1 4; do timeout 900 python tools/stream_bench.py --parts $p --model ggcn 2>&1 | tail -1; done
timeout 900 python bench.py --config reddit --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-reorder 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('resident gcn', d['ms_per_step'])"
