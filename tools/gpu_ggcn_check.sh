timeout 900 python -m pytest tests -x -q -m gpu -k "ggcn or dist" 2>&1 | tail -3
timeout 600 python bench.py --config blogcatalog10 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"
timeout 900 python bench.py --config powerlaw_ggcn --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"
