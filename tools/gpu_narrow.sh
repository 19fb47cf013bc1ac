timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python tools/sweep.py --quick > gpurun_out/sweep_quick.jsonl 2> gpurun_out/sweep.err; tail -2 gpurun_out/sweep.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['reordered_apply_vertex']['ms_per_step'], d['reordered_apply_vertex']['stages_ms'])"
timeout 600 python bench.py --config pubmed --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"
