for c in pubmed blogcatalog10 powerlaw_gcn powerlaw_ggcn; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-reorder 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), round(d['value']/1e9,3), 'e2e', round(d['e2e']['ms_per_step'],3), {k: round(v,2) for k,v in d['stages_ms'].items()})"
done
