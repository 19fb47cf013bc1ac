for cfg in "SG_HUB=0" "SG_HUB_KB=24" "SG_HUB_KB=48" "SG_HUB_KB=64" "SG_HUB_KB=100"; do
  echo "== $cfg"
  env $cfg timeout 120 python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print(d['ms_per_step'], s['L0.fwd.propagate'], s['L1.fwd.propagate'], s['L1.bwd.propagate'])"
done
