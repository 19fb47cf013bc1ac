timeout 900 python -m pytest tests -q -x -m gpu -k "propagate or model or ggcn or hub" 2>&1 | tail -2
timeout 300 python tools/narrow_ab.py 16 128 602 2>&1 | grep -v Warn | tail -1
timeout 900 python tools/sweep.py --quick 2>/dev/null | grep '"sum"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['dtype'], d['F'], d['avg_degree'], round(d['ms'],3), round(d['hbm_frac'],2))"
