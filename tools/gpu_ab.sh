timeout 900 python -m pytest tests -q -x -m gpu -k "segment_max or primitives or max" 2>&1 | tail -2
timeout 900 python tools/sweep.py --quick 2>/dev/null | grep '"max' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['reduction'], d['F'], d['avg_degree'], round(d['ms'],3), round(d['hbm_frac'],2))"
