SG_PROP_TEAM_MAXV=0 timeout 300 python tools/narrow_ab.py 4 8 16
for t in 16 0; do SG_PROP_TEAM_MAXV=$t timeout 900 python tools/sweep.py --quick 2>/dev/null | grep '"F": 16' | grep '"sum"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print($t, d['dtype'], d['avg_degree'], round(d['ms'],3), round(d['hbm_frac'],2))"; done
