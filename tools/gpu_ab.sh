timeout 300 python tools/narrow_ab.py 602 2>&1 | grep -v Warn | tail -1
SG_HUB=0 timeout 300 python tools/narrow_ab.py 602 2>&1 | grep -v Warn | tail -1
SG_HUB_KB=32 timeout 300 python tools/narrow_ab.py 602 2>&1 | grep -v Warn | tail -1
