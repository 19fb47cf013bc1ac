for c in 0 -1 50 100; do SG_CARVEOUT=$c timeout 300 python tools/narrow_ab.py 128 602 2>&1 | grep env; done
