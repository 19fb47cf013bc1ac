timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "hub or propagate_fwd or propagate_bwd" 2>&1 | tail -2
for cs in 1 2 4 8 16; do SG_HUB_CLUSTER=$cs timeout 300 python tools/narrow_ab.py 602 2>&1 | grep -v Warn | tail -1; done
for kb in 32 96; do SG_HUB_KB=$kb SG_HUB_CLUSTER=8 timeout 300 python tools/narrow_ab.py 602 2>&1 | grep -v Warn | tail -1; done
SG_HUB=0 timeout 300 python tools/narrow_ab.py 602 2>&1 | grep -v Warn | tail -1
