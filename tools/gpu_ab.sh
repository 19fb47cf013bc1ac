timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "max or mpgcn" 2>&1 | grep -E "^E  |passed|failed" | head -8
timeout 600 python tools/mp_time.py 2>&1 | tail -1
