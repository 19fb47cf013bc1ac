# round 2: config-shape parity + bf16 parity, then the whole GPU suite without -x (tolerance audit)
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_bf16.py -q -rf 2>&1 | tail -40 > gpurun_out/p_new.txt
timeout 1500 python -m pytest tests -q -m gpu -rf --deselect tests/test_gpu_configs.py --deselect tests/test_gpu_bf16.py 2>&1 | tail -40 > gpurun_out/p_all.txt
