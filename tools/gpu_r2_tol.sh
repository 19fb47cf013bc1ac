# round 2: bf16 GEMM + bf16 propagate tests; tolerance audit of the failing fp32 tests (needed floors)
timeout 900 python -m pytest tests/test_gpu_bf16.py -q -rf 2>&1 | grep -E "passed|failed|Error|needed|assert |FAILED" | head -60 > gpurun_out/t_bf16.txt
timeout 1500 python -m pytest tests -q -m gpu -rf 2>&1 | grep -E "passed|failed|needed floor|normwise|FAILED" > gpurun_out/t_all.txt
