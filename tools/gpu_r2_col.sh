# round 2: default 4 blocks/SM wide kernel -- bitwise gather tests; dist proxy per-chunk vs column passes
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3 > gpurun_out/c_test.txt
SG_PROXY_COLUMN=0 timeout 1200 python tools/dist_proxy.py reddit 1 2 4 8 > gpurun_out/c_proxy.jsonl 2> gpurun_out/c_proxy.err
SG_PROXY_COLUMN=1 timeout 1200 python tools/dist_proxy.py reddit 1 2 4 8 >> gpurun_out/c_proxy.jsonl 2>> gpurun_out/c_proxy.err
