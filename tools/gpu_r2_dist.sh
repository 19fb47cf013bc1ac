# round 2: column-pass sharding -- GPU dist tests (gloo ranks sharing the B200), proxy both modes, bench multi-rank path over gloo
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -3 > gpurun_out/d_test.txt
SG_PROXY_COLUMN=1 timeout 1200 python tools/dist_proxy.py reddit 1 2 4 8 > gpurun_out/d_proxy.jsonl 2> gpurun_out/d_proxy.err
SG_PROXY_COLUMN=0 timeout 1200 python tools/dist_proxy.py reddit 1 2 4 8 >> gpurun_out/d_proxy.jsonl 2>> gpurun_out/d_proxy.err
bash tools/gpu_dist_gloo.sh > gpurun_out/d_gloo.txt 2>&1
