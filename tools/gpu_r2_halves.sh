# column passes: one launch vs the column cut in two halves (proxy, compute only)
SG_PROXY_HALVES=0 timeout 1200 python tools/dist_proxy.py reddit 4 8 > gpurun_out/hv.jsonl 2> gpurun_out/hv.err
SG_PROXY_HALVES=1 timeout 1200 python tools/dist_proxy.py reddit 4 8 >> gpurun_out/hv.jsonl 2>> gpurun_out/hv.err
