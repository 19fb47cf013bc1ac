# dist proxy: per-rank stage breakdown, with and without simulated receives (SG_PROXY_RECV)
timeout 1500 python tools/dist_proxy.py reddit 1 8 > gpurun_out/p_base.jsonl 2> gpurun_out/p_base.err
SG_PROXY_RECV=1 timeout 1500 python tools/dist_proxy.py reddit 1 2 4 8 > gpurun_out/p_recv.jsonl 2> gpurun_out/p_recv.err
