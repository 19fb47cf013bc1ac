# subgroup size T of the per-rank column passes (proxy, N = 4, 8)
for T in auto 256 512 2048 4096; do
  SG_PROXY_SPLIT=$T timeout 1200 python tools/dist_proxy.py reddit 4 8 >> gpurun_out/sp.jsonl 2>> gpurun_out/sp.err
done
