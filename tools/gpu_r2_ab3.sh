# round 2: wide-row occupancy variants (4 / 5 blocks per SM, with / without in-register run detection) + graph-captured dist proxy
L=paper_1810_08403_b200
for lib in libsagann.so libsagann_wb4.so libsagann_wb4nr.so libsagann_wb5.so libsagann_wb4.so libsagann_wb4nr.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 400 python tools/sched_ab.py reddit f32 | sed "s/^{/{\"v\": \"$lib\", /" >> gpurun_out/ab3.jsonl 2>> gpurun_out/ab3.err
done
timeout 1200 python tools/dist_proxy.py reddit 1 2 4 8 > gpurun_out/ab3_proxy.jsonl 2> gpurun_out/ab3_proxy.err
