# round 2: occupancy variants of the row kernel (wide rows 4 blocks/SM; one-vector rows 4 blocks x DEPTH 4) + dist proxy stage breakdown
L=paper_1810_08403_b200
for lib in libsagann.so libsagann_wb4.so libsagann_v1b4d4.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 400 python tools/sched_ab.py reddit f32 >> gpurun_out/ab2.jsonl 2>> gpurun_out/ab2.err
done
timeout 1200 python tools/dist_proxy.py reddit 1 4 8 > gpurun_out/ab2_proxy.jsonl 2> gpurun_out/ab2_proxy.err
