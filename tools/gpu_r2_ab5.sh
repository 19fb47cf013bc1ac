# round 2: one-vector warp-row kernel: 2 blocks x 8 rows (default) vs 3 x 4, 4 x 3, 4 x 4 rows in flight, interleaved
L=paper_1810_08403_b200
for rep in 1 2; do
for lib in libsagann.so libsagann_v1b3d4.so libsagann_v1b4d3.so libsagann_v1b4d4b.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 400 python tools/sched_ab.py reddit f32 | sed "s/^{/{\"v\": \"$lib\", /" >> gpurun_out/ab5.jsonl 2>> gpurun_out/ab5.err
done
done
