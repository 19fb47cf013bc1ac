# round 2: one-vector (F <= 128) warp-row kernel at 3 blocks/SM with 4 / 5 / 6 rows in flight vs 2 blocks x 8
L=paper_1810_08403_b200
for lib in libsagann.so libsagann_v1b3d4.so libsagann_v1b3d5.so libsagann_v1b3d6.so libsagann.so libsagann_v1b3d5.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 400 python tools/sched_ab.py reddit f32 | sed "s/^{/{\"v\": \"$lib\", /" >> gpurun_out/ab4.jsonl 2>> gpurun_out/ab4.err
done
for lib in libsagann.so libsagann_v1b3d5.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 400 python tools/sched_ab.py blogcatalog10 f32 | sed "s/^{/{\"v\": \"$lib\", /" >> gpurun_out/ab4.jsonl 2>> gpurun_out/ab4.err
done
