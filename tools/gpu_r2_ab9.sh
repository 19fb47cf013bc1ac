# occupancy re-check with evict_last row loads: F = 128 rows 2x8 (default) / 4x3 / 3x4; wide rows 4 (default) / 3 blocks
L=paper_1810_08403_b200
for rep in 1 2; do
for lib in libsagann.so libsagann_e_v1b4d3.so libsagann_e_v1b3d4.so libsagann_e_wb3.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 400 python tools/sched_ab.py reddit f32 | sed "s/^{/{\"v\": \"$lib\", /" >> gpurun_out/ab9.jsonl 2>> gpurun_out/ab9.err
done
done
