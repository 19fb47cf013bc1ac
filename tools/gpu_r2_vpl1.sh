# A/B: one-vector fp32 rows (F = 128 passes) at 2 blocks/SM x 8 rows (default, 114 regs) vs 3 blocks x 8
# (libsagann_b3.so, 80 regs + 52 B spill) vs 3 blocks x 6 (libsagann_b3d6.so, 80 regs, no spill)
L=paper_1810_08403_b200
for i in 1 2 3; do
for lib in libsagann.so libsagann_b3.so libsagann_b3d6.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 600 python tools/sched_ab.py reddit >> gpurun_out/b_ab.jsonl 2>> gpurun_out/b_ab.err
done
done
