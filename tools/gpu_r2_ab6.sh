# round 2: bf16 storage epoch with the one-vector kernel variants (bf16 F = 128 rows: 8-byte vectors, 1.5x the fp32 rows in flight)
L=paper_1810_08403_b200
for rep in 1 2; do
for lib in libsagann.so libsagann_v1b3d4.so libsagann_v1b4d3.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 400 python tools/sched_ab.py reddit bf16 | sed "s/^{/{\"v\": \"$lib\", /" >> gpurun_out/ab6.jsonl 2>> gpurun_out/ab6.err
done
done
