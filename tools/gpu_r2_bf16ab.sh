# round 2: bf16 storage epoch -- wide bf16 rows (F = 602: 3 x 16-B vectors per lane) at 2 / 3 blocks per SM, 2 / 4 rows in flight
L=paper_1810_08403_b200
for lib in libsagann.so libsagann_b3.so libsagann_b2d4.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 400 python tools/sched_ab.py reddit bf16 | sed "s/^{/{\"v\": \"$lib\", /" >> gpurun_out/bf.jsonl 2>> gpurun_out/bf.err
done
timeout 400 python tools/sched_ab.py reddit f32 | sed "s/^{/{\"v\": \"f32\", /" >> gpurun_out/bf.jsonl 2>> gpurun_out/bf.err
