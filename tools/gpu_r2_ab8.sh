# round 2: L1 cache policy of the gathered-row loads (SG_ROW_LOAD 0 nc / 1 no_allocate / 2 evict_first / 3 evict_last / 4 cg)
L=paper_1810_08403_b200
for rep in 1 2; do
for lib in libsagann.so libsagann_ld1.so libsagann_ld2.so libsagann_ld3.so libsagann_ld4.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 400 python tools/sched_ab.py reddit f32 | sed "s/^{/{\"v\": \"$lib\", /" >> gpurun_out/ab8.jsonl 2>> gpurun_out/ab8.err
done
done
