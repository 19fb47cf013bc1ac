# round 2: G-GCN gated passes (two-operand rows) -- rows in flight 4 (default) vs 2 / 6, BlogCatalog x10 and power-law G-GCN
L=paper_1810_08403_b200
for rep in 1 2; do
for lib in libsagann.so libsagann_gd4.so libsagann_gd12.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 400 python tools/sched_ab.py blogcatalog10 f32 | sed "s/^{/{\"v\": \"$lib\", /" >> gpurun_out/ab7.jsonl 2>> gpurun_out/ab7.err
done
done
for lib in libsagann.so libsagann_gd4.so libsagann_gd12.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 900 python tools/sched_ab.py powerlaw_ggcn f32 | sed "s/^{/{\"v\": \"$lib\", /" >> gpurun_out/ab7.jsonl 2>> gpurun_out/ab7.err
done
