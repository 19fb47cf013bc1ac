# A/B round 2: batched in-order fold (out-of-line default / inline) vs end-of-pass combine; N=8 proxy for each
L=paper_1810_08403_b200
for i in 1 2 3; do
for lib in libsagann_old.so libsagann.so libsagann_inl.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 600 python tools/sched_ab.py reddit >> gpurun_out/c2_ab.jsonl 2>> gpurun_out/c2_ab.err
done
done
for lib in libsagann_old.so libsagann.so libsagann_inl.so; do
  echo "{\"lib\": \"$lib\"}" >> gpurun_out/c2_proxy.jsonl
  SG_LIB_PATH=$PWD/$L/$lib timeout 900 python tools/dist_proxy.py reddit 1 8 >> gpurun_out/c2_proxy.jsonl 2>> gpurun_out/c2_proxy.err
done
