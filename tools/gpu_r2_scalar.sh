# A/B: combine launch with one column per lane and 64 partials in flight (default) vs four-column
# vectors with 16 in flight (libsagann_vec.so); propagation GPU tests; N=8 proxy for both
timeout 1200 python -m pytest tests -q -m gpu -x -k "propagate or deep or hub or bf16 or ggcn or fused or staged" 2>&1 | tail -3 > gpurun_out/sc_pytest.txt
L=paper_1810_08403_b200
for i in 1 2; do
for lib in libsagann_vec.so libsagann.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 600 python tools/sched_ab.py reddit >> gpurun_out/sc_ab.jsonl 2>> gpurun_out/sc_ab.err
done
done
for lib in libsagann_vec.so libsagann.so; do
  echo "{\"lib\": \"$lib\"}" >> gpurun_out/sc_proxy.jsonl
  SG_LIB_PATH=$PWD/$L/$lib timeout 900 python tools/dist_proxy.py reddit 1 8 >> gpurun_out/sc_proxy.jsonl 2>> gpurun_out/sc_proxy.err
done
