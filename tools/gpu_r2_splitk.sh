# A/B: split-row partials folded by a separate combine launch (SG_SPLIT_KERNEL=1, default) vs the
# in-pass fold by the last subgroup's warp (libsagann_old.so: -DSG_SPLIT_KERNEL=0); N=8 proxy; GPU suite
L=paper_1810_08403_b200
for i in 1 2 3; do
for lib in libsagann_old.so libsagann.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 600 python tools/sched_ab.py reddit >> gpurun_out/s_ab.jsonl 2>> gpurun_out/s_ab.err
done
done
for lib in libsagann_old.so libsagann.so; do
  echo "{\"lib\": \"$lib\"}" >> gpurun_out/s_proxy.jsonl
  SG_LIB_PATH=$PWD/$L/$lib timeout 900 python tools/dist_proxy.py reddit 1 8 >> gpurun_out/s_proxy.jsonl 2>> gpurun_out/s_proxy.err
done
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/s_pytest.txt
