# A/B: split-row partials folded in order as they complete (SG_CHAIN_COMBINE, out-of-line / inline)
# vs the last subgroup combining all partials; then the GPU suite and the N=8 proxy on the default
L=paper_1810_08403_b200
for lib in libsagann_old.so libsagann.so libsagann_inl.so libsagann_old.so libsagann.so libsagann_inl.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 600 python tools/sched_ab.py reddit >> gpurun_out/c_ab.jsonl 2>> gpurun_out/c_ab.err
done
timeout 1500 python tools/dist_proxy.py reddit 1 8 > gpurun_out/c_proxy.jsonl 2> gpurun_out/c_proxy.err
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/c_pytest.txt
