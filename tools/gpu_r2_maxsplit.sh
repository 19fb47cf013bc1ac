# A/B: max-gather split rows combined by a second launch (default) vs in-pass (libsagann_old.so =
# -DSG_MAX_SPLIT_KERNEL=0), MP-GCN step stage times; max / MP-GCN GPU tests on the default
L=paper_1810_08403_b200
for i in 1 2; do
for lib in libsagann_old.so libsagann.so; do
  echo "{\"lib\": \"$lib\"}" >> gpurun_out/m_ab.jsonl
  SG_LIB_PATH=$PWD/$L/$lib timeout 600 python tools/mp_time.py >> gpurun_out/m_ab.jsonl 2>> gpurun_out/m_ab.err
done
done
timeout 1200 python -m pytest tests -q -m gpu -x -k "max or mpgcn or segment or unfused" 2>&1 | tail -5 > gpurun_out/m_pytest.txt
