# bf16 half-vector rows only on hub-heavy passes + max-gather combine launch for the backward only:
# sweep, bf16 / fp32 Reddit epochs, MP-GCN stages (default vs forward combine launch), GPU suite
timeout 900 python tools/sweep.py > gpurun_out/sweep_r02b.jsonl 2> gpurun_out/sweep_r02b.err
timeout 600 python tools/sched_ab.py reddit bf16 >> gpurun_out/v2_ab.jsonl 2>> gpurun_out/v2_ab.err
timeout 600 python tools/sched_ab.py reddit >> gpurun_out/v2_ab.jsonl 2>> gpurun_out/v2_ab.err
L=paper_1810_08403_b200
for lib in libsagann.so libsagann_fwd1.so libsagann.so libsagann_fwd1.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 600 python tools/mp_time.py >> gpurun_out/v2_mp.jsonl 2>> gpurun_out/v2_mp.err
done
timeout 2400 python -m pytest tests -q -m gpu -rs 2>&1 | grep -E "passed|failed|SKIPPED|FAILED|Error" > gpurun_out/v2_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v2_smoke.txt 2>&1
