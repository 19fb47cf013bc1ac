# round-2 baseline of HEAD: GPU suite, smoke, one bench line, launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/h_smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/h_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
