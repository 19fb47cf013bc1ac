nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g0_smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/g0_pytest.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g0_bench.json 2> gpurun_out/g0_bench.err
