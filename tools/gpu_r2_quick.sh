# quick GPU check: GPU test suite + one bench line (stage times)
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/q_pytest.txt
timeout 600 python bench.py --no-cpu-baseline --no-reorder > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
