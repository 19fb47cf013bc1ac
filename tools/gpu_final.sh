timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/final_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches.txt
cat gpurun_out/final_pytest.txt gpurun_out/final_smoke.txt; tail -c 600 gpurun_out/final_bench.json; head -c 300 gpurun_out/final_bench_ref.json; head -8 gpurun_out/launches.txt
