ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_steps.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-reorder > gpurun_out/bench_under_ncu.json 2>/dev/null
python tools/ncu_summary.py launches gpurun_out/launches_steps.csv > gpurun_out/launches_steps.txt
cat gpurun_out/launches_steps.txt | head -12
