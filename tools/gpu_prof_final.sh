bash tools/gpu_ncu_full.sh > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-reorder > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches.txt
head -18 gpurun_out/ncu_full_reddit.txt; head -6 gpurun_out/launches.txt
