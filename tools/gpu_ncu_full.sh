ncu --set full --clock-control none --import-source on -k regex:'prop_kernel|gemm_tma' --launch-skip 8 --launch-count 8 -o /tmp/step python tools/profile_step.py reddit 2 > /tmp/ncu_step.log 2>&1
tail -2 /tmp/ncu_step.log
python tools/ncu_summary.py report /tmp/step.ncu-rep > gpurun_out/ncu_full_reddit.txt
ncu -i /tmp/step.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/ncu_dram.csv
cat gpurun_out/ncu_full_reddit.txt | head -60
