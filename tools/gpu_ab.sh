ncu --set full --clock-control none --import-source on -k regex:prop_kernel --launch-skip 2 --launch-count 1 -o /tmp/narrow python tools/narrow_point.py 16 4 > /tmp/n.log 2>&1
tail -2 /tmp/n.log
python tools/ncu_summary.py report /tmp/narrow.ncu-rep
ncu -i /tmp/narrow.ncu-rep --page raw --csv --metrics l1tex__t_sector_hit_rate.pct,smsp__warps_eligible.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed | tail -2
