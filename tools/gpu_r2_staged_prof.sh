# ncu --set full of the staged L0 pass (stall reasons, source hot spots)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:staged --launch-skip 3 --launch-count 1 -f -o /tmp/st_full python tools/profile_step.py reddit 2 > gpurun_out/stp_full.log 2>&1
ncu -i /tmp/st_full.ncu-rep --page details --csv > gpurun_out/stp_details.csv 2>&1
ncu -i /tmp/st_full.ncu-rep --page source --csv --print-source sass > gpurun_out/stp_source.csv 2>&1
ls -la gpurun_out/
