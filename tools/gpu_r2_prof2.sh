# round 2: ncu --set full of the current L0 (F = 602, 4 blocks/SM) and L1 forward (F = 128) gathers
# prop_kernel launch order per epoch: L0 fwd, L1 fwd, L1 bwd -> skip one epoch (3 launches)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prop_kernel --launch-skip 3 --launch-count 2 -f -o /tmp/p2 python tools/profile_step.py reddit 2 > gpurun_out/p2.log 2>&1
ncu -i /tmp/p2.ncu-rep --page details --csv > gpurun_out/p2_details.csv 2>&1
ncu -i /tmp/p2.ncu-rep --page raw --csv > gpurun_out/p2_raw.csv 2>&1
