# round 2: GPU suite + epoch A/B (fp32 / bf16) + L0 ncu DRAM on the current kernel source
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | grep -E "passed|failed|needed floor|normwise|FAILED|Error" > gpurun_out/c_pytest.txt
for dt in f32 bf16; do timeout 300 python tools/sched_ab.py reddit $dt >> gpurun_out/c_ab.jsonl 2>> gpurun_out/c_ab.err; done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:prop_kernel --launch-skip 3 --launch-count 1 -f -o gpurun_out/c_dram_reddit python tools/profile_step.py reddit 2 > gpurun_out/c_dram_reddit.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:prop_kernel --launch-skip 2 --launch-count 1 -f -o gpurun_out/c_dram_noreuse python tools/noreuse_pass.py > gpurun_out/c_dram_noreuse.log 2>&1
