# round 2: wide-row block cap for passes without heavy rows -- gather tests, bench line (incl. the uniform no-reuse point)
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 > gpurun_out/cap_test.txt
timeout 900 python bench.py > gpurun_out/cap_bench.json 2> gpurun_out/cap_bench.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:prop_kernel --launch-skip 3 --launch-count 1 -f -o gpurun_out/cap_dram_reddit python tools/profile_step.py reddit 2 > gpurun_out/cap_dram_reddit.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:prop_kernel --launch-skip 2 --launch-count 1 -f -o gpurun_out/cap_dram_noreuse python tools/noreuse_pass.py > gpurun_out/cap_dram_noreuse.log 2>&1
