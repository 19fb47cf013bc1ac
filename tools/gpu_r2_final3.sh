# last measurement pass of round 2 on the committed HEAD: bench line, ncu DRAM records stamped on this
# kernel source, launch list, all model families' step times
set -x
timeout 900 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:prop_kernel --launch-skip 3 --launch-count 1 -f -o gpurun_out/h_dram_reddit python tools/profile_step.py reddit 2 > gpurun_out/h_dram_reddit.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:prop_kernel --launch-skip 2 --launch-count 1 -f -o gpurun_out/h_dram_noreuse python tools/noreuse_pass.py > gpurun_out/h_dram_noreuse.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/h_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-reorder --no-bf16 --no-noreuse > gpurun_out/h_launch_bench.log 2>&1
timeout 900 python tools/models_time.py > gpurun_out/h_models.txt 2> gpurun_out/h_models.err
