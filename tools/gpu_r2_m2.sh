# round 2 measurement pass (small outputs only: gpurun_out/ must stay < 64 MiB)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/m_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_unfused.py -q -rf -x 2>&1 | tail -30 > gpurun_out/m_unfused.txt
timeout 2400 python -m pytest tests -q -m gpu -rf --deselect tests/test_gpu_unfused.py 2>&1 | grep -E "passed|failed|needed floor|normwise|FAILED|Error" > gpurun_out/m_pytest.txt
timeout 900 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:prop_kernel --launch-skip 3 --launch-count 1 --csv python tools/profile_step.py reddit 2 > gpurun_out/m_dram_reddit.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:prop_kernel --launch-skip 2 --launch-count 1 --csv python tools/noreuse_pass.py > gpurun_out/m_dram_noreuse.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/m_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-reorder --no-bf16 --no-noreuse > gpurun_out/m_launch_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prop_kernel --launch-skip 3 --launch-count 1 -f -o /tmp/m_full_l0 python tools/profile_step.py reddit 2 > gpurun_out/m_full.log 2>&1
ncu -i /tmp/m_full_l0.ncu-rep --page details --csv > gpurun_out/m_full_l0_details.csv 2>&1
ncu -i /tmp/m_full_l0.ncu-rep --page raw --csv > gpurun_out/m_full_l0_raw.csv 2>&1
du -sh gpurun_out
