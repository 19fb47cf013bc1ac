# round 2 final measurement pass at the split-row combine-launch build: GPU suite, smoke, bench lines (all
# configs), reference arm, ncu DRAM records of the benched kernel source, launch list, multi-GPU proxy, ncu full
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rs 2>&1 | grep -E "passed|failed|SKIPPED|FAILED|Error" > gpurun_out/g_pytest.txt
timeout 900 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/g_ref.json 2> gpurun_out/g_ref.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:prop_kernel --launch-skip 3 --launch-count 1 -f -o gpurun_out/g_dram_reddit python tools/profile_step.py reddit 2 > gpurun_out/g_dram_reddit.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:prop_kernel --launch-skip 2 --launch-count 1 -f -o gpurun_out/g_dram_noreuse python tools/noreuse_pass.py > gpurun_out/g_dram_noreuse.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-reorder --no-bf16 --no-noreuse > gpurun_out/g_launch_bench.log 2>&1
timeout 1200 python tools/dist_proxy.py reddit 1 2 4 8 > gpurun_out/g_proxy.jsonl 2> gpurun_out/g_proxy.err
for c in pubmed blogcatalog10 powerlaw_gcn powerlaw_ggcn; do
  timeout 1200 python bench.py --config $c --no-cpu-baseline --no-noreuse --no-reorder --no-bf16 > gpurun_out/g_bench_$c.json 2> gpurun_out/g_bench_$c.err
done
ls -la gpurun_out | tail -40
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prop_kernel --launch-skip 3 --launch-count 2 -f -o /tmp/g_full python tools/profile_step.py reddit 2 > gpurun_out/g_full.log 2>&1
ncu -i /tmp/g_full.ncu-rep --page details --csv > gpurun_out/g_full_details.csv 2>&1
ncu -i /tmp/g_full.ncu-rep --page raw --csv > gpurun_out/g_full_raw.csv 2>&1
