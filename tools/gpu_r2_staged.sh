# round 2: source-staged gather -- bitwise test, epoch A/B (SG_STAGED=0/1, SG_STAGES=2/3), ncu of the staged passes
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k staged 2>&1 | tail -30 > gpurun_out/st_test.txt
if grep -q " passed" gpurun_out/st_test.txt && ! grep -q "failed" gpurun_out/st_test.txt; then
  for cfg in "0 3" "1 3" "1 2"; do
    set -- $cfg
    SG_STAGED=$1 SG_STAGES=$2 timeout 400 python tools/sched_ab.py reddit f32 | sed "s/^{/{\"staged\": $1, \"stages\": $2, /" >> gpurun_out/st_ab.jsonl 2>> gpurun_out/st_ab.err
  done
  M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum
  timeout 600 ncu --metrics $M --clock-control none -k regex:staged --launch-skip 3 --launch-count 3 --csv python tools/profile_step.py reddit 2 > gpurun_out/st_ncu.csv 2>&1
fi
