# A/B: split-subgroup queue order (row vs first source) x CTA-chunked work queue (1 / 8 / 24)
L=paper_1810_08403_b200
for lib in libsagann.so libsagann_q8.so libsagann_q24.so; do
  for order in row src; do
    SG_LIB_PATH=$PWD/$L/$lib SG_PLAN_ORDER=$order timeout 300 python tools/sched_ab.py reddit >> gpurun_out/s_ab.jsonl 2>> gpurun_out/s_ab.err
  done
done
# ncu: L2 / L1 traffic of the L0 pass, baseline vs q8+src
for cfg in "libsagann.so row" "libsagann_q8.so src"; do
  set -- $cfg
  SG_LIB_PATH=$PWD/$L/$1 SG_PLAN_ORDER=$2 timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:prop_kernel --launch-skip 3 --launch-count 1 --csv python tools/profile_step.py reddit 2 > gpurun_out/s_ncu_$1_$2.csv 2>&1
done
