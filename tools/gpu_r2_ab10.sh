# work-queue order of the packed light-row items: row order (src, default) vs by first source (all) / descending (all_desc)
for rep in 1 2; do
for o in src all all_desc; do
  SG_PLAN_ORDER=$o timeout 400 python tools/sched_ab.py reddit f32 >> gpurun_out/ab10.jsonl 2>> gpurun_out/ab10.err
done
done
