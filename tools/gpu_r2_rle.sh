# round 2: host RLE pass index on/off (epoch + stage times), unfused executor tests
timeout 600 python -m pytest tests/test_gpu_unfused.py -q -rf 2>&1 | tail -5 > gpurun_out/r_unfused.txt
for rle in 0 1; do
  SG_RLE=$rle timeout 300 python tools/sched_ab.py reddit f32 | sed "s/^{/{\"rle\": $rle, /" >> gpurun_out/r_ab.jsonl 2>> gpurun_out/r_ab.err
done
for rle in 0 1; do
  SG_RLE=$rle timeout 300 python tools/sched_ab.py reddit f32 | sed "s/^{/{\"rle\": $rle, /" >> gpurun_out/r_ab.jsonl 2>> gpurun_out/r_ab.err
done
