# sanitizer over the GPU kernel tests (memcheck all kernel tests, racecheck a subset), then the
# ncu launch list of the bench command and a summary of it
(compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -x -k "propagate or ggnn or gemm or max_gather or softmax or primitives or hub" 2>&1 | tail -3;
 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -x -k "propagate_fwd_bitwise or ggnn_typed or max_gather or gemm_tcgen05" 2>&1 | tail -3) > gpurun_out/sanitizer.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches.txt
tail -3 gpurun_out/sanitizer.txt; head -12 gpurun_out/launches.txt
