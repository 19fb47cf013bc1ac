timeout 2400 python tools/sweep.py > gpurun_out/sweep_full.jsonl 2> gpurun_out/sweep_full.err
wc -l gpurun_out/sweep_full.jsonl; tail -2 gpurun_out/sweep_full.err
compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_kernels.py -q -x -k "propagate_fwd_bitwise or ggnn_typed or max_gather or gemm_tcgen05 or hub" 2>&1 | tail -3 > gpurun_out/synccheck.txt
cat gpurun_out/synccheck.txt
