compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_kernels.py -q -x -k "max or ggnn or ggcn or segment_max or streaming" 2>&1 | tail -3
compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_kernels.py -q -x -k "max_gather_fwd_bwd_bitwise or segment_max_primitive or ggcn_propagate" 2>&1 | tail -3
compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_kernels.py -q -x -k "max_gather_fwd_bwd_bitwise or segment_max_primitive or ggcn_propagate" 2>&1 | tail -3
