# bf16 8-byte-vector rows at 4 blocks x 4: bf16 parity tests, bf16 epoch
timeout 1500 python -m pytest tests/test_gpu_bf16.py -q 2>&1 | tail -2 > gpurun_out/bb_test.txt
timeout 400 python tools/sched_ab.py reddit bf16 > gpurun_out/bb_ab.jsonl 2> gpurun_out/bb_ab.err
timeout 400 python tools/sched_ab.py reddit f32 >> gpurun_out/bb_ab.jsonl 2>> gpurun_out/bb_ab.err
