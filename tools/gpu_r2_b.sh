# round 2: GPU suite, NaN debug, epoch A/B f32/bf16, dist proxy
timeout 300 python tools/debug_nan.py > gpurun_out/b_nan.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | grep -E "passed|failed|needed floor|normwise|FAILED|Error|DID NOT" > gpurun_out/b_pytest.txt
for dt in f32 bf16; do timeout 300 python tools/sched_ab.py reddit $dt >> gpurun_out/b_ab.jsonl 2>> gpurun_out/b_ab.err; done
timeout 1200 python tools/dist_proxy.py reddit 1 2 4 8 > gpurun_out/b_proxy.jsonl 2> gpurun_out/b_proxy.err
