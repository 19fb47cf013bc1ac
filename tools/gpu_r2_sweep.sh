# BASELINE config 5 sweep at the round-2 final build (tools/sweep.py, full)
timeout 2700 python tools/sweep.py > gpurun_out/sweep_r02.jsonl 2> gpurun_out/sweep_r02.err
wc -l gpurun_out/sweep_r02.jsonl
