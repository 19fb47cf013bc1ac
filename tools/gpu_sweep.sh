timeout 2400 python tools/sweep.py > gpurun_out/sweep_full.jsonl 2> gpurun_out/sweep_full.err
wc -l gpurun_out/sweep_full.jsonl; tail -2 gpurun_out/sweep_full.err
