# re-validate HEAD after the 8-warp GEMM epilogue: smoke, GPU suite, bench, reference arm, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rs -x 2>&1 | tail -30 > gpurun_out/v_pytest.txt
timeout 900 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/v_ref.json 2> gpurun_out/v_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/v_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-reorder --no-bf16 --no-noreuse > gpurun_out/v_launch_bench.log 2>&1
