# evict_last row loads as default: full GPU suite, smoke, bench lines (reddit + bf16 + configs)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ld_smoke.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rs 2>&1 | grep -E "passed|failed|SKIPPED|FAILED|Error" > gpurun_out/ld_pytest.txt
timeout 900 python bench.py > gpurun_out/ld_bench.json 2> gpurun_out/ld_bench.err
for c in blogcatalog10 powerlaw_gcn powerlaw_ggcn; do
  timeout 1200 python bench.py --config $c --no-cpu-baseline --no-noreuse --no-reorder --no-bf16 > gpurun_out/ld_bench_$c.json 2> gpurun_out/ld_bench_$c.err
done
timeout 600 python tools/models_time.py > gpurun_out/ld_models.txt 2>&1
