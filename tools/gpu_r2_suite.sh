# full GPU suite + smoke at HEAD
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s_smoke.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rs 2>&1 | grep -E "passed|failed|SKIPPED|FAILED|Error" > gpurun_out/s_pytest.txt
