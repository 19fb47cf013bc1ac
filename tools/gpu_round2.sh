timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
ncu --set full --clock-control none --import-source on -k regex:prop_kernel --launch-skip 6 --launch-count 4 -o /tmp/ggcn_blog python tools/profile_step.py blogcatalog10 2 > /tmp/ncu_blog.log 2>&1
python tools/ncu_summary.py report /tmp/ggcn_blog.ncu-rep > gpurun_out/ggcn_blog_after.txt
