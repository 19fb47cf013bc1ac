ncu --set full --clock-control none --import-source on -k regex:prop_kernel --launch-skip 6 --launch-count 4 -o /tmp/ggcn_blog python tools/profile_step.py blogcatalog10 2 > /tmp/ncu_blog.log 2>&1
python tools/ncu_summary.py report /tmp/ggcn_blog.ncu-rep > gpurun_out/ggcn_blog.txt
ncu -i /tmp/ggcn_blog.ncu-rep --page source --csv --print-source sass -k regex:prop_kernel --launch-count 1 > gpurun_out/ggcn_blog_src.csv 2>&1
ncu --set full --clock-control none -k regex:prop_kernel --launch-skip 6 --launch-count 4 -o /tmp/ggcn_pl python tools/profile_step.py powerlaw_ggcn 2 2.5e8 > /tmp/ncu_pl.log 2>&1
python tools/ncu_summary.py report /tmp/ggcn_pl.ncu-rep > gpurun_out/ggcn_pl.txt
ls -la gpurun_out
