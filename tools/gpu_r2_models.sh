# model families (tools/models_time.py) with evict_last (default) vs ld.global.nc row loads; BlogCatalog x10 split T auto vs 4096
L=paper_1810_08403_b200
for rep in 1 2; do
for lib in libsagann.so libsagann_ld0.so; do
  echo "$lib $(SG_LIB_PATH=$PWD/$L/$lib timeout 600 python tools/models_time.py 2>/dev/null)" >> gpurun_out/mt.txt
done
done
for T in auto 4096 1024; do
  timeout 600 python bench.py --config blogcatalog10 --no-cpu-baseline --no-noreuse --no-reorder --no-bf16 --split-edges $T | python -c "import json,sys; b=json.load(sys.stdin); print('blogcatalog T=$T', b['ms_per_step'], b['stages_ms'])" >> gpurun_out/mt.txt 2>> gpurun_out/mt.err
done
