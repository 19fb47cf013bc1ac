# GEMM: is the converter warps' B-plane split on the critical path?  (gskip: B conversion skipped -- timing only)
L=paper_1810_08403_b200
for lib in libsagann.so libsagann_gskip.so libsagann.so libsagann_gskip.so; do
  echo "== $lib" >> gpurun_out/gm.txt
  SG_LIB_PATH=$PWD/$L/$lib timeout 300 python tools/gemm_bench.py >> gpurun_out/gm.txt 2>&1
done
