# GEMM converter warps 4 (default) vs 8: error-bound tests on the variant, shape timings
L=paper_1810_08403_b200
SG_LIB_PATH=$PWD/$L/libsagann_cw8.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "gemm" 2>&1 | tail -2 > gpurun_out/cw_test.txt
SG_LIB_PATH=$PWD/$L/libsagann_cw8.so timeout 900 python -m pytest tests/test_gpu_bf16.py -q -k "gemm" 2>&1 | tail -2 >> gpurun_out/cw_test.txt
for lib in libsagann.so libsagann_cw8.so libsagann.so libsagann_cw8.so; do
  echo "== $lib" >> gpurun_out/cw.txt
  SG_LIB_PATH=$PWD/$L/$lib timeout 300 python tools/gemm_bench.py >> gpurun_out/cw.txt 2>&1
done
