timeout 300 python tools/gemm_bench.py 2>&1 | tail -5
for kb in 64 100; do echo "== smem $kb KB"; SG_LIB_PATH=$PWD/paper_1810_08403_b200/libsagann_g$kb.so timeout 300 python tools/gemm_bench.py 2>&1 | tail -5; done
