P=$PWD/paper_1810_08403_b200
SG_LIB_PATH=$P/libsagann_ab.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "max or mpgcn or segment_max" 2>&1 | tail -1
for i in 1 2; do
for n in "" _ab; do
echo "lib$n $(SG_LIB_PATH=$P/libsagann$n.so timeout 600 python tools/mp_time.py 2>&1 | tail -1)"
done; done
