P=$PWD/paper_1810_08403_b200
SG_LIB_PATH=$P/libsagann_ab12.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "ggcn or propagate" 2>&1 | tail -1
for i in 1 2; do
for n in "" _ab12 _ab16; do
echo "lib$n $(SG_LIB_PATH=$P/libsagann$n.so timeout 600 python tools/models_time.py 2>&1 | tail -1)"
echo "lib$n $(SG_LIB_PATH=$P/libsagann$n.so timeout 600 python tools/narrow_ab.py 256 384 2>&1 | tail -1)"
done; done
