P=$PWD/paper_1810_08403_b200
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "max or mpgcn or segment_max or ggnn or commnet" 2>&1 | tail -1
for i in 1 2 3; do
for n in "" _ab; do
echo "lib$n $(SG_LIB_PATH=$P/libsagann$n.so timeout 600 python tools/mp_time.py 2>&1 | tail -1)"
done; done
timeout 600 python tools/sweep.py --quick 2>&1 | grep -i max | head -8
