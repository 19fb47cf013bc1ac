P=$PWD/paper_1810_08403_b200
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1
for i in 1 2; do
for n in "" _ab; do
echo "lib$n $(SG_LIB_PATH=$P/libsagann$n.so timeout 600 python tools/narrow_ab.py 160 256 384 512 2>&1 | tail -1)"
done; done
for n in "" _ab; do echo "lib$n $(SG_LIB_PATH=$P/libsagann$n.so timeout 600 python bench.py --config pubmed --steps 20 --no-cpu-baseline --no-e2e --no-reorder 2>/dev/null | python -c 'import sys,json; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')"; done
