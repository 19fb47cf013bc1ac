timeout 300 python tools/narrow_ab.py 16 64 128 2>&1 | grep env
for d in 16 32; do SG_LIB_PATH=$PWD/paper_1810_08403_b200/libsagann_b1d$d.so timeout 300 python tools/narrow_ab.py 16 64 128 2>&1 | grep env; done
