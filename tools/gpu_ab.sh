SG_LIB_PATH=$PWD/paper_1810_08403_b200/libsagann_ab.so timeout 300 python tools/narrow_ab.py 602 768 1024 2>&1 | grep -v Warn | tail -1
SG_LIB_PATH=$PWD/paper_1810_08403_b200/libsagann_ab6.so timeout 300 python tools/narrow_ab.py 602 768 1024 2>&1 | grep -v Warn | tail -1
timeout 300 python tools/narrow_ab.py 602 2>&1 | grep -v Warn | tail -1
