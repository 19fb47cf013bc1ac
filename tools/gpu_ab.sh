P=$PWD/paper_1810_08403_b200
for i in 1 2; do
for n in "" _ab _ab2; do
echo "lib$n $(SG_LIB_PATH=$P/libsagann$n.so timeout 600 python tools/narrow_ab.py 602 768 2>&1 | tail -1)"
done; done
