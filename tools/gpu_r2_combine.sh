# A/B: combine-launch loads in flight (U=16 default vs U=8: libsagann_u8.so), wide rows at 5 blocks/SM
# (libsagann_b5.so); N=8 proxy at T = auto / 512 / 2048 with the default build
L=paper_1810_08403_b200
for i in 1 2; do
for lib in libsagann_u8.so libsagann.so libsagann_b5.so; do
  SG_LIB_PATH=$PWD/$L/$lib timeout 600 python tools/sched_ab.py reddit >> gpurun_out/u_ab.jsonl 2>> gpurun_out/u_ab.err
done
done
timeout 900 python tools/dist_proxy.py reddit 1 8 >> gpurun_out/u_proxy.jsonl 2>> gpurun_out/u_proxy.err
SG_LIB_PATH=$PWD/$L/libsagann_u8.so timeout 900 python tools/dist_proxy.py reddit 8 >> gpurun_out/u_proxy.jsonl 2>> gpurun_out/u_proxy.err
for T in 512 2048; do
  SG_PROXY_SPLIT=$T timeout 900 python tools/dist_proxy.py reddit 8 >> gpurun_out/u_proxy.jsonl 2>> gpurun_out/u_proxy.err
done
