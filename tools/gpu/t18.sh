cd /root/repo
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:k_potrf_(bwd_)?warp' -c 2 -o gpurun_out/prof_warp -f python tools/prof_op.py potrf_bwd 32 1 65536 > gpurun_out/ncu_warp.log 2>&1
tail -2 gpurun_out/ncu_warp.log
