mkdir -p gpurun_out
# one full capture of the dominant kernel (128x128-tile DMMA GEMM) inside potrf_bwd n=4096
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:Cfg<\(int\)128' -s 2 -c 2 \
   -o gpurun_out/prof_gemm -f python tools/prof_op.py potrf_bwd 4096 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out/*.ncu-rep
