cd /root/repo
mkdir -p gpurun_out
cd tools/peaks
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1710_08717_b200/csrc -o chol_bench chol_bench.cu && ./chol_bench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1710_08717_b200/csrc -o lat lat.cu && ./lat
cd /root/repo
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:k_potrf_panel' -s 4 -c 1 -o gpurun_out/prof_panel -f python tools/prof_op.py potrf 4096 2 > gpurun_out/ncu_panel.log 2>&1
tail -2 gpurun_out/ncu_panel.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:k_trsv' -c 1 -o gpurun_out/prof_trsv -f python tools/prof_op.py trsv 4096 2 > gpurun_out/ncu_trsv.log 2>&1
tail -2 gpurun_out/ncu_trsv.log
