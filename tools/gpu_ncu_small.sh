# ncu --set full of the n <= 32 pullback kernel at batch 65536 (run under gpurun)
ncu --kernel-name regex:"k_potrf_bwd_dmma" -c 1 --set full --import-source on -o gpurun_out/ncu_small_bwd2 python tools/potrf_time.py 32:65536 > gpurun_out/ncu_small2.log 2>&1
ncu -i gpurun_out/ncu_small_bwd2.ncu-rep --page raw --csv > gpurun_out/ncu_small_raw2.csv 2>&1
ncu -i gpurun_out/ncu_small_bwd2.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_small_src2.csv 2>&1
