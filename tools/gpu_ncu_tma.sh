# ncu --set full of the TMA DGEMM launches of one potrf pullback at n = 4096 (run under gpurun)
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_dgemm_tma" -c 4 -o gpurun_out/ncu_tma python tools/potrf_bwd_only.py 4096 1 1 > gpurun_out/ncu_tma.log 2>&1
ncu -i gpurun_out/ncu_tma.ncu-rep --page raw --csv > gpurun_out/ncu_tma_raw.csv 2>&1
ncu -i gpurun_out/ncu_tma.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_tma_src.csv 2>&1
