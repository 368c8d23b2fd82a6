ncu --set full --clock-control none --import-source on -k regex:k_chol_chain_warp -s 2 -c 1 -o gpurun_out/c1_r01 python tools/prof_c1_chain.py > gpurun_out/ncu_c1.log 2>&1
ncu -i gpurun_out/c1_r01.ncu-rep --page raw --csv > gpurun_out/c1_raw.csv 2>&1
ncu -i gpurun_out/c1_r01.ncu-rep --page source --csv --print-source sass > gpurun_out/c1_src.csv 2>&1
tail -2 gpurun_out/ncu_c1.log
