cd /root/repo
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_chol_chain_warp|k_syevd_small|k_lq_panel|k_potrf_panel|k_trsv' -c 6 -o gpurun_out/prof_misc -f python tools/prof_misc.py > /dev/null 2>&1
ls -la gpurun_out/prof_misc.ncu-rep
