cd /root/repo
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_rbf_tiled|k_symcheck' -c 3 -o gpurun_out/prof_rbf -f python tools/prof_gp.py 4096 > gpurun_out/ncu_rbf.log 2>&1
tail -3 gpurun_out/ncu_rbf.log
