mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgemm_dmma -s 3 -c 1 -o gpurun_out/syrk64 -f python tools/potrf_time.py 4096:1 > gpurun_out/ncu_syrk.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_rbf_tiled|k_kskinny|k_square|k_add_transpose' -c 6 -o gpurun_out/gpmisc -f python tools/timeline_gp.py /tmp/x.json > gpurun_out/ncu_gpmisc.log 2>&1
ls -la gpurun_out/*.ncu-rep
