ncu --set full --clock-control none --import-source on -k regex:k_potrf_panel -s 40 -c 1 -o gpurun_out/panel_r01 python tools/panel_phases.py 4096 > gpurun_out/ncu_panel.log 2>&1
ncu -i gpurun_out/panel_r01.ncu-rep --page raw --csv > gpurun_out/panel_raw.csv 2>&1
ncu -i gpurun_out/panel_r01.ncu-rep --page source --csv --print-source sass > gpurun_out/panel_src.csv 2>&1
tail -3 gpurun_out/ncu_panel.log; ls -la gpurun_out/panel*
