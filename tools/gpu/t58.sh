cd /root/repo
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:Cfg<\(int\)128, \(int\)128, \(int\)64, \(int\)32, \(int\)32>, \(bool\)1' -c 2 -o gpurun_out/prof_gemm -f python tools/prof_op.py potrf_bwd 4096 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_potrf_panel|k_trsv' -s 1 -c 2 -o gpurun_out/prof_panel2 -f python tools/prof_op.py trsv 4096 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
