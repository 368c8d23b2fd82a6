cd /root/repo
mkdir -p gpurun_out
for spec in "syevd 64 1 1024" "gelqf 128 1 256"; do
  set -- $spec
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python tools/prof_op.py $spec > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/launches_$1.csv 12
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:k_potrf_warp|k_potrf_bwd_warp' -s 2 -c 2 -o gpurun_out/prof_warp32 -f python tools/prof_op.py potrf 32 3 65536 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:k_potrf_bwd_warp' -c 1 -o gpurun_out/prof_warp32b -f python tools/prof_op.py potrf_bwd 32 2 65536 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:syevd' -c 2 -o gpurun_out/prof_syevd -f python tools/prof_op.py syevd 64 1 1024 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:gelqf' -c 1 -o gpurun_out/prof_gelqf -f python tools/prof_op.py gelqf 128 1 256 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
