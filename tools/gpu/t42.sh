cd /root/repo
timeout 600 python -m pytest tests -x -q -m gpu -k "trsv or trsm" 2>&1 | tail -2
timeout 300 python tools/microbench.py --quick 2>&1 | grep -E "nrhs=1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_trsv.csv python tools/prof_op.py trsv 4096 3 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_trsv.csv 6 | grep trsv
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:k_trsv' -c 1 -o gpurun_out/prof_trsv2 -f python tools/prof_op.py trsv 4096 2 > /dev/null 2>&1
