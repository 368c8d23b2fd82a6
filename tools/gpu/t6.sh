mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_potrf.csv python tools/prof_op.py potrf 4096 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_trsv.csv python tools/prof_op.py trsv 4096 1 > /dev/null 2>&1
ls -la gpurun_out/
