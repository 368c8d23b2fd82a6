cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 1200 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-also --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_c2.csv 25
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c5.csv python tools/prof_c5.py 8192 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_c5.csv 30
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_p1024.csv python tools/prof_op.py potrf 1024 2 8 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_p1024.csv 15
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_p1024b.csv python tools/prof_op.py potrf_bwd 1024 2 8 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_p1024b.csv 15
timeout 600 python tools/microbench.py 2>&1 | tail -40
