# launch list of one C2 step (skip the first eval's launches)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 1200 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-also --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/ncu_bench.log
wc -l gpurun_out/launches_c2.csv
