mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_gp.py -x -q -m gpu 2>&1 | tail -15 > gpurun_out/t3.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
cat gpurun_out/t3.log; cat gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 1200 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-also --no-cpu-baseline > /dev/null 2>&1
wc -l gpurun_out/launches_c2.csv
