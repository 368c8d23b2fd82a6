mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/t4.log
cat gpurun_out/t4.log
for c in c1 potrf1024 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 2 2> gpurun_out/bench_$c.err | tee gpurun_out/bench_$c.json | cut -c1-600
  tail -3 gpurun_out/bench_$c.err
done
