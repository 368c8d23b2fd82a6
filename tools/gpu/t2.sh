set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_gp.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/t2.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/t2.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
cat gpurun_out/t2.log; cat gpurun_out/bench_c2.json; tail -20 gpurun_out/bench_c2.err
