cd /root/repo
timeout 600 python -m pytest tests -x -q -m gpu -k "chain or potrf_warp" 2>&1 | tail -4
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 2>gpurun_out/c1.err > gpurun_out/bench_c1.json; cat gpurun_out/bench_c1.json | cut -c1-1500; tail -3 gpurun_out/c1.err
