timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/microbench.py 2>&1 | grep -E "potrf_bwd n=4096|trsm n=4096 nrhs=4096|trmm n=4096|gemm 4096"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2> gpurun_out/bench_c2.err | cut -c1-250
