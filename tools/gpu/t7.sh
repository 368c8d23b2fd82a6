mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
python tools/microbench.py --quick 2>&1 | grep -E "potrf|trsm n=4096 nrhs=1\b|trsm n=4096 nrhs=4096 right=1 trans=0"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2> gpurun_out/bench_c2.err | cut -c1-400
