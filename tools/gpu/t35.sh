cd /root/repo
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/microbench.py 2>&1 | grep -E "gemm 4096|potrf_bwd n=4096|trmm n=4096|\"potrf n=4096|n=128 batch=8192"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2> gpurun_out/bench_c2.err | cut -c1-200
