cd /root/repo
timeout 300 python -m pytest tests -x -q -m gpu -k "potrf" 2>&1 | tail -3
for m in 2 3; do echo "MODE=$m"; DLA_POTRF_MODE=$m timeout 300 python tools/microbench.py 2>&1 | grep -E "\"potrf n=(1024|4096)\""; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2> gpurun_out/bench_c2.err | cut -c1-200
