cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for p in 0 1; do echo "PRIO=$p"; DLA_POTRF_PRIO=$p python tools/microbench.py 2>&1 | grep -E "^.*potrf n=(1024|2048|4096)"; DLA_POTRF_PRIO=$p timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2> gpurun_out/bench_c2.err | cut -c1-200; done
