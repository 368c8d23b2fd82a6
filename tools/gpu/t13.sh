cd /root/repo
./tools/peaks/chol_bench 2>&1 | tail -16
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for nb in 64 128; do echo "NB=$nb"; DLA_POTRF_NB=$nb python tools/microbench.py 2>&1 | grep -E "^.*potrf n=(1024|2048|4096)"; done
for nb in 64 128; do echo "NB=$nb"; DLA_POTRF_NB=$nb timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2> gpurun_out/bench_c2.err | cut -c1-200; done
