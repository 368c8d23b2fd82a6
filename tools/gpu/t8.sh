mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
python tools/microbench.py 2>&1 | grep -E "potrf|trsm n=4096|n=1024" | grep -v graph
for c in c5 potrf1024; do timeout 600 python bench.py --config $c --steps 5 --warmup 2 2>/dev/null | cut -c1-300; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2> gpurun_out/bench_c2.err | cut -c1-300
