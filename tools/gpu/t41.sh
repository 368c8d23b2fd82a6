cd /root/repo
timeout 600 python -m pytest tests -x -q -m gpu -k "trsv or trsm or gp or potrf_forward" 2>&1 | tail -3
timeout 300 python tools/microbench.py --quick 2>&1 | grep -E "nrhs=1"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-200
