cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/microbench.py 2>&1 | grep -E "\"potrf n=(1024|4096)\"|potrf_bwd n=4096|n=128 batch=8192|n=32 batch=65536"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-200
timeout 600 python bench.py --config potrf1024 --steps 10 --warmup 3 2>/dev/null | cut -c1-300
