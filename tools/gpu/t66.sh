cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "potrf or gp or c5" 2>&1 | tail -2
python tools/microbench.py 2>&1 | grep -E "potrf_bwd n=(1024|4096)|n=128 batch=8192"
python bench.py --config potrf1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-200
python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | cut -c1-200
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-150
