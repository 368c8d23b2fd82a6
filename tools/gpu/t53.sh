cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "syevd" 2>&1 | tail -3
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 2>/dev/null | cut -c1-400
