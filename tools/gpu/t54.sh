cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "gelqf or c5" 2>&1 | tail -5
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 2>/dev/null | cut -c1-700
timeout 600 python bench.py --config c5 --steps 3 --warmup 2 2>/dev/null | cut -c1-300
