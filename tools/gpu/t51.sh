cd /root/repo
python tools/potrf_check.py
python tools/potrf_content.py
python tools/graph_vs_eager.py
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-130
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
