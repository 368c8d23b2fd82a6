cd /root/repo
for d in 1 2 3; do echo "depth $d"; DLA_POTRF_DEPTH=$d python tools/potrf_content.py; DLA_POTRF_DEPTH=$d python tools/graph_vs_eager.py; DLA_POTRF_DEPTH=$d python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-130; done
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
