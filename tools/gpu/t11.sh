timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in c5 c1 c3 c4 potrf1024; do timeout 600 python bench.py --config $c --steps 5 --warmup 2 2>/dev/null | cut -c1-250; done
