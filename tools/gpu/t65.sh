cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "split or gp or potrf_backward" 2>&1 | tail -2
for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-150; done
python tools/timeline_gp.py 2>&1 | grep -v -i warn | tail -12
