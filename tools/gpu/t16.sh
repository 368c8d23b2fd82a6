cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python tools/microbench.py 2>&1 | grep -E "batch=65536|n=32 batch=1|n=1024\"|potrf n=4096"
for c in c1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-220; done
