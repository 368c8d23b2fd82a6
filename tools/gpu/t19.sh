cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "potrf" 2>&1 | tail -2
for m in 1 2; do echo "MINB=$m"; DLA_WARP_MINB=$m python tools/microbench.py 2>&1 | grep -E "n=32 batch=65536"; done
