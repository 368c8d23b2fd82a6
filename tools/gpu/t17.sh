cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "potrf" 2>&1 | tail -3
python tools/microbench.py 2>&1 | grep -E "n=32 batch=65536"
