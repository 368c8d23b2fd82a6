cd /root/repo
for d in 1 2 3; do DLA_POTRF_DEPTH=$d python tools/potrf_check.py; done
