cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "potrf or gemm or gp" 2>&1 | tail -2
for r in 0 32 -1 96; do
  echo "reserve $r"
  DLA_POTRF_RESERVE=$r timeout 300 python tools/microbench.py --quick 2>&1 | grep -E "\"potrf n=4096\""
  DLA_POTRF_RESERVE=$r timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-150
done
