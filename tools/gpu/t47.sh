cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "potrf or gp or chain or potri" 2>&1 | tail -2
for d in 1 2 3 4; do
  echo "depth $d"
  export DLA_POTRF_DEPTH=$d
  timeout 300 python tools/microbench.py 2>&1 | grep -E "\"potrf n=(1024|4096)\""
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-150
  timeout 600 python bench.py --config potrf1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-200
done
