for f in 0 1 2 3; do
  echo "== DLA_GEMM_FORCE=$f"
  DLA_GEMM_FORCE=$f timeout 120 python tools/potrf_time.py 1024:8 4096:1 128:512
  DLA_GEMM_FORCE=$f timeout 120 python bench.py --no-cpu-baseline --no-also 2>&1 | tail -1 | cut -c1-120
done
