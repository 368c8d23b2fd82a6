for v in "DLA_GEMM_MASKED_TILE=128" "DLA_GEMM_MASKED_TILE=64"; do
  echo "== $v"
  env $v timeout 120 python tools/potrf_time.py 1024:8 4096:1 128:512 2048:1 512:8
  env $v timeout 120 python tools/gemm_time.py
  env $v timeout 120 python bench.py --no-cpu-baseline --no-also 2>&1 | tail -1 | cut -c1-120
  env $v timeout 200 python bench.py --config c5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-160
  env $v timeout 200 python bench.py --config c3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-160
done
