# L2 prefetch of the C tile in the DMMA GEMM (DLA_GEMM_CPREFETCH): rank-64 update, C2, potrf 1024 x 8
for v in 0 1; do
  echo "cpre=$v"
  DLA_GEMM_CPREFETCH=$v python tools/syrk_k64.py 2>&1 | head -2
  echo "  C2: $(DLA_GEMM_CPREFETCH=$v python bench.py --steps 20 --warmup 3 --no-also --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["parity"]["grad_rel"])')"
  echo "  potrf1024: $(DLA_GEMM_CPREFETCH=$v python bench.py --config potrf1024 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-160)"
done
