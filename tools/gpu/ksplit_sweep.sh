# intra-CTA split-K (CfgS2) for triangular / masked products: tests, then the
# potrf 1024 x 8 and C2 lines against DLA_GEMM_KSPLIT
python -m pytest tests/test_gpu_ops.py tests/test_gpu_golden_big.py tests/test_gpu_gp.py tests/test_gpu_gemm_tma.py -x -q 2>&1 | tail -2
for v in 0 256 512 1024; do
  echo "ksplit=$v potrf1024: $(DLA_GEMM_KSPLIT=$v python bench.py --config potrf1024 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d.get("split_api"))' 2>&1 | cut -c1-300)"
done
for v in 0 512; do
  echo "ksplit=$v C2: $(DLA_GEMM_KSPLIT=$v python bench.py --steps 20 --warmup 3 --no-also --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["parity"]["grad_rel"])')"
done
