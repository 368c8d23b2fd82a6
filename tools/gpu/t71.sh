cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "gemm or trmm or trsm or potrf or gelqf or syrk" 2>&1 | tail -1
for tc in 0 1; do DLA_SGEMM_TC=$tc python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print([(x['dtype'], round(x['ms'],3)) for x in d['per_dtype']])"; done
CUDA_MODULE_LOADING=EAGER timeout 600 compute-sanitizer --tool memcheck python tools/tc_check.py 2>&1 | grep -E "ERROR SUMMARY"
