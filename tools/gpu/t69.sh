cd /root/repo
for tc in 0 1; do
  export DLA_SGEMM_TC=$tc
  echo "DLA_SGEMM_TC=$tc"
  python tools/tc_check.py 2>&1 | tail -1
  python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print([(x['dtype'], round(x['ms'],3)) for x in d['per_dtype']])"
done
unset DLA_SGEMM_TC
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
