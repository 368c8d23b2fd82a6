# C2 step time vs the early-inverse T1 grid cap (DLA_GP_EARLY_CTAS)
for v in 0 148 222 296 444; do
  echo "cap=$v $(DLA_GP_EARLY_CTAS=$v python bench.py --steps 20 --warmup 3 --no-also --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["parity"]["grad_rel"])')"
done
