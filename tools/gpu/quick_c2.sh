# C2 step timing (+ variants by env) and one GP kernel timeline
timeout 300 python -m pytest tests -m gpu -x -q -k "gp or golden or potrf_modes or c5" 2>&1 | tail -2
for v in "" "DLA_GP_FUSED_TAIL=0"; do
  env $v timeout 120 python bench.py --no-cpu-baseline --no-also 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('C2 [$v]', d['ms_per_step'], d['e2e']['ms_per_step'], d['parity'])"
done
timeout 120 python tools/timeline_gp.py gpurun_out/tlgp.json > /dev/null 2>&1
