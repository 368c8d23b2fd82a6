b() { python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],3))"; }
for cfg in "" "DLA_POTRF_RESERVE=16" "DLA_POTRF_RESERVE=40" "DLA_POTRF_GROUP=2" "DLA_POTRF_PRIO=0" ""; do echo -n "[$cfg] "; env $cfg bash -c "$(declare -f b); b"; done
