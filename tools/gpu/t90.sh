python -m pytest tests -x -q -m gpu -k "gp or potrf or chain" 2>&1 | tail -1
for i in 1 2 3; do for L in libdla_alt.so libdla_b200.so; do echo -n "$L "; DLA_LIB_PATH=paper_1710_08717_b200/$L python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],3))"; done; done
