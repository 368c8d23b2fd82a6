for L in libdla_b200.so; do echo "== $L"; DLA_LIB_PATH=paper_1710_08717_b200/$L python tools/kernel_times_gp.py 2>&1 | grep -v -i warn | grep -E "square|tri_copy|add_trans|sumlogdiag|finalize"; done
for i in 1 2; do for L in libdla_alt.so libdla_b200.so; do echo -n "$L "; DLA_LIB_PATH=paper_1710_08717_b200/$L python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],3))"; done; done
python -m pytest tests -x -q -m gpu 2>&1 | tail -2
