cd /root/repo
python tools/graph_vs_eager.py
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['ms_per_step_eager'])"
