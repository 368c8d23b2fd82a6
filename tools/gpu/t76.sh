cd /root/repo
python tools/potrf_check.py 2>&1 | grep -v "relerr=[0-9.]*e-1[5-7]"
timeout 900 python -m pytest tests -x -q -m gpu -k "potrf or gp or c5 or chain" 2>&1 | tail -1
python tools/graph_vs_eager.py
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-110
python bench.py --config potrf1024 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], [(x['batch'], round(x['ms'],2)) for x in d['batch_sweep']])"
