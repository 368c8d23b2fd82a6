cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "potrf or c5 or gp or chain" 2>&1 | tail -1
python tools/potrf_check.py 2>&1 | grep -v "relerr=[0-9.]*e-1[5-7]"
python tools/microbench.py 2>&1 | grep -E "n=128 batch=8192"
python bench.py --config potrf1024 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], [(x['batch'], round(x['ms'],2), round(x['frac_of_fp64_peak'],3)) for x in d['batch_sweep']])"
python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | cut -c1-150
