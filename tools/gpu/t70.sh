cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print([(x['dtype'], round(x['ms'],3)) for x in d['per_dtype']])"
timeout 600 compute-sanitizer --tool racecheck python tools/tc_check.py 2>&1 | grep -E "RACECHECK SUMMARY|worst"
timeout 600 compute-sanitizer --tool memcheck python tools/tc_check.py 2>&1 | grep -E "ERROR SUMMARY|worst"
