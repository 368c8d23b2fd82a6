cd /root/repo
for lib in libdla_b200_bp32.so libdla_b200_bp16.so; do
  export DLA_LIB_PATH=/root/repo/paper_1710_08717_b200/$lib
  echo $lib
  timeout 900 python -m pytest tests -x -q -m gpu -k "gelqf" 2>&1 | tail -1
  timeout 600 python bench.py --config c3 --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print([(x['dtype'], round(x['ms'],3)) for x in d['per_dtype']])"
done
