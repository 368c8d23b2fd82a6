for z in 50 75 90 100; do
  echo "== ZERO_AT=$z"; DLA_POTRF_ZERO_AT=$z python tools/potrf_time.py 4096:1 1024:8 2>&1 | cut -c1-60
done
python bench.py 2>&1 | grep "^{" | cut -c1-160
