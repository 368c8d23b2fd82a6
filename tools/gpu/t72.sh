cd /root/repo
for v in "DLA_POTRF_NB=64" "DLA_POTRF_NB=128" "DLA_POTRF_MODE=3"; do
  echo $v
  env $v python tools/graph_vs_eager.py
  env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-110
done
