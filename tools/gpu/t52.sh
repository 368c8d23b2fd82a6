cd /root/repo
for g in 1 2 3 4; do echo "group $g"; export DLA_POTRF_GROUP=$g; python tools/potrf_check.py 2>&1 | grep -v "relerr=[0-9.]*e-1[5-7]" ; python tools/graph_vs_eager.py; python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-130; done
