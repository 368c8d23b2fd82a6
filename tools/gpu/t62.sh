cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/potrf_check.py 2>&1 | grep -v "relerr=[0-9.]*e-1[5-7]"
python tools/microbench.py --quick 2>&1 | grep -E "potrf_bwd n=4096|\"potrf n=4096|gemm 4096"
for c in c2 potrf1024 c3 c5; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-150; done
