cd /root/repo
for lib in libdla_b200_m.so libdla_b200_s4.so libdla_b200_s4k512.so; do
  export DLA_LIB_PATH=/root/repo/paper_1710_08717_b200/$lib
  echo $lib
  python tools/potrf_check.py 2>&1 | grep -v "relerr=[0-9.]*e-1[5-7]"
  python tools/graph_vs_eager.py
  python tools/microbench.py 2>&1 | grep -E "potrf_bwd n=(1024|4096)|trsm n=4096 nrhs=4096 right=0 trans=0|n=128 batch=8192|n=32 batch"
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-130
  python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | cut -c1-130
  python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | cut -c1-130
done
