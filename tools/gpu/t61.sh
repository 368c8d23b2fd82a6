cd /root/repo
for lib in libdla_b200_def.so libdla_b200_all.so; do
  export DLA_LIB_PATH=/root/repo/paper_1710_08717_b200/$lib
  echo $lib
  python tools/microbench.py --quick 2>&1 | grep -E "potrf_bwd n=4096|\"potrf n=4096|trsm n=4096 nrhs=4096 right=0 trans=0|gemm 4096|trmm"
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-130
done
