cd /root/repo
for lib in libdla_b200_k32.so libdla_b200_k16.so; do
  echo $lib
  export DLA_LIB_PATH=/root/repo/paper_1710_08717_b200/$lib
  timeout 300 python tools/microbench.py 2>&1 | grep -E "\"potrf n=(1024|4096)\"|potrf_bwd n=(1024|4096)|n=128 batch=8192|gemm 4096"
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2>/dev/null | cut -c1-150
  timeout 600 python bench.py --config potrf1024 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-200
done
