cd /root/repo
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for m in 2 3; do echo "MODE=$m"; DLA_POTRF_MODE=$m timeout 300 python tools/microbench.py 2>&1 | grep -E "\"potrf n=(1024|4096)\""; done
./tools/peaks/tiles_trace 4096 > gpurun_out/tiles_trace_4096.csv 2>/dev/null
./tools/peaks/tiles_trace 1024 > gpurun_out/tiles_trace_1024.csv 2>/dev/null
