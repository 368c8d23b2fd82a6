cd /root/repo
mkdir -p gpurun_out
./tools/peaks/tiles_trace 4096 > gpurun_out/tiles_trace_4096.csv
./tools/peaks/tiles_trace 1024 > gpurun_out/tiles_trace_1024.csv
