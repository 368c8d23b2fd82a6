cd /root/repo
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:dgemm_dmma -s 250 -c 250 --csv --log-file gpurun_out/gemm_traffic.csv python bench.py --steps 1 --warmup 0 --no-also --no-cpu-baseline > /dev/null 2>&1
wc -l gpurun_out/gemm_traffic.csv
