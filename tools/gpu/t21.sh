cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/prof_c5.py 8192 > /dev/null 2>&1
wc -l gpurun_out/c5_launches.csv
