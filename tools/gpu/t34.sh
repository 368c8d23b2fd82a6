cd /root/repo
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-also > /dev/null 2>&1
