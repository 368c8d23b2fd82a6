cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "c5 or gemm or chain or gp" 2>&1 | tail -2
python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python tools/prof_c5.py 8192 > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/launches_c5.csv 30 | grep -E "total|skinny|ml_"
