cd /root/repo
timeout 900 python -m pytest tests -x -q -m gpu -k "gelqf or gemm" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gelqf3.csv python tools/prof_op.py gelqf 128 1 256 > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/launches_gelqf3.csv 12
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 2>/dev/null | cut -c1-600
