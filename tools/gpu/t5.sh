mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/t5.log
cat gpurun_out/t5.log
python tools/microbench.py --quick 2>&1 | tail -30
