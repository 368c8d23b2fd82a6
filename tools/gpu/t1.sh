set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -m gpu 2>&1 | tail -40 > gpurun_out/t1.log
cat gpurun_out/t1.log
