# one full ncu capture of the Kalman kernel at the bench shape (4096 x (h = d = 8, T = 128))
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_kalman -c 1 \
   -o gpurun_out/ncu_kalman_r02f -f python bench.py --config kalman --steps 1 --warmup 3 --no-cpu-baseline \
   > gpurun_out/ncu_kalman.log 2>&1
tail -2 gpurun_out/ncu_kalman.log
