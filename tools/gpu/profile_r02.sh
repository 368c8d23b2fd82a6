# Round-2 profile set (run on one B200 via gpurun; outputs in gpurun_out/, summaries copied to profiles/)
set -x
mkdir -p gpurun_out
# 1. launch list of one C2 step (cold-cache serialized per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 400 --csv \
  --log-file gpurun_out/launches_c2_r02.csv python bench.py --steps 1 --warmup 2 --no-also --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
# 2. per-GEMM traffic + tensor activity in one C2 step
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:dgemm_dmma -s 200 -c 120 --csv --log-file gpurun_out/gemm_traffic_c2_r02.csv \
  python bench.py --steps 1 --warmup 2 --no-also --no-cpu-baseline > gpurun_out/ncu_t.log 2>&1
# 3. full captures of the top kernels
F="ncu --set full --clock-control none --import-source on"
timeout 600 $F -k regex:'dgemm_dmma<Cfg<64, 64, 32, 32, 16, 4>, true' -s 3 -c 1 -o gpurun_out/full_zgemm -f python tools/prof_gp.py > /dev/null 2>&1
timeout 600 $F -k regex:k_potrf_panel -s 100 -c 1 -o gpurun_out/full_panel -f python tools/prof_gp.py > /dev/null 2>&1
timeout 600 $F -k regex:k_rbf_bwd_sym -c 1 -o gpurun_out/full_rbfsym -f python tools/prof_gp.py > /dev/null 2>&1
timeout 600 $F -k regex:k_syrk_tma -s 1 -c 1 -o gpurun_out/full_syrktma -f python tools/syrk_time.py > /dev/null 2>&1
timeout 600 $F -k regex:k_syevd_small -c 1 -o gpurun_out/full_syevd -f python tools/prof_op.py syevd 64 1 1024 > /dev/null 2>&1
timeout 600 $F -k regex:k_kalman -c 1 -o gpurun_out/full_kalman -f python bench.py --config kalman --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 $F -k regex:k_chol_chain_warp -s 2 -c 1 -o gpurun_out/full_c1chain -f python tools/prof_c1_chain.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
