for cfg in 0 1; do
echo "== cfg $cfg"
DLA_SYRK_CFG=$cfg timeout 120 python tools/syrk_time.py 2>&1 | head -6
DLA_SYRK_CFG=$cfg timeout 120 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_syrk_tma -c 1 python tools/syrk_time.py 2>&1 | grep -E "duration|tensor|warps_active" | head -12
DLA_SYRK_CFG=$cfg timeout 120 python tools/potrf_time.py 4096:1 1024:8 2048:1
done
DLA_SYRK_TMA=0 timeout 120 python tools/potrf_time.py 4096:1 1024:8 2048:1
