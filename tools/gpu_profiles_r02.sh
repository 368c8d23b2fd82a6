# Round-2 profile refresh (run under gpurun): C2 launch list (serialised,
# cold-cache per-launch times) + ncu --set full captures of this round's new
# kernels at their bench shapes.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_r02c.csv python bench.py --steps 2 --warmup 1 --no-also --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_potrf_bwd_dmma|k_potrf128|k_trtri128|k_chol_chain_dmma|k_matvec_rows" -c 6 -o gpurun_out/ncu_full_r02c python tools/sanitize_cases.py > /dev/null 2>&1
python tools/potrf_bwd_only.py 32 65536 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_potrf_bwd_dmma" -c 1 -o gpurun_out/ncu_full_bwd32_r02c python tools/potrf_bwd_only.py 32 65536 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:"k_trtri128|k_potrf128" -c 2 -o gpurun_out/ncu_full_128_r02c python tools/timeline_c5.py 2048 > /dev/null 2>&1
ls -la gpurun_out/
