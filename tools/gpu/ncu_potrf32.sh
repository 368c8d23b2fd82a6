# one full ncu capture of the n = 32 warp-per-matrix forward at 65536 x 32^2 fp64
mkdir -p gpurun_out
python tools/potrf32_once.py > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_potrf_warp -s 1 -c 1 \
   -o gpurun_out/ncu_potrf32_r02f -f python tools/potrf32_once.py > gpurun_out/ncu_potrf32.log 2>&1
tail -2 gpurun_out/ncu_potrf32.log
