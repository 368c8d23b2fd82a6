cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/microbench.py 2>&1 | grep -E "^.*potrf n=(1024|2048|4096)|trsm n=4096 nrhs=1|potrf_bwd n=4096\""
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-also 2> gpurun_out/bench_c2.err | cut -c1-200
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:k_potrf_panel' -s 30 -c 1 -o gpurun_out/prof_panel -f python tools/prof_op.py potrf 4096 2 > gpurun_out/ncu_panel.log 2>&1
tail -2 gpurun_out/ncu_panel.log
