cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cut -c1-300 gpurun_out/bench_c2.json
for c in c1 potrf1024 c3 c4 c5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; cut -c1-150 gpurun_out/bench_$c.json; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; cut -c1-150 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 700 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-also --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_c2.csv 8
CUDA_MODULE_LOADING=EAGER timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_cases.py 2>&1 | grep -E "ERROR SUMMARY" | head -3
CUDA_MODULE_LOADING=EAGER timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_cases.py 2>&1 | grep -E "ERROR SUMMARY|RACE" | head -3
