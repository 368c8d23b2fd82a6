cd /root/repo
mkdir -p gpurun_out
for p in 1 2 3; do DLA_TILES_PER_SM=$p ./tools/peaks/tiles_trace 4096 > gpurun_out/tiles_trace_4096_p$p.csv 2>/dev/null; DLA_TILES_PER_SM=$p ./tools/peaks/tiles_trace 1024 > gpurun_out/tiles_trace_1024_p$p.csv 2>/dev/null; done
