python tools/shard_gmres_trace.py 65536 50 f32 2>&1 | tail -3
DENSOLVE_SHARD_TRACE=1 python tools/shard_gmres_trace.py 65536 50 f32 2> gpurun_out/shgm_trace.txt | tail -2
grep -c wait gpurun_out/shgm_trace.txt; head -5 gpurun_out/shgm_trace.txt; tail -5 gpurun_out/shgm_trace.txt
