mkdir -p gpurun_out
export DENSOLVE_SHARD_TIMEOUT_S=10
for cfg in "0,0 300" "0,0,0 301" "0,0,0,0 257" "0,0,0,0 1024" "0,0,0,0,0 300" "0,0,0,0,0,0,0,0 1000"; do
  set -- $cfg
  timeout 120 python tools/shard_debug.py $1 $2 2>&1 | tail -2
done
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q --durations=5 > gpurun_out/sh_tests.log 2>&1; echo "tests $?"; tail -12 gpurun_out/sh_tests.log
