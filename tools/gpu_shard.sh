mkdir -p gpurun_out
export DENSOLVE_SHARD_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/sh_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/sh_tests.log
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 120 python tools/shard_debug.py 0,0,0,0,0,0,0,0 1000 2>&1 | tail -2
timeout 300 python tools/shard_rate.py 32768 100 2>&1 | tail -3
