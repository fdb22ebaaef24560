mkdir -p gpurun_out
export DENSOLVE_SHARD_TIMEOUT_S=60
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q -k edge > gpurun_out/sh_tests.log 2>&1; echo "tests $?"; tail -25 gpurun_out/sh_tests.log
