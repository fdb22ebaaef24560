mkdir -p gpurun_out
export DENSOLVE_SHARD_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q --durations=5 > gpurun_out/sh_tests.log 2>&1; echo "tests $?"; tail -30 gpurun_out/sh_tests.log
timeout 600 python tools/shard_gmres_rate.py 65536 50 f32 2>&1 | tail -4
timeout 600 python tools/shard_gmres_rate.py 32768 30 f64 2>&1 | tail -4
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:gemm64 -s 1 -c 1 -o gpurun_out/gemm_full_r02d -f python tools/profile_run.py gemm 16384 16384 512 > /dev/null 2>&1; echo "gemm full $?"
