timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -3
timeout 300 python tools/shard_gmres_rate.py 65536 50 f32 2>&1 | tail -3
timeout 300 python tools/shard_gmres_rate.py 32768 30 f64 2>&1 | tail -3
