timeout 120 python tools/gemv_small.py 4096 2>&1 | grep -v Warn | tail -1
timeout 600 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_config_parity.py -q -x -k "gmres or GMRES" 2>&1 | tail -2
