timeout 900 python -m pytest tests/test_gpu_direct.py tests/test_gpu_panel_kernels.py tests/test_gpu_cholesky.py -q -x 2>&1 | tail -2
python tools/lu_rate.py 16384 3 2>&1 | grep "LU n"
python tools/lu_rate.py 32768 2 2>&1 | grep "LU n"
