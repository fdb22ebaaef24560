for w in 0 4 2; do DENSOLVE_GEMV_WIDE=$w timeout 120 python tools/gemv_small.py 4096 2>&1 | grep -v Warn | tail -1 | sed "s/^/wide=$w /"; done
DENSOLVE_GEMV_WIDE=4 timeout 600 python -m pytest tests/test_gpu_krylov.py -q -x 2>&1 | tail -2
