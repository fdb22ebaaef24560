for ns in 32 200 1000; do DENSOLVE_GMRES_POLL_NS=$ns timeout 120 python tools/gemv_small.py 4096 2>&1 | grep -v Warn | tail -1 | sed "s/^/poll=$ns /"; done
DENSOLVE_GEMV_CHUNK=112 timeout 120 python tools/gemv_small.py 4096 2>&1 | grep -v Warn | tail -1 | sed "s/^/chunk112 /"
DENSOLVE_GEMV_CHUNK=256 timeout 120 python tools/gemv_small.py 4096 2>&1 | grep -v Warn | tail -1 | sed "s/^/chunk256 /"
DENSOLVE_GMRES_PERSIST=0 timeout 120 python tools/gemv_small.py 4096 2>&1 | grep -v Warn | tail -1 | sed "s/^/nopersist /"
