for c in default 56 112 128 256 512 1024; do
  if [ $c = default ]; then python tools/gemv_small.py 4096; else DENSOLVE_GEMV_CHUNK=$c python tools/gemv_small.py 4096; fi
done 2>&1 | grep -v Warn
