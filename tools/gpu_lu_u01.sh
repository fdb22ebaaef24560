# A/B of the fused U01 kernel (DENSOLVE_LU_U01_FUSED=1, default) vs the TRSM / GEMM launch
# chain (=0); factors must hash the same in each pair.
for n in 4096 8192 16384 32768; do
  for f in 0 1 0 1; do
    DENSOLVE_LU_U01_FUSED=$f timeout 300 python tools/lu_rate.py $n 3 2>&1 | tail -1 | sed "s/^/u01=$f /"
  done
done
