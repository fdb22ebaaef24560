# A/B of the trailing-GEMM SM reservation beside the LU look-ahead panel (DENSOLVE_LU_RESERVE
# = 0 off, r = reserve while the predicted GEMM time <= r x the side stream's); factors must
# hash the same in every row.
for n in 16384 32768; do
  for r in 0 1 2 0 1; do
    DENSOLVE_LU_RESERVE=$r timeout 300 python tools/lu_rate.py $n 3 2>&1 | tail -1
  done
done
