for nb in 512 384 256 768; do
  DENSOLVE_LU_NB=$nb python tools/lu_rate.py 16384 2 2>&1 | grep "LU n" | sed "s/^/NB=$nb /"
done
for nb in 512 768; do
  DENSOLVE_LU_NB=$nb python tools/lu_rate.py 32768 2 2>&1 | grep "LU n" | sed "s/^/NB=$nb /"
done
