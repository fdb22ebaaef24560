for n in 16384 32768; do
  python tools/lu_rate.py $n 3
  DENSOLVE_PANEL_ROWS=128 DENSOLVE_PANEL_TPR=2 DENSOLVE_PANEL_KERNEL=2 python tools/lu_rate.py $n 3
  DENSOLVE_PANEL_ROWS=128 DENSOLVE_PANEL_TPR=2 python tools/lu_rate.py $n 3
  DENSOLVE_PANEL_ROWS=160 DENSOLVE_PANEL_TPR=2 python tools/lu_rate.py $n 3
done 2>&1 | grep "LU n"
