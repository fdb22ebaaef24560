for n in 2048 4096 8192; do
  DENSOLVE_GEMM_TMA=0 python tools/lu_tma_check.py run /tmp/l0_$n.npz $n > /dev/null && python tools/lu_tma_check.py run /tmp/l1_$n.npz $n > /dev/null && echo "n=$n" && python tools/lu_tma_check.py cmp /tmp/l0_$n.npz /tmp/l1_$n.npz
done
