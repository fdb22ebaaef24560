for i in 1 2 3; do TRIALS=150 python tools/gemm_concurrent.py 2>&1 | tail -1; done
DENSOLVE_GEMM_TMA=0 python tools/lu_tma_check.py run /tmp/l0.npz 8192 > /dev/null
for i in 1 2; do python tools/lu_tma_check.py run /tmp/l1.npz 8192 > /dev/null && python tools/lu_tma_check.py cmp /tmp/l0.npz /tmp/l1.npz 2>/dev/null | head -2; done
python tools/gemm_rate.py 16384 64 256 512
for c in default 112 56; do
  if [ $c = default ]; then python tools/gemv_small.py 4096; else DENSOLVE_GEMV_CHUNK=$c python tools/gemv_small.py 4096; fi
done 2>&1 | grep -v Warn
DENSOLVE_GEMM32_SMALL=1 python tools/gemm_check.py /tmp/s0.npz f32 && python tools/gemm_check.py /tmp/s1.npz f32 && python tools/gemm_check.py --compare /tmp/s0.npz /tmp/s1.npz
echo "== fp32 64x64"; DENSOLVE_GEMM32_SMALL=1 GEMM_RATE_F32=1 python tools/gemm_rate.py 16384 64 512
echo "== fp32 128x128"; GEMM_RATE_F32=1 python tools/gemm_rate.py 16384 64 512
