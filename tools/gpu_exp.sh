# GMRES C2 with the 64-register cluster kernel (co-resident with 2 GEMV CTAs per SM)
for c in default 112 56 224; do
  if [ $c = default ]; then python tools/gemv_small.py 4096; else DENSOLVE_GEMV_CHUNK=$c python tools/gemv_small.py 4096; fi
done 2>&1 | grep -v Warn
# fp32 GEMM: large-tile kernel vs the 64x64 one (bitwise) and rates
DENSOLVE_GEMM32_SMALL=1 python tools/gemm_check.py /tmp/s0.npz f32 && python tools/gemm_check.py /tmp/s1.npz f32 && python tools/gemm_check.py --compare /tmp/s0.npz /tmp/s1.npz
echo "== fp32 64x64"; DENSOLVE_GEMM32_SMALL=1 GEMM_RATE_F32=1 python tools/gemm_rate.py 16384 64 512
echo "== fp32 128x128"; GEMM_RATE_F32=1 python tools/gemm_rate.py 16384 64 512
