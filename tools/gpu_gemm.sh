mkdir -p gpurun_out
DENSOLVE_GEMM_TMA=0 python tools/gemm_check.py /tmp/g0.npz && python tools/gemm_check.py /tmp/g1.npz && python tools/gemm_check.py --compare /tmp/g0.npz /tmp/g1.npz
echo "== cp.async"; DENSOLVE_GEMM_TMA=0 python tools/gemm_rate.py 16384 64 256 512
echo "== TMA"; python tools/gemm_rate.py 16384 64 256 512
cuobjdump -sass paper_1511_07207_b200/libdensolve_b200.so | grep -c UTMALDG
