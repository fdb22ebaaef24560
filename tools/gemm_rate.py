"""DMMA GEMM throughput (C -= A B, the LU trailing update): python tools/gemm_rate.py n K..."""
import os
import sys
from ctypes import c_void_p

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import _lib, get_backend  # noqa: E402

be = get_backend("b200")
ctx = be.ctx
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
dt, code = torch.float64, _lib.DS_F64
if os.environ.get("GEMM_RATE_F32") == "1":
    dt, code = torch.float32, _lib.DS_F32
n = int(sys.argv[1])
for K in [int(v) for v in sys.argv[2:]]:
    A = torch.rand((n, K), dtype=dt, device="cuda")
    B = torch.rand((K, n), dtype=dt, device="cuda")
    C = torch.rand((n, n), dtype=dt, device="cuda")

    def gemm():
        _lib.check(ctx.lib.ds_gemm(ctx.handle, code, n, n, K, -1.0, c_void_p(A.data_ptr()), n,
                                   c_void_p(B.data_ptr()), K, 1.0, c_void_p(C.data_ptr()), n,
                                   c_void_p(C.data_ptr()), n))
    gemm()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        gemm()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"GEMM {dt} {n}x{n}x{K}: {ms:.3f} ms  {2 * n * n * K / ms / 1e9:.2f} TFLOP/s", flush=True)
    del A, B, C
