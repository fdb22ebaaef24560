"""Time device-resident blocked LU (b=64) at several n, look-ahead on/off, plus the
K=256 trailing GEMM alone.  python tools/lu_probe.py 8192 16384 32768"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import get_backend, lu_factor_blocked  # noqa: E402
from paper_1511_07207_b200.device import DeviceArray  # noqa: E402

be = get_backend("b200")
ctx = be.ctx
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)


def timed(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in [int(v) for v in sys.argv[1:]]:
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    At = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g).mul_(2.0).sub_(1.0)
    dA = DeviceArray(ctx, (n, n), np.float64)
    ctx.lib.ds_memcpy_d2d(ctx.handle, dA.ptr, At.data_ptr(), 8 * n * n)
    del At
    torch.cuda.synchronize()
    for la in ("1", "0"):
        os.environ["DENSOLVE_LU_LOOKAHEAD"] = la
        ms = timed(lambda: lu_factor_blocked(dA, 64, be))
        print(f"LU n={n} lookahead={la}: {ms:.2f} ms  {2 * n**3 / 3 / ms / 1e9:.2f} TFLOP/s", flush=True)
    os.environ["DENSOLVE_LU_LOOKAHEAD"] = "1"
    del dA
    torch.cuda.empty_cache()
    for K in (256, 512):
        A = torch.rand((n, K), dtype=torch.float64, device="cuda")
        B = torch.rand((K, n), dtype=torch.float64, device="cuda")
        C = torch.rand((n, n), dtype=torch.float64, device="cuda")
        from ctypes import c_void_p
        from paper_1511_07207_b200 import _lib

        def gemm():
            _lib.check(ctx.lib.ds_gemm(ctx.handle, _lib.DS_F64, n, n, K, -1.0,
                                       c_void_p(A.data_ptr()), n, c_void_p(B.data_ptr()), K, 1.0,
                                       c_void_p(C.data_ptr()), n, c_void_p(C.data_ptr()), n))
        ms = timed(gemm, 3)
        print(f"GEMM {n}x{n}x{K}: {ms:.3f} ms  {2 * n * n * K / ms / 1e9:.2f} TFLOP/s", flush=True)
        del A, B, C
        torch.cuda.empty_cache()
