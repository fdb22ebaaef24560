import sys, os
sys.path.insert(0, '/root/repo')
from ctypes import c_void_p
import numpy as np, torch
from paper_1511_07207_b200 import _lib, get_backend
be = get_backend("b200"); ctx = be.ctx
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
for (n, dt, code, es) in [(65536, torch.float32, _lib.DS_F32, 4), (32768, torch.float64, _lib.DS_F64, 8), (46341, torch.float64, _lib.DS_F64, 8)]:
    A = torch.empty((n, n), dtype=dt, device="cuda"); A.fill_(0.5)
    x = torch.ones(n, dtype=dt, device="cuda"); y = torch.empty_like(x)
    f = lambda: _lib.check(ctx.lib.ds_gemv(ctx.handle, code, n, n, c_void_p(A.data_ptr()), n, c_void_p(x.data_ptr()), c_void_p(y.data_ptr())))
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10): f()
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"n={n} {dt}: {ms:.3f} ms/GEMV = {n*n*es/ms/1e6:.0f} GB/s", flush=True)
    del A
    torch.cuda.empty_cache()
