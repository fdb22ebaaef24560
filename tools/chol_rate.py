"""Cholesky timing (device-resident SPD): python tools/chol_rate.py n"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import cholesky_factor, get_backend  # noqa: E402
from paper_1511_07207_b200.device import DeviceArray  # noqa: E402

be = get_backend("b200")
ctx = be.ctx
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
n = int(sys.argv[1])
g = torch.Generator(device="cuda")
g.manual_seed(0)
A = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g).mul_(2).sub_(1)
A.add_(A.t().clone()).mul_(0.5)
A.diagonal().add_(n ** 0.5)
dA = DeviceArray(ctx, (n, n), np.float64)
ctx.lib.ds_memcpy_d2d(ctx.handle, dA.ptr, A.data_ptr(), 8 * n * n)
del A
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    f = cholesky_factor(dA, 64, be)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    del f
    print(f"Cholesky n={n} NB={os.environ.get('DENSOLVE_CHOL_NB', '512')}: {ms:.1f} ms  {n**3 / 3 / ms / 1e9:.2f} TFLOP/s",
          flush=True)
