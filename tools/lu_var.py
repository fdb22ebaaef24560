"""Repeat device-resident LU timings to expose run-to-run variance: python tools/lu_var.py n reps"""
import os
import sys

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
n, reps = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda")
g.manual_seed(1)
At = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g).mul_(2.0).sub_(1.0)
dA = DeviceArray(ctx, (n, n), np.float64)
for la in ("1", "0", "1"):
    os.environ["DENSOLVE_LU_LOOKAHEAD"] = la
    ts = []
    for _ in range(reps):
        ctx.lib.ds_memcpy_d2d(ctx.handle, dA.ptr, At.data_ptr(), 8 * n * n)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lu_factor_blocked(dA, 64, be)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"n={n} lookahead={la}: " + " ".join(f"{t:.1f}" for t in ts) + " ms", flush=True)
