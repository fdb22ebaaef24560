"""Device-resident LU timing (best of reps, look-ahead on): python tools/lu_rate.py n [reps]"""
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
n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device="cuda")
g.manual_seed(1)
At = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g).mul_(2.0).sub_(1.0)
dA = DeviceArray(ctx, (n, n), np.float64)
ts = []
for _ in range(reps + 1):
    ctx.lib.ds_memcpy_d2d(ctx.handle, dA.ptr, At.data_ptr(), 8 * n * n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    f = lu_factor_blocked(dA, 64, be)
    e1.record(stream)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
best = min(ts[1:])
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith(("DENSOLVE_PANEL", "DENSOLVE_LU")))
import hashlib  # noqa: E402
digest = hashlib.sha256(np.ascontiguousarray(dA.to_host()).tobytes()).hexdigest()[:16]
print(f"LU n={n}: best {best:.2f} ms = {2 / 3 * n ** 3 / best / 1e9:.1f} TFLOP/s  runs {[round(t, 1) for t in ts[1:]]}  {tag}"
      f"  factors sha256 {digest}", flush=True)
