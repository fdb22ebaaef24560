"""Per-iteration CG cost vs the bare GEMV: python tools/cg_overhead.py [n]
(difference of 200- and 100-iteration solves, so the per-solve setup cancels)."""
import os
import sys
from ctypes import c_void_p

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import SolverConfig, _lib, cg_solve, get_backend  # noqa: E402
from paper_1511_07207_b200.device import DeviceArray  # noqa: E402
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
be = get_backend("b200")
ctx = be.ctx
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
At, bt = bench.spd_fast_device(n, 0, torch, "cuda", be)
dA = DeviceArray(ctx, (n, n), np.float64)
ctx.lib.ds_memcpy_d2d(ctx.handle, dA.ptr, At.data_ptr(), 8 * n * n)
db = DeviceArray(ctx, (n,), np.float64)
ctx.lib.ds_memcpy_d2d(ctx.handle, db.ptr, bt.data_ptr(), 8 * n)
dx0 = DeviceArray(ctx, (n,), np.float64)
ctx.lib.ds_memset(ctx.handle, dx0.ptr, 0, 8 * n)
del At


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


t100 = timed(lambda: cg_solve(dA, db, dx0, SolverConfig(tolerance=1e-300, max_iterations=100), be))
t200 = timed(lambda: cg_solve(dA, db, dx0, SolverConfig(tolerance=1e-300, max_iterations=200), be))
dy = DeviceArray(ctx, (n,), np.float64)


def gemvs():
    for _ in range(100):
        _lib.check(ctx.lib.ds_gemv(ctx.handle, _lib.DS_F64, n, n, c_void_p(dA.ptr), dA.ld, c_void_p(db.ptr),
                                   c_void_p(dy.ptr)))


tg = timed(gemvs)
print(f"n={n}: CG 100 it {t100:.2f} ms, 200 it {t200:.2f} ms -> {(t200 - t100) * 10:.1f} us/iteration; "
      f"setup {t100 - (t200 - t100):.2f} ms; bare GEMV (partial + reduce) {tg * 10:.1f} us", flush=True)
