"""GMRES(30) C2 cycle and the bare GEMV at n=4096 under the current DENSOLVE_GEMV_CHUNK."""
import os
import sys
from ctypes import c_void_p

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import SolverConfig, _lib, get_backend, gmres_solve  # noqa: E402
from paper_1511_07207_b200.device import DeviceArray  # noqa: E402
from paper_1511_07207_b200.harness import ProblemSpec, generate_problem  # noqa: E402

be = get_backend("b200")
ctx = be.ctx
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
n, m = int(sys.argv[1]), 30
A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=n, seed=0, precision="f64"))
dA, db, dx0 = be.stage_in(A, b, np.zeros_like(b))
cfg = SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = timed(lambda: gmres_solve(dA, db, dx0, cfg, be))
dy = DeviceArray(ctx, (n,), dA.dtype)
gm = timed(lambda: _lib.check(ctx.lib.ds_gemv(ctx.handle, dA.dcode, n, n, c_void_p(dA.ptr), dA.ld, c_void_p(db.ptr),
                                              c_void_p(dy.ptr))), 50)
print(f"chunk={os.environ.get('DENSOLVE_GEMV_CHUNK', 'default')}: GMRES(30) n={n}: {ms:.3f} ms/cycle "
      f"{30 / ms * 1e3:.0f} it/s; bare GEMV {gm * 1e3:.1f} us = {8 * n * n / gm / 1e6:.0f} GB/s", flush=True)
