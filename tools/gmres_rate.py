"""GMRES one-cycle timing (device-resident): python tools/gmres_rate.py n m [fp32]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import SolverConfig, get_backend, gmres_solve  # noqa: E402
from paper_1511_07207_b200.harness import ProblemSpec, generate_problem  # noqa: E402

be = get_backend("b200")
ctx = be.ctx
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
n, m = int(sys.argv[1]), int(sys.argv[2])
prec = "f32" if len(sys.argv) > 3 else "f64"
A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=n, seed=0, precision=prec))
dA, db, dx0 = be.stage_in(A, b, np.zeros_like(b))
cfg = SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m)
for mode in ("cluster", "fused", "split", "cluster"):
    os.environ["DENSOLVE_GMRES_ORTH"] = "cluster" if mode == "cluster" else "grid"
    os.environ["DENSOLVE_GMRES_FUSED"] = "1" if mode == "fused" else "0"
    fz = mode
    gmres_solve(dA, db, dx0, cfg, be)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        x, rep = gmres_solve(dA, db, dx0, cfg, be)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"GMRES({m}) n={n} {prec} fused={fz}: {ms:.3f} ms/cycle  {rep.iterations / ms * 1e3:.0f} it/s  "
          f"launches={rep.kernel_launches}", flush=True)

# the bare GEMVs of one cycle (33 = 30 Arnoldi + residual + true residual + x update) back to back
from ctypes import c_void_p  # noqa: E402
from paper_1511_07207_b200 import _lib  # noqa: E402
from paper_1511_07207_b200.device import DeviceArray  # noqa: E402
dy = DeviceArray(ctx, (n,), dA.dtype)


def gemvs():
    for _ in range(33):
        _lib.check(ctx.lib.ds_gemv(ctx.handle, dA.dcode, n, n, c_void_p(dA.ptr), dA.ld, c_void_p(db.ptr),
                                   c_void_p(dy.ptr)))


gemvs()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(10):
    gemvs()
e1.record(stream)
torch.cuda.synchronize()
print(f"33 bare GEMVs n={n}: {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
