"""Short driver for ncu captures: python tools/profile_run.py {cg,gemv,lu,gmres,chol,gemm,trsm} [n]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_07207_b200 import (SolverConfig, cg_solve, cholesky_factor, get_backend,  # noqa: E402
                                   gmres_solve, lu_factor_blocked)
from paper_1511_07207_b200.device import DeviceArray  # noqa: E402
from paper_1511_07207_b200.harness import ProblemSpec, generate_problem  # noqa: E402

what = sys.argv[1]
be = get_backend("b200")
ctx = be.ctx
rng = np.random.default_rng(0)
if what in ("cg", "gemv"):
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    R = rng.uniform(-1, 1, (n, n))
    A = np.asfortranarray((R + R.T) * 0.5 + np.sqrt(n) * np.eye(n))
    del R
    b = A @ rng.uniform(-1, 1, n)
    dA, db, dx0 = be.stage_in(A, b, np.zeros(n))
    if what == "cg":
        cg_solve(dA, db, dx0, SolverConfig(tolerance=1e-300, max_iterations=10), be)
    else:
        from ctypes import c_void_p
        dy = DeviceArray(ctx, (n,), np.float64)
        for _ in range(5):
            ctx.lib.ds_gemv(ctx.handle, 1, n, n, c_void_p(dA.ptr), dA.ld, c_void_p(db.ptr), c_void_p(dy.ptr))
        ctx.synchronize()
elif what == "lu":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    A = np.asfortranarray(rng.uniform(-1, 1, (n, n)))
    dA = be.stage_in(A)
    lu_factor_blocked(dA, 64, be)
    ctx.synchronize()
elif what == "gemm":
    m, n, k = (int(v) for v in sys.argv[2:5])
    A = np.asfortranarray(rng.uniform(-1, 1, (m, k)))
    B = np.asfortranarray(rng.uniform(-1, 1, (k, n)))
    C = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    dA, dB, dC = be.stage_in(A, B, C)
    for _ in range(3):
        be.gemm(-1.0, dA, dB, 1.0, dC, out=dC)
    ctx.synchronize()
elif what == "trsm":
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    L = np.asfortranarray(np.tril(rng.uniform(-1, 1, (64, 64))))
    B = np.asfortranarray(rng.uniform(-1, 1, (64, m)))
    dL, dB = be.stage_in(L, B)
    for _ in range(3):
        be.trsm_lower_unit(dL, dB)
    ctx.synchronize()
elif what == "gmres":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    A, b, _ = generate_problem(ProblemSpec("general_nonsymmetric", n, 0))
    dA, db, dx0 = be.stage_in(A, b, np.zeros(n))
    gmres_solve(dA, db, dx0, SolverConfig(tolerance=1e-300, restart_m=30, max_iterations=30), be)
    ctx.synchronize()
elif what == "chol":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    R = rng.uniform(-1, 1, (n, n))
    A = np.asfortranarray((R + R.T) * 0.5 + np.sqrt(n) * np.eye(n))
    del R
    dA = be.stage_in(A)
    cholesky_factor(dA, 64, be)
    ctx.synchronize()
print("done", what)
