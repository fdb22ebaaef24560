"""Golden vectors for the SURVEY.md §8f rows (BiCGSTAB, Cholesky), produced by
running the REFERENCE implementation itself in the build container:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_next.py
Writes tests/golden/golden_next.npz (committed; the GPU box never imports the
reference).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import densolve as ds  # noqa: E402
from densolve.harness import ProblemSpec, generate_problem  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_next.npz")

# name, kind, n, seed, tol, max_it, precision
BICG_CASES = [
    ("n64s9", "general_nonsymmetric", 64, 9, 1e-4, None, "f64"),       # test_krylov.py:177-183
    ("fixed7", "general_nonsymmetric", 32, 1, 1e-300, 7, "f64"),       # test_krylov.py:185-196
    ("n17fix6", "general_nonsymmetric", 17, 0, 1e-300, 6, "f64"),      # test_acceptance.py:88-102
    ("n200fix6", "general_nonsymmetric", 200, 0, 1e-300, 6, "f64"),
    ("n512s0", "general_nonsymmetric", 512, 0, 1e-8, None, "f64"),
    ("n512s3", "general_nonsymmetric", 512, 3, 1e-10, None, "f64"),
    ("c2_tol8", "general_nonsymmetric", 4096, 0, 1e-8, None, "f64"),
    ("f32_n256", "general_nonsymmetric", 256, 1, 1e-4, None, "f32"),
    ("dd_n128", "diag_dominant", 128, 2, 1e-10, None, "f64"),
]

# name, n, seed, b, precision
CHOL_CASES = [
    ("n16b4", 16, 5, 4, "f64"),     # test_direct.py:158-162
    ("n64b16", 64, 7, 16, "f64"),
    ("n200b64", 200, 3, 64, "f64"),  # ragged last panel
    ("n256b64", 256, 11, 64, "f64"),  # test_direct.py:256-260
    ("n256b1", 256, 1, 1, "f64"),
    ("n96b500", 96, 2, 500, "f64"),  # b > n clamps
    ("f32n64", 64, 4, 64, "f32"),
    ("n1024b64", 1024, 0, 64, "f64"),
]


def main():
    g: dict[str, np.ndarray] = {}

    def put(key, val):
        g[key] = np.asarray(val)

    # ---- BiCGSTAB (krylov.py:185-253) ----
    for name, kind, n, seed, tol, mi, prec in BICG_CASES:
        A, b, _ = generate_problem(ProblemSpec(kind=kind, n=n, seed=seed, precision=prec))
        be = ds.ReferenceBackend()
        x, rep = ds.bicgstab_solve(A, b, np.zeros_like(b), ds.SolverConfig(tolerance=tol, max_iterations=mi), be)
        put(f"bi_{name}_spec", np.array([kind, str(n), str(seed), repr(tol), str(mi), prec]))
        put(f"bi_{name}_iters", rep.iterations)
        put(f"bi_{name}_hist", np.array(rep.residual_history))
        put(f"bi_{name}_x", x)
        put(f"bi_{name}_conv", rep.converged)
        put(f"bi_{name}_breakdown", str(rep.breakdown))
        c = be.counters
        put(f"bi_{name}_counts", np.array([c.gemv_calls, c.dot_calls, c.axpy_calls, c.nrm2_calls]))
    put("bi_names", np.array([c[0] for c in BICG_CASES]))
    # KATs: identity (1 iteration, x = b), exact x0 (0 iterations), rho breakdown (rotation)
    rng = np.random.default_rng(5)
    bI = rng.standard_normal(8)
    x, rep = ds.bicgstab_solve(np.asfortranarray(np.eye(8)), bI, np.zeros(8), ds.SolverConfig(),
                               ds.ReferenceBackend())
    put("bi_eye_b", bI)
    put("bi_eye_x", x)
    put("bi_eye_iters", rep.iterations)
    A = np.asfortranarray([[0.0, 1.0], [-1.0, 0.0]])
    x, rep = ds.bicgstab_solve(A, np.array([1.0, 0.0]), np.zeros(2), ds.SolverConfig(), ds.ReferenceBackend())
    put("bi_rot_iters", rep.iterations)
    put("bi_rot_breakdown", str(rep.breakdown))
    put("bi_rot_hist", np.array(rep.residual_history))
    put("bi_rot_x", x)

    # ---- Cholesky (direct.py:87-120, 166-171) ----
    for name, n, seed, bsz, prec in CHOL_CASES:
        A, b, _ = generate_problem(ProblemSpec(kind="spd", n=n, seed=seed, precision=prec))
        f = ds.cholesky_factor(A, bsz, ds.BlockedBackend())
        x = ds.cholesky_solve(f, b)
        put(f"ch_{name}_spec", np.array([str(n), str(seed), str(bsz), prec]))
        if n <= 256:
            put(f"ch_{name}_L", f.l)
        put(f"ch_{name}_Lsum", np.array([np.sum(f.l, dtype=np.float64), np.sum(np.abs(f.l), dtype=np.float64),
                                          np.sum(np.diag(f.l), dtype=np.float64)]))
        put(f"ch_{name}_x", x)
    put("ch_names", np.array([c[0] for c in CHOL_CASES]))
    # NotSpdError index KAT (test_direct.py:164-168)
    try:
        ds.cholesky_factor(np.asfortranarray(np.diag([1.0, -1.0])), 2, ds.ReferenceBackend())
        put("ch_notspd_index", -1)
    except ds.NotSpdError as e:
        put("ch_notspd_index", e.index)
    # a pivot failing deep inside a later panel: spd with one negative eigen-direction
    rng = np.random.default_rng(77)
    M = rng.uniform(-1, 1, (96, 96))
    S = np.asfortranarray(M @ M.T + 96 * np.eye(96))
    S[70, 70] = -5.0
    try:
        ds.cholesky_factor(S, 32, ds.ReferenceBackend())
        put("ch_notspd70_index", -1)
    except ds.NotSpdError as e:
        put("ch_notspd70_index", e.index)
    put("ch_notspd70_A", S)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
