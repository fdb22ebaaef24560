"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the reference is importable there, not on the GPU
box):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
Writes tests/golden/golden.npz (committed).  Each case records the reference's
outputs (iterations, residual histories, restart cycles, pivots, packed
factors or their checksums, solutions) plus SHA-256 digests of generated
inputs, so the oracle restatement, the package's generators and the CUDA path
can all be pinned to the reference without importing it at test time.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import densolve as ds  # noqa: E402
from densolve.harness import ProblemSpec, generate_problem, generate_well_separated  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asfortranarray(a)).tobytes(order="F")).hexdigest()


def main():
    g: dict[str, np.ndarray] = {}

    def put(key, val):
        g[key] = np.asarray(val)

    # ---- generator digests (harness.py:77-123) ----
    gen_cases = [("spd", 16, 7, "f64"), ("spd", 64, 7, "f64"), ("spd", 1024, 0, "f64"),
                 ("general_nonsymmetric", 48, 2, "f64"), ("general_nonsymmetric", 512, 0, "f64"),
                 ("general_nonsymmetric", 4096, 0, "f64"), ("general_nonsymmetric", 256, 1, "f32"),
                 ("diag_dominant", 16, 2, "f64"), ("identity", 3, 0, "f64")]
    for i, (kind, n, seed, prec) in enumerate(gen_cases):
        A, b, xt = generate_problem(ProblemSpec(kind=kind, n=n, seed=seed, precision=prec))
        put(f"gen{i}_spec", np.array([kind, str(n), str(seed), prec]))
        put(f"gen{i}_shaA", np.array(sha(A)))
        put(f"gen{i}_shab", np.array(sha(b)))
    put("gen_count", len(gen_cases))
    for i, (n, seed) in enumerate([(64, 3), (256, 0), (512, 5)]):
        A = generate_well_separated(n, seed=seed)
        put(f"ws{i}_spec", np.array([n, seed]))
        put(f"ws{i}_sha", np.array(sha(A)))

    # ---- CG (krylov.py:36-72) ----
    cg_cases = [("c1s0", "spd", 1024, 0, 1e-8, None), ("c1s1", "spd", 1024, 1, 1e-8, None),
                ("c1s2", "spd", 1024, 2, 1e-8, None), ("n64s7", "spd", 64, 7, 1e-10, None),
                ("fixed", "spd", 256, 3, 1e-300, 25), ("f32", "spd", 256, 4, 1e-4, None)]
    for name, kind, n, seed, tol, mi in cg_cases:
        prec = "f32" if name == "f32" else "f64"
        A, b, _ = generate_problem(ProblemSpec(kind=kind, n=n, seed=seed, precision=prec))
        be = ds.ReferenceBackend()
        x, rep = ds.cg_solve(A, b, np.zeros_like(b), ds.SolverConfig(tolerance=tol, max_iterations=mi), be)
        put(f"cg_{name}_spec", np.array([kind, str(n), str(seed), prec, repr(tol), str(mi)]))
        put(f"cg_{name}_iters", rep.iterations)
        put(f"cg_{name}_hist", np.array(rep.residual_history))
        put(f"cg_{name}_x", x)
        put(f"cg_{name}_conv", rep.converged)
        put(f"cg_{name}_counts", np.array([be.counters.gemv_calls, be.counters.dot_calls,
                                           be.counters.axpy_calls, be.counters.nrm2_calls]))

    # CG on k distinct eigenvalues (test_acceptance.py:108-121 recipe), n=64
    for k in (1, 3, 5):
        for seed in range(3):
            rng = np.random.default_rng([seed, k])
            n = 64
            Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
            lam = np.repeat(np.linspace(1.0, 2.0, k), n // k + 1)[:n]
            A = (Q * lam) @ Q.T
            A = np.asfortranarray(np.tril(A) + np.tril(A, -1).T)
            b = rng.standard_normal(n)
            x, rep = ds.cg_solve(A, b, np.zeros(n), ds.SolverConfig(tolerance=1e-10), ds.ReferenceBackend())
            put(f"cgk{k}_{seed}_A", A)
            put(f"cgk{k}_{seed}_b", b)
            put(f"cgk{k}_{seed}_iters", rep.iterations)
            put(f"cgk{k}_{seed}_x", x)

    # ---- GMRES (krylov.py:75-182) ----
    gm_cases = [("n48s2_mgs", 48, 2, 1e-8, 35, "modified", None, "f64"),
                ("n48s2_cgs", 48, 2, 1e-8, 35, "classical", None, "f64"),
                ("n128s8_r20", 128, 8, 1e-10, 20, "modified", None, "f64"),
                ("n64s4_r5", 64, 4, 1e-12, 5, "modified", None, "f64"),
                ("n64s4_r5_cgs", 64, 4, 1e-12, 5, "classical", None, "f64"),
                ("c2_tol4", 4096, 0, 1e-4, 30, "modified", None, "f64"),
                ("c2_tol8", 4096, 0, 1e-8, 30, "modified", None, "f64"),
                ("c2_fixed", 4096, 0, 1e-300, 30, "modified", 30, "f64"),
                ("n512s0_r35", 512, 0, 1e-4, 35, "modified", None, "f64"),
                ("f32_n256", 256, 1, 1e-4, 35, "modified", None, "f32"),
                ("cap7", 96, 5, 1e-300, 3, "classical", 7, "f64")]
    for name, n, seed, tol, m, orth, mi, prec in gm_cases:
        A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=n, seed=seed, precision=prec))
        be = ds.BlockedBackend()
        cfg = ds.SolverConfig(tolerance=tol, restart_m=m, orthogonalization=orth, max_iterations=mi)
        x, rep = ds.gmres_solve(A, b, np.zeros_like(b), cfg, be)
        put(f"gm_{name}_spec", np.array([str(n), str(seed), repr(tol), str(m), orth, str(mi), prec]))
        put(f"gm_{name}_iters", rep.iterations)
        put(f"gm_{name}_hist", np.array(rep.residual_history))
        put(f"gm_{name}_cycles", np.array(rep.restart_cycles))
        put(f"gm_{name}_conv", rep.converged)
        put(f"gm_{name}_x", x)
        put(f"gm_{name}_counts", np.array([be.counters.gemv_calls, be.counters.dot_calls,
                                           be.counters.axpy_calls, be.counters.nrm2_calls,
                                           be.counters.scal_calls]))
    # rotation KAT (test_krylov.py:99-109)
    A = np.asfortranarray([[0.0, 1.0], [-1.0, 0.0]])
    x, rep = ds.gmres_solve(A, np.array([1.0, 0.0]), np.zeros(2), ds.SolverConfig(tolerance=1e-12),
                            ds.ReferenceBackend())
    put("gm_rot_iters", rep.iterations)
    put("gm_rot_x", x)
    put("gm_rot_breakdown", str(rep.breakdown))

    # ---- LU (direct.py:25-84) ----
    A = generate_well_separated(64, seed=3)
    ref = ds.lu_factor_unblocked(A, ds.ReferenceBackend())
    put("lu_ws64_unb_packed", ref.packed)
    put("lu_ws64_unb_piv", ref.pivots)
    for bsz in (1, 8, 32, 64):
        f = ds.lu_factor_blocked(A, bsz, ds.ReferenceBackend())
        put(f"lu_ws64_b{bsz}_packed", f.packed)
        put(f"lu_ws64_b{bsz}_piv", f.pivots)
    rng = np.random.default_rng(1234)
    U = np.asfortranarray(rng.uniform(-1.0, 1.0, size=(128, 128)))
    put("lu_u128_A", U)
    for bsz in (8, 32):
        f = ds.lu_factor_blocked(U, bsz, ds.ReferenceBackend())
        put(f"lu_u128_b{bsz}_packed", f.packed)
        put(f"lu_u128_b{bsz}_piv", f.pivots)
    f = ds.lu_factor_unblocked(U, ds.ReferenceBackend())
    put("lu_u128_unb_packed", f.packed)
    put("lu_u128_unb_piv", f.pivots)
    # harness LU family (identity pivots) and a pivoting uniform family at larger n
    for n in (512, 1024):
        A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=n, seed=0))
        f = ds.lu_factor_blocked(A, 64, ds.BlockedBackend())
        x = ds.lu_solve(f, b)
        put(f"lu_gn{n}_piv", f.pivots)
        put(f"lu_gn{n}_x", x)
        put(f"lu_gn{n}_packsum", np.array([np.sum(f.packed), np.sum(np.abs(f.packed))]))
    for n in (256, 512):
        A = np.asfortranarray(np.random.default_rng([0, n, 1]).uniform(-1.0, 1.0, (n, n)))
        f = ds.lu_factor_blocked(A, 64, ds.BlockedBackend())
        b = np.random.default_rng([0, n, 2]).uniform(-1.0, 1.0, n)
        put(f"lu_uni{n}_piv", f.pivots)
        put(f"lu_uni{n}_x", ds.lu_solve(f, b))
        put(f"lu_uni{n}_packsum", np.array([np.sum(f.packed), np.sum(np.abs(f.packed))]))
    # fp32 family (test_direct.py:120-131 shape)
    A32 = np.asfortranarray(np.random.default_rng(64).uniform(-1.0, 1.0, (64, 64)).astype(np.float32))
    f = ds.lu_factor_blocked(A32, 64, ds.ReferenceBackend())
    put("lu_f32_64_A", A32)
    put("lu_f32_64_packed", f.packed)
    put("lu_f32_64_piv", f.pivots)
    # KATs (test_direct.py:42-56)
    f = ds.lu_factor_unblocked(np.asfortranarray([[4.0, 3.0], [6.0, 3.0]]), ds.ReferenceBackend())
    put("lu_kat2_packed", f.packed)
    put("lu_kat2_piv", f.pivots)

    # ---- nrm2 / dot semantics (backends.py:109-132) ----
    be = ds.ReferenceBackend()
    put("nrm2_big", be.nrm2(np.array([1e300, 1e300])))
    put("nrm2_34", be.nrm2(np.array([3.0, 4.0])))
    put("iamax_tie", be.iamax(np.array([2.0, -2.0])))

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
