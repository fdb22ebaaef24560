"""BiCGSTAB parity on the B200 against the reference's golden vectors
(test_krylov.py:163-205 / test_acceptance.py:88-102 patterns, re-targeted).

Tolerances: iterations |dit| <= 1 (identical in practice); residual history
rtol 1e-6 on the common prefix (fp64; fixed-iteration runs excepted, they walk
into round-off); solution ||dx||_inf <= 1e-8 ||x_ref||_inf (fp64), 1e-3 (fp32);
breakdown tags identical; counter tallies identical when iterations match.
"""
import numpy as np
import pytest

from oracle import densolve_oracle as O
from paper_1511_07207_b200 import DegenerateRhsError, SolverConfig, bicgstab_solve, solve_system
from paper_1511_07207_b200.harness import ProblemSpec, generate_problem

pytestmark = pytest.mark.gpu

BI = ["n64s9", "fixed7", "n17fix6", "n200fix6", "n512s0", "n512s3", "c2_tol8", "f32_n256", "dd_n128"]


@pytest.mark.parametrize("name", BI)
def test_bicgstab_matches_reference_golden(backend, golden_next, name):
    kind, n, seed, tol, mi, prec = [str(s) for s in golden_next[f"bi_{name}_spec"]]
    A, b, _ = generate_problem(ProblemSpec(kind=kind, n=int(n), seed=int(seed), precision=prec))
    cfg = SolverConfig(tolerance=float(tol), max_iterations=None if mi == "None" else int(mi))
    x, rep = bicgstab_solve(A, b, np.zeros_like(b), cfg, backend)
    it_ref = int(golden_next[f"bi_{name}_iters"])
    assert abs(rep.iterations - it_ref) <= 1
    assert rep.converged == bool(golden_next[f"bi_{name}_conv"])
    assert str(rep.breakdown) == str(golden_next[f"bi_{name}_breakdown"])
    assert len(rep.residual_history) == rep.iterations + 1
    h_ref = golden_next[f"bi_{name}_hist"]
    k = min(len(h_ref), len(rep.residual_history))
    if "fix" not in name:
        np.testing.assert_allclose(rep.residual_history[:k], h_ref[:k], rtol=1e-6 if prec == "f64" else 1e-2)
    xr = golden_next[f"bi_{name}_x"]
    if "fix" not in name:
        xt = 1e-8 if prec == "f64" else 1e-3
        assert np.linalg.norm(x - xr, np.inf) <= xt * np.linalg.norm(xr, np.inf)
    assert x.dtype == A.dtype
    gv, dt, ax, nr = (int(v) for v in golden_next[f"bi_{name}_counts"])
    c = backend.counters
    if rep.iterations == it_ref:
        assert (c.gemv_calls, c.dot_calls, c.axpy_calls, c.nrm2_calls) == (gv, dt, ax, nr)


def test_bicgstab_cost_law(backend):
    # test_acceptance.py:88-102: exactly +6 axpy, +4 dot, +2 gemv per full iteration
    for n in (17, 64, 200):
        A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=n, seed=0))
        backend.counters.reset()
        _, rep = bicgstab_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-300, max_iterations=6), backend)
        assert rep.iterations == 6
        c = backend.counters
        assert (c.axpy_calls - 1, c.dot_calls - 1, c.gemv_calls - 1) == (36, 24, 12)


def test_bicgstab_identity_one_iteration(backend, golden_next):
    b = golden_next["bi_eye_b"]
    x, rep = bicgstab_solve(np.asfortranarray(np.eye(8)), b, np.zeros(8), SolverConfig(), backend)
    assert rep.converged and rep.iterations == 1  # early exit on ||s||
    np.testing.assert_array_equal(x, golden_next["bi_eye_x"])


def test_bicgstab_exact_x0_zero_iterations(backend):
    A, b, xt = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=32, seed=2))
    x, rep = bicgstab_solve(A, A @ xt, xt, SolverConfig(), backend)
    assert rep.converged and rep.iterations == 0


def test_bicgstab_rho_breakdown(backend, golden_next):
    A = np.asfortranarray([[0.0, 1.0], [-1.0, 0.0]])
    x, rep = bicgstab_solve(A, np.array([1.0, 0.0]), np.zeros(2), SolverConfig(), backend)
    assert not rep.converged
    assert rep.breakdown == "rho-breakdown" == str(golden_next["bi_rot_breakdown"])
    assert rep.iterations == int(golden_next["bi_rot_iters"])
    assert len(rep.residual_history) == rep.iterations + 1


def test_bicgstab_degenerate_rhs(backend):
    with pytest.raises(DegenerateRhsError):
        bicgstab_solve(np.asfortranarray(np.eye(4)), np.zeros(4), np.zeros(4), SolverConfig(), backend)


def test_bicgstab_matches_oracle_seeds(backend):
    for seed in range(5):
        A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=384, seed=seed))
        x, rep = bicgstab_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-10), backend)
        xo, ro = O.bicgstab(A, b, np.zeros_like(b), 1e-10)
        assert abs(rep.iterations - ro["iterations"]) <= 1 and rep.converged
        assert np.linalg.norm(x - xo, np.inf) <= 1e-8 * np.linalg.norm(xo, np.inf)


def test_solve_system_bicgstab(backend):
    A, b, xt = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=128, seed=4))
    x, rep = solve_system("bicgstab", A, b, None, SolverConfig(tolerance=1e-10), backend)
    assert rep.converged
    assert np.linalg.norm(x - xt) <= 1e-8 * np.linalg.norm(xt)


def test_bicgstab_device_resident(backend):
    A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=256, seed=1))
    dA, db, dx0 = backend.stage_in(A, b, np.zeros_like(b))
    dx, rep = bicgstab_solve(dA, db, dx0, SolverConfig(tolerance=1e-10), backend)
    x = backend.stage_out(dx)
    xo, _ = O.bicgstab(A, b, np.zeros_like(b), 1e-10)
    assert np.linalg.norm(x - xo, np.inf) <= 1e-8 * np.linalg.norm(xo, np.inf)
