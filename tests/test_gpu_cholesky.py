"""Cholesky parity on the B200 against the reference's golden vectors
(test_direct.py:133-173, 245-260 patterns, re-targeted).

Tolerances: a single panel (b >= n, n <= 64) is bitwise the reference's (exact
panel kernels, no GEMM); otherwise
||L - L_ref||_max <= 100 n u max|L_ref| (the trailing update is grouped into
K = 256 DMMA SYRKs) and the reference's own residual bound
||L L^T - A||_F <= 10 n u ||A||_F holds; solutions ||dx||_inf <= 1e-9 ||x||_inf
(fp64), 1e-3 (fp32).
"""
import numpy as np
import pytest

from paper_1511_07207_b200 import (NotSpdError, SolverConfig, cholesky_factor, cholesky_solve,
                                   relative_residual, solve_system, unit_roundoff)
from paper_1511_07207_b200.harness import ProblemSpec, generate_problem

pytestmark = pytest.mark.gpu

CH = ["n16b4", "n64b16", "n200b64", "n256b64", "n256b1", "n96b500", "f32n64", "n1024b64"]


@pytest.mark.parametrize("name", CH)
def test_cholesky_matches_reference_golden(backend, golden_next, name):
    n, seed, bsz, prec = [str(s) for s in golden_next[f"ch_{name}_spec"]]
    n, bsz = int(n), int(bsz)
    A, b, _ = generate_problem(ProblemSpec(kind="spd", n=n, seed=int(seed), precision=prec))
    f = cholesky_factor(A, bsz, backend)
    L = f.l
    assert L.dtype == A.dtype and np.array_equal(L, np.tril(L))
    u = unit_roundoff(A.dtype)
    if f"ch_{name}_L" in golden_next.files:
        Lr = golden_next[f"ch_{name}_L"]
        assert np.max(np.abs(L - Lr)) <= 100 * n * u * np.max(np.abs(Lr))
    s = golden_next[f"ch_{name}_Lsum"]
    np.testing.assert_allclose(np.sum(np.diag(L), dtype=np.float64), s[2], rtol=1e-12 if prec == "f64" else 1e-5)
    L64, A64 = L.astype(np.float64), A.astype(np.float64)
    assert np.linalg.norm(L64 @ L64.T - A64) <= 10 * n * u * np.linalg.norm(A64)
    x = cholesky_solve(f, b)
    xr = golden_next[f"ch_{name}_x"]
    tol = 1e-9 if prec == "f64" else 1e-3
    assert np.linalg.norm(x - xr, np.inf) <= tol * np.linalg.norm(xr, np.inf)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [4, 16, 64, 256])
def test_cholesky_residual_bound(backend, dtype, n):
    u = unit_roundoff(dtype)
    for seed in range(5):
        A, _, _ = generate_problem(ProblemSpec(kind="spd", n=n, seed=seed,
                                               precision="f32" if dtype is np.float32 else "f64"))
        L = cholesky_factor(A, min(64, n), backend).l.astype(np.float64)
        assert np.linalg.norm(L @ L.T - A.astype(np.float64)) <= 10 * n * u * np.linalg.norm(A.astype(np.float64))


@pytest.mark.parametrize("n", [1, 7, 33, 64])
def test_cholesky_single_panel_bitwise(backend, n):
    # one panel: diagonal-block + row kernels reproduce the reference column loop bit for bit
    from oracle import densolve_oracle as O
    A, _, _ = generate_problem(ProblemSpec(kind="spd", n=n, seed=3))
    np.testing.assert_array_equal(cholesky_factor(A, n, backend).l, O.cholesky_factor(A, n))
    A = np.asfortranarray(np.random.default_rng(n).uniform(-1, 1, (n + 100, n + 100)))
    A = np.asfortranarray(A @ A.T + (n + 100) * np.eye(n + 100))
    # rows below a 64-wide first panel (then one GEMM-updated trailing block): the first
    # 64 columns are still bitwise
    Lg = cholesky_factor(A, 64, backend).l
    np.testing.assert_array_equal(Lg[:, :64], O.cholesky_factor(A, 64)[:, :64])


def test_cholesky_kats(backend):
    f = cholesky_factor(np.asfortranarray(np.eye(3)), 2, backend)
    assert np.array_equal(f.l, np.eye(3))
    assert np.array_equal(cholesky_solve(f, np.array([1.0, 2.0, 3.0])), np.array([1.0, 2.0, 3.0]))
    A = np.asfortranarray([[4.0, 2.0], [2.0, 3.0]])
    f = cholesky_factor(A, 2, backend)
    assert np.allclose(f.l, [[2.0, 0.0], [1.0, np.sqrt(2.0)]])
    x = cholesky_solve(f, np.array([6.0, 5.0]))
    assert np.allclose(A @ x, [6.0, 5.0])


def test_cholesky_not_spd_index(backend, golden_next):
    with pytest.raises(NotSpdError) as e:
        cholesky_factor(np.asfortranarray(np.diag([1.0, -1.0])), 2, backend)
    assert e.value.index == int(golden_next["ch_notspd_index"]) == 1
    with pytest.raises(NotSpdError) as e:
        cholesky_factor(golden_next["ch_notspd70_A"], 32, backend)
    assert e.value.index == int(golden_next["ch_notspd70_index"]) == 70
    with pytest.raises(NotSpdError):
        cholesky_factor(np.asfortranarray([[1.0, 2.0], [0.0, 1.0]]), 2, backend)


def test_cholesky_solve_residual_large(backend):
    # multi-outer-panel path (NB = 256, several trailing SYRKs, ragged edge)
    A, b, _ = generate_problem(ProblemSpec(kind="spd", n=1500, seed=11))
    f = cholesky_factor(A, 64, backend)
    x = cholesky_solve(f, b)
    assert relative_residual(A, x, b) <= 1e-10
    x2, rep = solve_system("cholesky", A, b, None, SolverConfig(block_size_b=64), backend)
    assert rep.converged and rep.iterations == 0 and rep.final_relative_residual <= 1e-10


def test_cholesky_counters(backend):
    # reference tallies (direct.py:103-119): scal per column, ger in-panel, one gemm per panel
    n, b = 40, 16
    A, _, _ = generate_problem(ProblemSpec(kind="spd", n=n, seed=0))
    backend.counters.reset()
    cholesky_factor(A, b, backend)
    c = backend.counters
    assert c.scal_calls == n - 1
    assert c.gemm_calls == 2
    assert c.ger_calls == sum(1 for i in range(n) if i + 1 < min((i // b + 1) * b, n))


def test_cholesky_device_resident_no_mutation(backend):
    A, b, _ = generate_problem(ProblemSpec(kind="spd", n=300, seed=2))
    dA = backend.stage_in(A)
    f = cholesky_factor(dA, 64, backend)
    assert np.array_equal(backend.stage_out(dA), A)  # A never mutated
    x = backend.stage_out(cholesky_solve(f, backend.stage_in(b)))
    assert relative_residual(A, x, b) <= 1e-10
