"""LU / triangular-solve parity on the B200 (test_direct.py, test_acceptance.py
criteria 5/7/8 patterns) against golden vectors from the reference.

Contract (north_star): identical pivot sequence; solution within a stated
relative tolerance.  The panel arithmetic reproduces NumPy's rounding, so the
UNBLOCKED factorization (and blocked with b = n) is bitwise the reference's.
"""
import numpy as np
import pytest

from oracle import densolve_oracle as O
from paper_1511_07207_b200 import (DimensionError, SingularMatrixError, backward_substitution,
                                   forward_substitution, lu_factor_blocked, lu_factor_unblocked,
                                   lu_solve, permutation_matrix, permutation_sign, relative_residual,
                                   unit_roundoff)
from paper_1511_07207_b200.harness import ProblemSpec, generate_problem, generate_well_separated

pytestmark = pytest.mark.gpu


def lu_residual(A, f):
    P = permutation_matrix(f.pivots, f.n, dtype=np.float64)
    return np.linalg.norm(P @ A.astype(np.float64) - f.lower().astype(np.float64) @ f.upper().astype(np.float64))


def test_unblocked_bitwise_reference(backend, golden):
    A = generate_well_separated(64, seed=3)
    f = lu_factor_unblocked(A, backend)
    assert np.array_equal(f.pivots, golden["lu_ws64_unb_piv"])
    assert np.array_equal(f.packed, golden["lu_ws64_unb_packed"])
    U = golden["lu_u128_A"]
    f = lu_factor_unblocked(U, backend)
    assert np.array_equal(f.pivots, golden["lu_u128_unb_piv"])
    assert np.array_equal(f.packed, golden["lu_u128_unb_packed"])


def test_blocked_full_width_is_unblocked_bitwise(backend, rng):
    A = np.asfortranarray(rng.uniform(-1.0, 1.0, size=(24, 24)))
    ref = lu_factor_unblocked(A, backend)
    blk = lu_factor_blocked(A, 24, backend)
    assert np.array_equal(ref.pivots, blk.pivots) and np.array_equal(ref.packed, blk.packed)
    Wo, po, _ = O.lu_factor_unblocked(A)
    assert np.array_equal(ref.packed, Wo) and np.array_equal(ref.pivots, po)


@pytest.mark.parametrize("b", [1, 8, 32, 64])
def test_blocked_well_separated_vs_reference(backend, golden, b):
    A = generate_well_separated(64, seed=3)
    f = lu_factor_blocked(A, b, backend)
    assert np.array_equal(f.pivots, golden[f"lu_ws64_b{b}_piv"])
    u = unit_roundoff(np.float64)
    assert np.max(np.abs(f.packed - golden[f"lu_ws64_b{b}_packed"])) <= 100 * 64 * u * np.max(np.abs(A))


@pytest.mark.parametrize("b", [8, 32])
def test_blocked_uniform_vs_reference(backend, golden, b):
    A = golden["lu_u128_A"]
    f = lu_factor_blocked(A, b, backend)
    assert np.array_equal(f.pivots, golden[f"lu_u128_b{b}_piv"])
    np.testing.assert_allclose(f.packed, golden[f"lu_u128_b{b}_packed"], rtol=0, atol=1e-11)
    assert lu_residual(A, f) <= 10 * 128 * unit_roundoff(np.float64) * np.linalg.norm(A)


def test_kats(backend):
    f = lu_factor_unblocked(np.asfortranarray([[0.0, 1.0], [1.0, 0.0]]), backend)
    assert list(f.pivots) == [1, 1]
    assert np.array_equal(f.lower(), np.eye(2)) and np.array_equal(f.upper(), np.eye(2))
    A = np.asfortranarray([[4.0, 3.0], [6.0, 3.0]])
    f = lu_factor_unblocked(A, backend)
    assert f.pivots[0] == 1 and f.packed[1, 0] == pytest.approx(2.0 / 3.0)
    assert np.allclose(f.upper(), [[6.0, 3.0], [0.0, 1.0]])
    f = lu_factor_unblocked(np.asfortranarray([[1.0, 2.0], [2.0, 4.0]]), backend)
    assert f.singular
    with pytest.raises(SingularMatrixError):
        lu_solve(f, np.ones(2))


def test_oversized_block_warns(backend, rng):
    A = np.asfortranarray(rng.uniform(-1.0, 1.0, size=(8, 8)))
    with pytest.warns(UserWarning):
        f = lu_factor_blocked(A, 100, backend)
    assert not f.singular
    with pytest.raises(ValueError):
        lu_factor_blocked(A, 0, backend)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [4, 16, 64, 256])
def test_residual_families(backend, dtype, n):
    rng = np.random.default_rng(n)
    u = unit_roundoff(dtype)
    for seed in range(25):
        A = np.asfortranarray(rng.uniform(-1.0, 1.0, size=(n, n)).astype(dtype))
        f = lu_factor_blocked(A, min(64, n), backend)
        assert lu_residual(A, f) <= 10 * n * u * np.linalg.norm(A.astype(np.float64))
        Wo, po, _ = O.lu_factor_blocked(A, min(64, n))
        assert np.array_equal(f.pivots, po)


def test_f32_golden(backend, golden):
    f = lu_factor_blocked(golden["lu_f32_64_A"], 64, backend)
    assert np.array_equal(f.pivots, golden["lu_f32_64_piv"])
    assert np.array_equal(f.packed, golden["lu_f32_64_packed"])


@pytest.mark.parametrize("n", [512, 1024])
def test_harness_family_identity_pivots(backend, golden, n):
    A, b, _ = generate_problem(ProblemSpec(kind="general_nonsymmetric", n=n, seed=0))
    f = lu_factor_blocked(A, 64, backend)
    assert np.array_equal(f.pivots, golden[f"lu_gn{n}_piv"])
    x = lu_solve(f, b)
    np.testing.assert_allclose(x, golden[f"lu_gn{n}_x"], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("n", [256, 512])
def test_uniform_family_pivots_and_solution(backend, golden, n):
    A = np.asfortranarray(np.random.default_rng([0, n, 1]).uniform(-1.0, 1.0, (n, n)))
    b = np.random.default_rng([0, n, 2]).uniform(-1.0, 1.0, n)
    f = lu_factor_blocked(A, 64, backend)
    assert np.array_equal(f.pivots, golden[f"lu_uni{n}_piv"])
    x = lu_solve(f, b)
    xr = golden[f"lu_uni{n}_x"]
    assert np.linalg.norm(x - xr, np.inf) <= 1e-9 * np.linalg.norm(xr, np.inf)


def test_acceptance_criterion5_pivot_agreement(backend):
    u = unit_roundoff(np.float64)
    for n in (64, 256, 512):
        for seed in range(4):
            A = generate_well_separated(n, seed=seed)
            ref = lu_factor_unblocked(A, backend)
            assert np.linalg.norm(permutation_matrix(ref.pivots, n) @ A - ref.lower() @ ref.upper()) \
                <= 10 * n * u * np.linalg.norm(A)
            for b in (1, 8, 64, n):
                blk = lu_factor_blocked(A, b, backend)
                assert np.array_equal(ref.pivots, blk.pivots)


def test_level3_dominance_and_flop_law(backend):
    A = generate_well_separated(1024, seed=0)
    backend.counters.reset()
    lu_factor_blocked(A, 64, backend)
    c = backend.counters
    assert c.gemm_flops / c.total_flops() > 0.90
    for n in (256, 512, 1024):
        backend.counters.reset()
        lu_factor_unblocked(generate_well_separated(n, seed=1), backend)
        model = 2.0 * n ** 3 / 3.0
        assert abs(backend.counters.total_flops() - model) / model < 0.05


@pytest.mark.slow
def test_lu_uniform_2048_pivots_vs_oracle(backend):
    n = 2048
    A = np.asfortranarray(np.random.default_rng([1, n, 1]).uniform(-1.0, 1.0, (n, n)))
    f = lu_factor_blocked(A, 64, backend)
    W, piv, _ = O.lu_factor_blocked(A, 64)
    assert np.array_equal(f.pivots, piv)
    assert np.max(np.abs(f.packed - W)) <= 1e-9 * np.max(np.abs(W))


def test_substitution(backend, rng):
    assert np.array_equal(forward_substitution(np.asfortranarray(np.eye(3)), np.array([1.0, 2.0, 3.0])),
                          np.array([1.0, 2.0, 3.0]))
    L = np.asfortranarray([[1.0, 0.0], [0.5, 1.0]])
    assert np.array_equal(forward_substitution(L, np.array([2.0, 3.0]), unit_diagonal=True), np.array([2.0, 2.0]))
    U = np.asfortranarray([[2.0, 1.0], [0.0, 4.0]])
    assert np.array_equal(backward_substitution(U, np.array([4.0, 8.0])), np.array([1.0, 2.0]))
    for n in (64, 1000, 4099):
        L = np.asfortranarray(np.tril(rng.uniform(-1.0, 1.0, size=(n, n)), -1) / n + np.eye(n))
        b = rng.standard_normal(n)
        y = forward_substitution(L, b, unit_diagonal=True)
        assert np.linalg.norm(L @ y - b) <= 10 * n * unit_roundoff(np.float64) * np.linalg.norm(b)
        Uu = np.asfortranarray(np.triu(rng.uniform(-1.0, 1.0, size=(n, n)), 1) / n + 4.0 * np.eye(n))
        x = backward_substitution(Uu, b)
        assert np.linalg.norm(Uu @ x - b) <= 10 * n * unit_roundoff(np.float64) * np.linalg.norm(b)
    with pytest.raises(SingularMatrixError, match="row 1"):
        forward_substitution(np.asfortranarray(np.diag([1.0, 0.0])), np.ones(2))
    with pytest.raises(SingularMatrixError, match="row 0"):
        backward_substitution(np.asfortranarray(np.diag([0.0, 1.0])), np.ones(2))
    with pytest.raises(DimensionError):
        forward_substitution(np.asfortranarray(np.eye(3)), np.ones(2))


def test_lu_solve_kats(backend, rng):
    f = lu_factor_unblocked(np.asfortranarray(np.eye(3)), backend)
    assert np.array_equal(lu_solve(f, np.array([1.0, 2.0, 3.0])), np.array([1.0, 2.0, 3.0]))
    f = lu_factor_unblocked(np.asfortranarray([[0.0, 1.0], [1.0, 0.0]]), backend)
    assert np.array_equal(lu_solve(f, np.array([5.0, 7.0])), np.array([7.0, 5.0]))
    n = 256
    A = np.asfortranarray(rng.uniform(-1.0, 1.0, size=(n, n)) + 2 * n * np.eye(n))
    b = rng.standard_normal(n)
    x = lu_solve(lu_factor_blocked(A, 64, backend), b)
    assert relative_residual(A, x, b) <= 1e-10
    with pytest.raises(DimensionError):
        lu_solve(lu_factor_blocked(A, 64, backend), np.ones(3))


@pytest.mark.parametrize("seed", range(8))
def test_determinant_consistency(backend, seed):
    rng = np.random.default_rng(seed)
    A = np.asfortranarray(rng.uniform(-1.0, 1.0, size=(5, 5)))
    f = lu_factor_unblocked(A, backend)
    det = permutation_sign(f.pivots) * np.prod(np.diag(f.upper()))
    assert det == pytest.approx(np.linalg.det(A), rel=1e-8)


def test_relative_residual_device(backend, rng):
    A = np.asfortranarray(rng.standard_normal((8, 8)))
    x, b = rng.standard_normal(8), rng.standard_normal(8)
    assert relative_residual(A, x, b) == pytest.approx(O.relative_residual(A, x, b), rel=1e-13)
    assert relative_residual(np.asfortranarray(np.eye(2)), np.zeros(2), np.array([3.0, 4.0])) == 1.0


# ---- larger / ragged shapes through the register-row panel kernel (several CTA
# layouts: 256-row CTAs, the 4-threads-per-row tail, ragged last panels).  The pivot
# oracle at these sizes is LAPACK getrf (scipy), which SURVEY.md §8c validated to give
# the reference's pivots on these families.
@pytest.mark.parametrize("n,b", [(3001, 64), (4096, 64), (2500, 48), (1300, 100)])
def test_lu_large_ragged_pivots_vs_lapack(backend, n, b):
    sl = pytest.importorskip("scipy.linalg")
    A = np.asfortranarray(np.random.default_rng([n, b]).uniform(-1.0, 1.0, (n, n)))
    f = lu_factor_blocked(A, b, backend)
    lu_ref, piv_ref = sl.lu_factor(A)
    np.testing.assert_array_equal(f.pivots, piv_ref)
    # same pivots; factors agree to summation-order noise relative to the factor scale
    # (LAPACK's recursive blocking groups the trailing updates differently again)
    d = np.max(np.abs(f.packed - lu_ref)) / np.max(np.abs(lu_ref))
    assert d <= 1e-12 * n, d
    xt = np.random.default_rng(1).uniform(-1, 1, n)
    x = lu_solve(f, A @ xt)
    assert np.linalg.norm(x - xt) <= 1e-8 * np.linalg.norm(xt)


def test_lu_large_singular_column(backend):
    # an exactly zero column in the middle of a large matrix: singular flag, the
    # reference's semantics (skip scale / rank-1 update, keep going), pivots = LAPACK's
    sl = pytest.importorskip("scipy.linalg")
    n = 2000
    A = np.asfortranarray(np.random.default_rng(5).uniform(-1.0, 1.0, (n, n)))
    A[:, 1234] = 0.0
    f = lu_factor_blocked(A, 64, backend)
    assert f.singular
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, piv_ref = sl.lu_factor(A, check_finite=False)
    np.testing.assert_array_equal(f.pivots[:1234], piv_ref[:1234])
    with pytest.raises(Exception):
        lu_solve(f, np.ones(n))


def test_lu_f32_large(backend):
    sl = pytest.importorskip("scipy.linalg")
    n = 2048
    A = np.asfortranarray(np.random.default_rng(11).uniform(-1.0, 1.0, (n, n)).astype(np.float32))
    f = lu_factor_blocked(A, 64, backend)
    assert f.packed.dtype == np.float32
    _, piv_ref = sl.lu_factor(A.astype(np.float64))
    # fp32 rounding may legitimately flip a near-tie; nearly all pivots agree
    assert np.mean(f.pivots == piv_ref) > 0.99
    xt = np.random.default_rng(2).uniform(-1, 1, n).astype(np.float32)
    x = lu_solve(f, A @ xt)
    assert np.linalg.norm(x - xt) <= 1e-2 * np.linalg.norm(xt)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_lu_lookahead_bitwise_equals_serial(backend, monkeypatch, dtype):
    """The look-ahead schedule (next panel factored on a side stream while the trailing GEMM
    runs on the main stream, L-column swaps on a third) computes exactly what the serial
    schedule computes: same kernels, same operands, disjoint columns.  Guards the concurrent
    TMA-fed GEMMs (a stage refill racing in-flight fragment loads once broke this at n=8192)."""
    from paper_1511_07207_b200 import lu_factor_blocked

    n = 8192
    A = np.asfortranarray(np.random.default_rng(n).uniform(-1, 1, (n, n)).astype(dtype))
    monkeypatch.setenv("DENSOLVE_LU_LOOKAHEAD", "1")
    f1 = lu_factor_blocked(A, 64, backend)
    monkeypatch.setenv("DENSOLVE_LU_LOOKAHEAD", "0")
    f0 = lu_factor_blocked(A, 64, backend)
    assert np.array_equal(np.asarray(f1.pivots), np.asarray(f0.pivots))
    assert np.array_equal(f1.packed, f0.packed)
