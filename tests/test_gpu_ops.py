"""Op-contract parity on the B200 (backends.py:104-200 tests, re-targeted).

Elementwise ops (axpy, scal, ger) must be BITWISE equal to NumPy: the kernels
round each binary operation exactly as the reference's NumPy expressions do.
Reductions are compared with the reference tests' own tolerances.
"""
import numpy as np
import pytest

from paper_1511_07207_b200 import DimensionError, PrecisionError, to_device

pytestmark = pytest.mark.gpu


def fmat(rng, m, n, dtype=np.float64):
    return np.asfortranarray(rng.uniform(-1.0, 1.0, size=(m, n)).astype(dtype))


def kahan_dot(x, y):
    s = c = 0.0
    for xi, yi in zip(x, y):
        t = s + (xi * yi - c)
        c = (t - s) - (xi * yi - c)
        s = t
    return s


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_axpy_scal_bitwise(backend, rng, dtype):
    for n in (1, 7, 100, 4099):
        x, y = rng.standard_normal(n).astype(dtype), rng.standard_normal(n).astype(dtype)
        assert np.array_equal(backend.axpy(0.37, x, y), y + 0.37 * x)
        assert np.array_equal(backend.scal(-2.5, x), -2.5 * x)
    x = rng.standard_normal(6).astype(dtype)
    assert np.array_equal(backend.scal(1.0, x), x)
    assert np.array_equal(backend.scal(0.0, x), np.zeros(6, dtype))


def test_axpy_errors(backend):
    with pytest.raises(DimensionError):
        backend.axpy(1.0, np.zeros(2), np.zeros(3))
    with pytest.raises(PrecisionError):
        backend.axpy(1.0, np.zeros(2, np.float32), np.zeros(2))


def test_dot_and_nrm2(backend, rng):
    assert backend.dot(np.array([1.0, 2.0, 3.0]), np.array([4.0, 5.0, 6.0])) == 32.0
    x, y = rng.standard_normal(1000), rng.standard_normal(1000)
    assert backend.dot(x, y) == pytest.approx(kahan_dot(x, y), rel=1e-12)
    assert backend.dot(np.zeros(5), np.zeros(5)) == 0.0
    assert backend.dot(np.array([0.0, 1e-30, 0.0]), np.array([0.0, 1e-30, 0.0])) > 0.0
    assert backend.nrm2(np.array([3.0, 4.0])) == pytest.approx(5.0)
    assert backend.nrm2(np.zeros(4)) == 0.0
    big = backend.nrm2(np.array([1e300, 1e300]))
    assert np.isfinite(big) and big == pytest.approx(np.sqrt(2.0) * 1e300, rel=1e-14)
    assert np.isnan(backend.nrm2(np.array([1.0, np.nan])))
    assert backend.nrm2(np.array([1.0, np.inf])) == np.inf
    z = rng.standard_normal(100000)
    assert backend.nrm2(z) == pytest.approx(np.linalg.norm(z), rel=1e-13)


def test_iamax_semantics(backend, rng):
    assert backend.iamax(np.array([1.0, -3.0, 2.0])) == 1
    assert backend.iamax(np.array([2.0, -2.0])) == 0
    x = rng.standard_normal(100000)
    assert backend.iamax(x) == int(np.argmax(np.abs(x)))
    x[5000] = np.nan
    x[7000] = np.nan
    assert backend.iamax(x) == int(np.argmax(np.abs(x))) == 5000
    with pytest.raises(DimensionError):
        backend.iamax(np.zeros(0))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("shape", [(5, 5), (32, 32), (33, 17), (1000, 999), (4096, 4096), (3, 5000)])
def test_gemv(backend, rng, dtype, shape):
    A = fmat(rng, *shape, dtype=dtype)
    x = rng.standard_normal(shape[1]).astype(dtype)
    ref = A.astype(np.float64) @ x.astype(np.float64)
    tol = 1e-13 if dtype == np.float64 else 1e-6
    got = backend.gemv(A, x)
    assert got.dtype == dtype
    np.testing.assert_allclose(got, ref, rtol=tol, atol=tol * np.abs(ref).max())


def test_gemv_small_exact(backend):
    A = np.asfortranarray([[1.0, 2.0], [3.0, 4.0]])
    assert np.array_equal(backend.gemv(A, np.ones(2)), np.array([3.0, 7.0]))
    with pytest.raises(DimensionError):
        backend.gemv(np.asfortranarray(np.eye(3)), np.zeros(4))


def test_gemv_c_order_input(backend, rng):
    A = np.ascontiguousarray(rng.uniform(-1, 1, (300, 200)))
    x = rng.standard_normal(200)
    np.testing.assert_allclose(backend.gemv(A, x), A @ x, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_ger_bitwise(backend, rng, dtype):
    A, x, y = fmat(rng, 67, 45, dtype), rng.standard_normal(67).astype(dtype), rng.standard_normal(45).astype(dtype)
    assert np.array_equal(backend.ger(A, 0.3, x, y), A + 0.3 * np.outer(x, y))
    assert np.array_equal(backend.ger(A, -1.0, x, y), A + -1.0 * np.outer(x, y))
    out = A.copy(order="F")
    r = backend.ger(out, 2.0, x, y, out=out)
    assert r is out and np.array_equal(out, A + 2.0 * np.outer(x, y))


def naive_gemm(alpha, A, B, beta, C):
    return alpha * (A.astype(np.float64) @ B.astype(np.float64)) + beta * C


@pytest.mark.parametrize("mnk", [(4, 3, 4), (64, 64, 64), (130, 70, 33), (257, 129, 64), (1000, 600, 64)])
def test_gemm_fp64_dmma(backend, rng, mnk):
    m, n, k = mnk
    A, B, C = fmat(rng, m, k), fmat(rng, k, n), fmat(rng, m, n)
    u = np.finfo(np.float64).eps / 2
    exp = naive_gemm(0.7, A, B, -0.2, C)
    got = backend.gemm(0.7, A, B, -0.2, C)
    assert np.max(np.abs(got - exp)) <= 50 * k * u * (np.max(np.abs(exp)) + 1)
    # LU form out = C - A B
    got = backend.gemm(-1.0, A, B, 1.0, C)
    exp = C - A @ B
    assert np.max(np.abs(got - exp)) <= 50 * k * u * (np.max(np.abs(exp)) + 1)


def test_gemm_misaligned_views(backend, rng):
    # odd leading dimensions force the 8-byte cp.async path
    W = fmat(rng, 131, 131)
    dW = to_device(W, backend.ctx)
    A, B, C = W[1:100, 3:40], W[3:40, 5:77], W[1:100, 5:77]
    got = backend.gemm(-1.0, np.asfortranarray(A), np.asfortranarray(B), 1.0, np.asfortranarray(C))
    np.testing.assert_allclose(got, C - A @ B, rtol=1e-12, atol=1e-12)
    assert dW.shape == (131, 131)


def test_gemm_fp32(backend, rng):
    A, B, C = fmat(rng, 100, 50, np.float32), fmat(rng, 50, 70, np.float32), fmat(rng, 100, 70, np.float32)
    got = backend.gemm(1.3, A, B, 0.4, C)
    exp = naive_gemm(1.3, A, B, 0.4, C)
    assert np.max(np.abs(got - exp)) <= 50 * 50 * 6e-8 * (np.max(np.abs(exp)) + 1)


def test_gemm_errors_and_counter(backend, rng):
    with pytest.raises(DimensionError):
        backend.gemm(1.0, fmat(rng, 3, 4), fmat(rng, 3, 4), 0.0, fmat(rng, 3, 4))
    A = fmat(rng, 4, 4)
    backend.counters.reset()
    backend.gemm(1.0, A, A, 0.0, A)
    assert backend.counters.gemm_calls == 1 and backend.counters.gemm_flops == 2 * 4 * 4 * 4


@pytest.mark.parametrize("b", [2, 8, 64, 65, 100])
def test_trsm(backend, rng, b):
    L = fmat(rng, b, b)
    B = fmat(rng, b, 37)
    Lu = np.tril(L, -1) + np.eye(b)
    Z = backend.trsm_lower_unit(L, B)
    scale = np.linalg.norm(np.linalg.solve(Lu, B))
    assert np.linalg.norm(Lu @ Z - B) <= 1e-10 * max(1.0, scale)
    U = np.triu(fmat(rng, b, b)) + 2 * np.eye(b)
    np.testing.assert_allclose(U @ backend.trsm_upper(np.asfortranarray(U), B), B, atol=1e-9)


def test_trsm_small_kat(backend):
    L = np.asfortranarray([[1.0, 0.0], [0.5, 1.0]])
    Z = backend.trsm_lower_unit(L, np.asfortranarray([[2.0], [3.0]]))
    assert np.allclose(Z[:, 0], [2.0, 2.0])


def test_each_call_increments_one_counter(backend):
    ops = [("axpy", (1.0, np.ones(3), np.ones(3))), ("dot", (np.ones(3), np.ones(3))),
           ("nrm2", (np.ones(3),)), ("scal", (2.0, np.ones(3))), ("iamax", (np.ones(3),)),
           ("gemv", (np.asfortranarray(np.eye(3)), np.ones(3))),
           ("ger", (np.asfortranarray(np.eye(3)), 1.0, np.ones(3), np.ones(3))),
           ("trsm_lower_unit", (np.asfortranarray(np.eye(3)), np.asfortranarray(np.eye(3))))]
    for op, args in ops:
        before = backend.counters.snapshot()
        getattr(backend, op)(*args)
        after = backend.counters
        assert after.total_calls() == before.total_calls() + 1
        key = "trsm" if op.startswith("trsm") else op
        assert getattr(after, f"{key}_calls") == getattr(before, f"{key}_calls") + 1


def test_staging_roundtrip(backend, rng):
    A = fmat(rng, 37, 19)
    dA = backend.stage_in(A)
    assert dA.shape == (37, 19) and dA.ld % 4 == 0
    assert np.array_equal(backend.stage_out(dA), A)
    C = np.ascontiguousarray(A)
    assert np.array_equal(backend.stage_out(backend.stage_in(C)), A)
    x = rng.standard_normal(11)
    assert np.array_equal(backend.stage_out(backend.stage_in(x)), x)


def test_device_resident_chain(backend, rng):
    A = fmat(rng, 500, 500)
    x = rng.standard_normal(500)
    dA, dx = backend.stage_in(A, x)
    dy = backend.gemv(dA, dx)  # stays on device
    assert hasattr(dy, "ptr")
    np.testing.assert_allclose(backend.stage_out(dy), A @ x, rtol=1e-12, atol=1e-12)


def test_stage_in_async_pipelined_solves(backend):
    # two device buffer sets, the next upload in flight while the current solve runs
    from paper_1511_07207_b200 import SolverConfig, cg_solve, pinned_empty
    from paper_1511_07207_b200.device import DeviceArray
    from paper_1511_07207_b200.harness import ProblemSpec, generate_problem
    outs = []
    probs = [generate_problem(ProblemSpec(kind="spd", n=300, seed=s)) for s in range(4)]
    pinned = []
    for A, b, _ in probs:
        Ap = pinned_empty(A.shape, A.dtype)
        Ap[...] = A
        bp = pinned_empty(b.shape, b.dtype)
        bp[...] = b
        pinned.append((Ap, bp, np.zeros_like(b)))
    ctx = backend.ctx
    bufs = [(DeviceArray(ctx, (300, 300), np.float64), DeviceArray(ctx, (300,), np.float64),
             DeviceArray(ctx, (300,), np.float64)) for _ in range(2)]
    backend.stage_in_async(*pinned[0], out=bufs[0])
    for s in range(4):
        if s + 1 < 4:
            backend.stage_in_async(*pinned[s + 1], out=bufs[(s + 1) % 2])
        x, rep = cg_solve(*bufs[s % 2], SolverConfig(tolerance=1e-10), backend)
        outs.append(x.to_host())
    for (A, b, _), x in zip(probs, outs):
        xs, _ = cg_solve(A, b, np.zeros_like(b), SolverConfig(tolerance=1e-10), backend)
        np.testing.assert_array_equal(x, xs)


def test_gemm_concurrent_streams_bitwise():
    """Two DMMA GEMMs running at the same time on two library contexts (two streams) give
    the bits of the same GEMMs run one after the other (TMA stage-reuse ordering)."""
    from ctypes import c_void_p

    from paper_1511_07207_b200 import _lib
    from paper_1511_07207_b200.device import DeviceArray

    c1, c2 = _lib.Context(0), _lib.Context(0)
    n, K = 4096, 512
    rng = np.random.default_rng(11)
    ops = []
    for ctx in (c1, c2):
        A = DeviceArray.from_host(np.asfortranarray(rng.random((n, K))), ctx)
        B = DeviceArray.from_host(np.asfortranarray(rng.random((K, n))), ctx)
        C = DeviceArray.from_host(np.asfortranarray(rng.random((n, n))), ctx)
        ops.append((ctx, A, B, C))

    def gemm(ctx, A, B, C, out):
        _lib.check(ctx.lib.ds_gemm(ctx.handle, _lib.DS_F64, n, n, K, -1.0, c_void_p(A.ptr), A.ld, c_void_p(B.ptr),
                                   B.ld, 1.0, c_void_p(C.ptr), C.ld, c_void_p(out.ptr), out.ld))

    refs = []
    for ctx, A, B, C in ops:
        out = DeviceArray(ctx, (n, n), np.float64)
        gemm(ctx, A, B, C, out)
        refs.append(out.to_host())
    outs = [DeviceArray(ctx, (n, n), np.float64) for ctx, *_ in ops]
    for _ in range(40):
        for (ctx, A, B, C), out in zip(ops, outs):
            gemm(ctx, A, B, C, out)
        for (ctx, *_), out, ref in zip(ops, outs, refs):
            assert np.array_equal(out.to_host(), ref)
