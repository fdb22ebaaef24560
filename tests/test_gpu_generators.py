"""Device generators (csrc/ds_gen.cu) against the reference's NumPy recipes
(harness.py:73-104): the PCG64 stream, every harness kind and the C3 uniform
recipe, fp64 and fp32, ragged sizes across NumPy's pairwise-sum split points
(n < 8, = 128, 129, ...), and the reference-produced golden SHA-256 digests."""
import ctypes
import hashlib

import numpy as np
import pytest

from paper_1511_07207_b200 import _lib
from paper_1511_07207_b200 import harness as H
from paper_1511_07207_b200.device import DeviceArray

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asfortranarray(a)).tobytes(order="F")).hexdigest()


def _raw(be, words, off, rows, cols, colmajor, dtype):
    ctx = be.ctx
    ld = rows if colmajor else cols
    d = DeviceArray(ctx, (rows * cols,), dtype)
    _lib.check(ctx.lib.ds_rng_uniform(ctx.handle, _lib.dtype_code(dtype), words.ctypes.data_as(ctypes.c_void_p),
                                      off, rows, cols, -1.0, 1.0, int(colmajor), ctypes.c_void_p(d.ptr), ld))
    flat = d.to_host()
    return flat.reshape((rows, cols), order="F" if colmajor else "C")


@pytest.mark.parametrize("off", [0, 1, 12345, 2 ** 33 + 7])
@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (70, 130), (129, 64)])
@pytest.mark.parametrize("colmajor", [False, True])
def test_pcg64_stream_bitwise(b200, off, shape, colmajor):
    rng = np.random.default_rng([7, 4096, 2])
    words = H.pcg64_words(rng)
    rng.bit_generator.advance(off)
    want = rng.uniform(-1.0, 1.0, size=shape)
    got = _raw(b200, words, off, *shape, colmajor, np.float64)
    assert np.array_equal(got, want)
    got32 = _raw(b200, words, off, *shape, colmajor, np.float32)
    assert np.array_equal(got32, want.astype(np.float32))


SIZES = [1, 5, 8, 64, 128, 129, 300, 1000]


@pytest.mark.parametrize("kind", ["diag_dominant", "general_nonsymmetric", "uniform"])
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_exact_kinds_bitwise(b200, kind, n, prec):
    if kind == "uniform":
        A, b, xt = H.generate_uniform(n, 3, prec)
    else:
        A, b, xt = H.generate_problem(H.ProblemSpec(kind=kind, n=n, seed=3, precision=prec))
    dA, db, dx = H.generate_problem_device(kind, n, 3, prec, b200)
    assert np.array_equal(dA.to_host(), A)
    assert np.array_equal(dx.to_host(), xt)
    # b = A x_true through the library GEMV (fp64 accumulation) vs NumPy's BLAS
    tol = 1e-13 if prec == "f64" else 2e-6
    np.testing.assert_allclose(db.to_host(), b, rtol=tol, atol=tol * np.abs(A).sum(axis=1).max())


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_spd_matches_recipe(b200, n, prec):
    A, b, xt = H.generate_problem(H.ProblemSpec(kind="spd", n=n, seed=4, precision=prec))
    dA, db, dx = H.generate_problem_device("spd", n, 4, prec, b200)
    G = dA.to_host()
    assert np.array_equal(G, G.T)  # exactly symmetric (harness.py:91)
    assert np.array_equal(dx.to_host(), xt)
    # M^T M: DMMA SYRK vs NumPy's BLAS, differing in summation order only
    tol = 1e-14 if prec == "f64" else 1e-7
    assert np.max(np.abs(G.astype(np.float64) - A)) <= tol * np.max(np.abs(A)) * max(1.0, np.sqrt(n) / 8)
    np.testing.assert_allclose(db.to_host(), b, rtol=1e-5 if prec == "f32" else 1e-12,
                               atol=(1e-5 if prec == "f32" else 1e-12) * np.abs(A).sum(axis=1).max())


def test_golden_digests_of_the_reference(b200, golden):
    """Device A / x_true reproduce the SHA-256 digests recorded by running the reference
    generator itself (tests/golden/make_golden.py) for the exactly restated kinds."""
    seen = 0
    for i in range(int(golden["gen_count"])):
        kind, n, seed, prec = [str(s) for s in golden[f"gen{i}_spec"]]
        if kind not in ("diag_dominant", "general_nonsymmetric"):
            continue
        dA, _, _ = H.generate_problem_device(kind, int(n), int(seed), prec, b200, rhs=False)
        assert sha(dA.to_host()) == str(golden[f"gen{i}_shaA"]), (kind, n, seed, prec)
        seen += 1
    assert seen > 0
