"""Full-size (BASELINE.json configs) checks through size-independent properties
(the oracle cannot run at these sizes).  Inputs are generated on the
device with torch (seeded) and handed to the public API as DeviceArrays.

* C4 CG n=32768 fp64: converges, the TRUE residual ||b - A x|| / ||b|| (device) meets the
  tolerance the recursive residual claims, residual history monotone-ish and tiny.
* C3 LU n=16384 fp64 (uniform, pivoting family): pivots[k] >= k, |L| <= 1 (partial
  pivoting), lu_solve backward error ~ n u.
* C5 GMRES(50) n=65536 fp32 (one cycle): the Arnoldi basis from workspace_sink is
  orthonormal to fp32 accuracy and the LS estimate matches the true residual.
* Cholesky n=32768 fp64: L L^T x = b solved to ~n u.
"""
import numpy as np
import pytest

from paper_1511_07207_b200 import (SolverConfig, cg_solve, cholesky_factor, cholesky_solve, get_backend,
                                   gmres_solve, lu_factor_blocked, lu_solve, relative_residual)
from paper_1511_07207_b200.device import DeviceArray

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def be():
    return get_backend("b200")


def _dev(be, t, dtype):
    # torch produced t on its own stream and may recycle t's memory once it is freed: order
    # the library's copy after torch's kernels and finish it before returning
    n = t.shape[0]
    d = DeviceArray(be.ctx, tuple(t.shape[::-1]) if t.dim() == 2 else (n,), dtype)
    torch.cuda.synchronize()
    be.ctx.lib.ds_memcpy_d2d(be.ctx.handle, d.ptr, t.data_ptr(), t.numel() * t.element_size())
    be.ctx.synchronize()
    return d


def _spd(n, seed, dtype=torch.float64):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    A = torch.rand((n, n), dtype=dtype, device="cuda", generator=g).mul_(2.0).sub_(1.0)
    A.add_(A.t().clone()).mul_(0.5)
    A.diagonal().add_(float(n) ** 0.5)
    xt = torch.rand(n, dtype=dtype, device="cuda", generator=g).mul_(2.0).sub_(1.0)
    return A, A @ xt, xt


def test_c4_cg_full_size(be):
    n = 32768
    A, b, xt = _spd(n, 0)
    dA, db = _dev(be, A, np.float64), _dev(be, b, np.float64)
    dx0 = DeviceArray(be.ctx, (n,), np.float64)
    be.ctx.lib.ds_memset(be.ctx.handle, dx0.ptr, 0, 8 * n)
    del A
    x, rep = cg_solve(dA, db, dx0, SolverConfig(tolerance=1e-10), be)
    assert rep.converged and rep.iterations < 60
    assert rep.final_relative_residual <= 1e-10
    true_res = relative_residual(dA, x, db)
    assert true_res <= 1e-9  # recursive and true residual agree to a few ulps of growth
    xh = be.stage_out(x)
    assert np.linalg.norm(xh - xt.cpu().numpy()) <= 1e-8 * np.linalg.norm(xt.cpu().numpy())


def test_c3_lu_full_size(be):
    n = 16384
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    A = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g).mul_(2.0).sub_(1.0)
    dA = _dev(be, A, np.float64)
    del A
    f = lu_factor_blocked(dA, 64, be)
    assert not f.singular
    piv = np.asarray(f.pivots)
    assert np.all(piv >= np.arange(n)) and np.all(piv < n)
    P = be.stage_out(f.packed)
    L = np.tril(P, -1)
    assert np.max(np.abs(L)) <= 1.0  # partial pivoting: |l_ij| <= 1
    xt = np.random.default_rng(3).uniform(-1, 1, n)
    b = be.stage_out(dA) @ xt
    x = lu_solve(f, b)
    assert np.linalg.norm(x - xt) <= 1e-7 * np.linalg.norm(xt)


def test_c5_gmres_fp32_one_cycle(be):
    n, m = 65536, 50
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    A = torch.empty((n, n), dtype=torch.float32, device="cuda")
    for c0 in range(0, n, 4096):
        A[c0:c0 + 4096] = torch.rand((4096, n), dtype=torch.float32, device="cuda", generator=g).mul_(2.0).sub_(1.0)
    A.diagonal().add_(1.5 * float(n) ** 0.5)
    xt = torch.rand(n, dtype=torch.float32, device="cuda", generator=g).mul_(2.0).sub_(1.0)
    b = A.t() @ xt
    dA, db = _dev(be, A, np.float32), _dev(be, b, np.float32)
    del A
    dx0 = DeviceArray(be.ctx, (n,), np.float32)
    be.ctx.lib.ds_memset(be.ctx.handle, dx0.ptr, 0, 4 * n)
    sink = []
    x, rep = gmres_solve(dA, db, dx0, SolverConfig(tolerance=1e-300, restart_m=m, max_iterations=m), be,
                         workspace_sink=sink)
    assert rep.iterations == m and len(sink) == 1 and sink[0]["inner"] == m
    V = sink[0]["V"].astype(np.float64)
    G = V.T @ V
    assert np.max(np.abs(G - np.eye(m + 1))) <= 1e-4  # CGS2 keeps the basis orthonormal
    true_res = relative_residual(dA, x, db)
    assert abs(rep.final_relative_residual - true_res) <= 1e-3 * max(true_res, 1e-7)


def test_cholesky_full_size(be):
    n = 32768
    A, b, xt = _spd(n, 2)
    dA, db = _dev(be, A, np.float64), _dev(be, b, np.float64)
    del A
    f = cholesky_factor(dA, 64, be)
    x = cholesky_solve(f, db)
    assert relative_residual(dA, x, db) <= 1e-12
    xh = be.stage_out(x)
    assert np.linalg.norm(xh - xt.cpu().numpy()) <= 1e-10 * np.linalg.norm(xt.cpu().numpy())
