"""CG and restarted GMRES(m) on the B200 (drop-in for densolve.krylov).

Entry points keep the reference signatures, tolerances, stopping rules,
history conventions and exceptions:
  cg_solve(A, b, x0, cfg, backend)                      krylov.py:36-72
  gmres_solve(A, b, x0, cfg, backend, workspace_sink)   krylov.py:75-182
The whole iteration runs in libdensolve_b200 (ds_cg / ds_gmres): one streamed
GEMV per iteration with fused reductions, all scalars and convergence decisions
on the device.  The backend's counters receive the reference's logical op
tallies (gemv/dot/axpy/nrm2/scal per iteration) so cost-law checks hold.

Numerical contract vs the reference: elementwise updates are
bitwise NumPy-identical; reductions are fp64, deterministic, summed in a
different order.  ``orthogonalization="modified"`` runs CGS with one
re-orthogonalisation (CGS2) instead of sequential MGS (north_star: "fused
classical Gram-Schmidt with reorthogonalisation"); ``"classical"`` is the
reference's single-pass CGS exactly.
"""

from __future__ import annotations

import ctypes
import time
from ctypes import c_void_p

import numpy as np

from . import _lib
from .backends import as_b200
from .core import (NotSpdError, SolveReport, SolverConfig, check_system)
from .device import DeviceArray, is_device, to_device
from .sharded import ShardedB200Backend, cg_solve_sharded, gmres_solve_rows


def _tally_cg(be, n: int, iterations: int):
    # setup (krylov.py:45-52): nrm2(b), gemv, axpy, nrm2(r), dot(r,r)
    be.tally("nrm2", 2 * n, 2)
    be.tally("gemv", 2 * n * n)
    be.tally("axpy", 2 * n)
    be.tally("dot", 2 * n)
    if iterations:
        k = iterations  # per iteration: 1 gemv, 2 dot, 3 axpy, 1 nrm2 (krylov.py:55-65)
        be.tally("gemv", 2 * n * n * k, k)
        be.tally("dot", 2 * n * 2 * k, 2 * k)
        be.tally("axpy", 2 * n * 3 * k, 3 * k)
        be.tally("nrm2", 2 * n * k, k)


def cg_solve(A, b, x0, cfg: SolverConfig, backend=None):
    """Conjugate gradients for SPD systems; one streamed matvec per iteration."""
    t0 = time.perf_counter()
    be = as_b200(backend)
    n = check_system(A, b, x0)
    if isinstance(be, ShardedB200Backend):  # rows over several GPUs (sharded.py)
        x, report, info = cg_solve_sharded(A, b, x0, cfg, be)
        _tally_cg(be, n, info.iterations)
        report.wall_time = time.perf_counter() - t0
        return x, report
    ctx = be.ctx
    dA, db, dx0 = to_device(A, ctx), to_device(b, ctx), to_device(x0, ctx)
    dx = DeviceArray(ctx, (n,), dA.dtype)
    cap = int(cfg.iteration_cap(n))
    hist = np.empty(cap + 1, dtype=np.float64)
    info = _lib.SolveInfo()
    st = ctx.lib.ds_cg(ctx.handle, dA.dcode, n, c_void_p(dA.ptr), dA.ld, c_void_p(db.ptr),
                       c_void_p(dx0.ptr), c_void_p(dx.ptr), float(cfg.tolerance), cap, 1,
                       hist.ctypes.data_as(c_void_p), cap + 1, ctypes.byref(info))
    if st == _lib.DS_ENOTSPD:
        raise NotSpdError(_lib.last_error(), index=None)
    _lib.check(st)
    _tally_cg(be, n, info.iterations)
    history = hist[: info.history_len].tolist()
    report = SolveReport(converged=bool(info.converged), iterations=int(info.iterations),
                         final_relative_residual=float(info.final_relative_residual),
                         residual_history=history)
    x = dx if is_device(x0) else dx.to_host()
    report.wall_time = time.perf_counter() - t0
    report.kernel_launches = int(info.kernel_launches)
    return x, report


def _tally_gmres(be, n: int, report: SolveReport, residual_evals: int):
    # per residual evaluation (krylov.py:104-105): gemv + axpy + nrm2
    be.tally("gemv", 2 * n * n * residual_evals, residual_evals)
    be.tally("axpy", 2 * n * residual_evals, residual_evals)
    be.tally("nrm2", 2 * n * residual_evals, residual_evals)
    starts = list(report.restart_cycles or [])
    ends = starts[1:] + [report.iterations]
    for ci, (s, e) in enumerate(zip(starts, ends)):
        inner = e - s
        be.tally("scal", n)  # V[:,0] = scal(1/beta, r) (krylov.py:123)
        for k in range(inner):
            be.tally("gemv", 2 * n * n)
            be.tally("dot", 2 * n * (k + 1), k + 1)
            be.tally("axpy", 2 * n * (k + 1), k + 1)
            be.tally("nrm2", 2 * n)
            last = ci == len(starts) - 1 and k == inner - 1
            if not (last and report.breakdown == "happy-breakdown"):
                be.tally("scal", n)
        # cycle end: x = axpy(1, gemv(V[:, :inner], y), x) (krylov.py:167)
        be.tally("gemv", 2 * n * inner)
        be.tally("axpy", 2 * n)


def gmres_solve(A, b, x0, cfg: SolverConfig, backend=None, workspace_sink: list | None = None):
    """Restarted GMRES(m) with on-device Arnoldi (CGS2/CGS) and Givens least squares."""
    t0 = time.perf_counter()
    be = as_b200(backend)
    n = check_system(A, b, x0)
    if isinstance(be, ShardedB200Backend):  # rows over several GPUs (sharded.py)
        if workspace_sink is not None:
            raise ValueError("workspace_sink is not supported by the sharded backend (V lives in row shards)")
        be.tally("nrm2", 2 * n)
        x, report, info = gmres_solve_rows(A, b, x0, cfg, be)
        _tally_gmres(be, n, report, int(info.residual_evals))
        report.wall_time = time.perf_counter() - t0
        return x, report
    ctx = be.ctx
    m = int(cfg.restart_m)
    dA, db, dx0 = to_device(A, ctx), to_device(b, ctx), to_device(x0, ctx)
    dx = DeviceArray(ctx, (n,), dA.dtype)
    be.tally("nrm2", 2 * n)  # _rhs_norm (krylov.py:87)
    cap = int(cfg.iteration_cap(n))
    hist = np.empty(cap + 2, dtype=np.float64)
    cycles = np.empty(cap + 2, dtype=np.int64)
    info = _lib.SolveInfo()
    dt = dA.dtype

    sink_cb = _lib.SINK_FN(0)
    if workspace_sink is not None:
        def _sink(user, pV, pH, inner, beta):
            V = np.ctypeslib.as_array(ctypes.cast(pV, ctypes.POINTER(np.ctypeslib.as_ctypes_type(dt))),
                                      shape=(n * (m + 1),)).reshape((n, m + 1), order="F").copy(order="F")
            H = np.ctypeslib.as_array(ctypes.cast(pH, ctypes.POINTER(np.ctypeslib.as_ctypes_type(dt))),
                                      shape=((m + 1) * m,)).reshape((m + 1, m), order="F").copy(order="F")
            workspace_sink.append({"V": V, "H": H, "inner": int(inner), "beta": float(beta)})

        sink_cb = _lib.SINK_FN(_sink)
    orth = _lib.DS_ORTH_CLASSICAL if cfg.orthogonalization == "classical" else _lib.DS_ORTH_MODIFIED
    st = ctx.lib.ds_gmres(ctx.handle, dA.dcode, n, c_void_p(dA.ptr), dA.ld, c_void_p(db.ptr),
                          c_void_p(dx0.ptr), c_void_p(dx.ptr), float(cfg.tolerance), cap, m, orth,
                          hist.ctypes.data_as(c_void_p), cap + 2, cycles.ctypes.data_as(c_void_p),
                          cap + 2, sink_cb, None, ctypes.byref(info))
    _lib.check(st)
    report = SolveReport(converged=bool(info.converged), iterations=int(info.iterations),
                         final_relative_residual=float(info.final_relative_residual),
                         residual_history=hist[: info.history_len].tolist(),
                         breakdown="happy-breakdown" if info.breakdown == _lib.DS_BREAKDOWN_HAPPY else None,
                         restart_cycles=[int(c) for c in cycles[: info.cycles_len]])
    _tally_gmres(be, n, report, int(info.residual_evals))
    x = dx if is_device(x0) else dx.to_host()
    report.wall_time = time.perf_counter() - t0
    report.kernel_launches = int(info.kernel_launches)
    return x, report


# loop-exit stages reported by ds_bicgstab in SolveInfo.error_index
_BI_RHO_TOP, _BI_RV_ZERO, _BI_OMEGA, _BI_EARLY, _BI_DONE = 1, 2, 3, 4, 5


def _tally_bicgstab(be, n: int, iterations: int, stage: int):
    """Logical op tallies of krylov.py:185-253 (setup :195-206, full iteration :216-245)."""
    be.tally("nrm2", 2 * n)  # _rhs_norm
    be.tally("gemv", 2 * n * n)
    be.tally("axpy", 2 * n)
    be.tally("dot", 2 * n)
    be.tally("nrm2", 2 * n)
    full = iterations - (1 if stage == _BI_EARLY else 0)
    if full:
        be.tally("gemv", 2 * n * n * 2 * full, 2 * full)
        be.tally("dot", 2 * n * 4 * full, 4 * full)
        be.tally("axpy", 2 * n * 6 * full, 6 * full)
        be.tally("nrm2", 2 * n * 2 * full, 2 * full)
    if stage in (_BI_RV_ZERO, _BI_OMEGA, _BI_EARLY):
        # partial last pass: p update (2 axpy), v = A p, r0hat'v
        be.tally("axpy", 2 * n * 2, 2)
        be.tally("gemv", 2 * n * n)
        be.tally("dot", 2 * n)
    if stage in (_BI_OMEGA, _BI_EARLY):
        be.tally("axpy", 2 * n)  # s
        be.tally("nrm2", 2 * n)
    if stage == _BI_OMEGA:
        be.tally("gemv", 2 * n * n)
        be.tally("dot", 2 * n * 2, 2)
    if stage == _BI_EARLY:
        be.tally("axpy", 2 * n)  # x += alpha p


def bicgstab_solve(A, b, x0, cfg: SolverConfig, backend=None):
    """BiCGSTAB with the shadow residual fixed at r0 (krylov.py:185-253): two streamed
    matvecs per iteration with fused dot/norm epilogues, device-side breakdown tests."""
    t0 = time.perf_counter()
    be = as_b200(backend)
    n = check_system(A, b, x0)
    if isinstance(be, ShardedB200Backend):  # rows over several GPUs (sharded.py)
        x, report, info = cg_solve_sharded(A, b, x0, cfg, be)
        _tally_cg(be, n, info.iterations)
        report.wall_time = time.perf_counter() - t0
        return x, report
    ctx = be.ctx
    dA, db, dx0 = to_device(A, ctx), to_device(b, ctx), to_device(x0, ctx)
    dx = DeviceArray(ctx, (n,), dA.dtype)
    cap = int(cfg.iteration_cap(n))
    hist = np.empty(cap + 1, dtype=np.float64)
    info = _lib.SolveInfo()
    st = ctx.lib.ds_bicgstab(ctx.handle, dA.dcode, n, c_void_p(dA.ptr), dA.ld, c_void_p(db.ptr),
                             c_void_p(dx0.ptr), c_void_p(dx.ptr), float(cfg.tolerance), cap,
                             hist.ctypes.data_as(c_void_p), cap + 1, ctypes.byref(info))
    _lib.check(st)
    _tally_bicgstab(be, n, int(info.iterations), int(info.error_index))
    bd = {_lib.DS_BREAKDOWN_RHO: "rho-breakdown", _lib.DS_BREAKDOWN_OMEGA: "omega-breakdown"}
    report = SolveReport(converged=bool(info.converged), iterations=int(info.iterations),
                         final_relative_residual=float(info.final_relative_residual),
                         residual_history=hist[: info.history_len].tolist(),
                         breakdown=bd.get(int(info.breakdown)))
    x = dx if is_device(x0) else dx.to_host()
    report.wall_time = time.perf_counter() - t0
    report.kernel_launches = int(info.kernel_launches)
    return x, report
