"""Blocked LU with partial pivoting and triangular solves on the B200
(drop-in for densolve.direct).

  lu_factor_blocked(A, b, backend)   direct.py:50-84
  lu_factor_unblocked(A, backend)    direct.py:25-47   (== blocked with b = n, bitwise)
  lu_solve(f, b)                     direct.py:155-163
  forward_substitution(L, b, unit_diagonal=False)   direct.py:123-136
  backward_substitution(U, y)                        direct.py:139-152
  cholesky_factor(A, b, backend)                     direct.py:87-120
  cholesky_solve(f, b)                               direct.py:166-171

Factorization runs in libdensolve_b200 (ds_lu_factor): cooperative panel kernel
(first-max pivot search, swap, reciprocal scale, rank-1 panel update — NumPy
rounding, bitwise the reference's), laswp, unit-lower TRSM and an FP64 DMMA
trailing-update GEMM per panel.  Counters get the reference's per-column and
per-panel tallies (iamax / scal / ger / trsm / gemm).
"""

from __future__ import annotations

import ctypes
import warnings
from ctypes import c_int32, c_int64, c_void_p

import numpy as np

from . import _lib
from .backends import B200Backend, as_b200
from .core import (CholeskyFactor, DimensionError, LuFactors, NotSpdError, SingularMatrixError,
                   check_precision, check_square)
from .device import DeviceArray, is_device, to_device
from .sharded import ShardedB200Backend, lu_factor_block_cyclic_api


def _tally_lu(be, n: int, b: int, zero_cols: np.ndarray, blocked: bool):
    """The reference's per-column / per-panel counter tallies (direct.py:66-83), in closed
    form: scal and ger per non-zero pivot column, trsm and gemm per panel."""
    c = be.counters
    c.iamax_calls += n
    i = np.arange(n, dtype=np.int64)
    bf = np.minimum((i // b + 1) * b, n)
    live = (zero_cols[:n] == 0) & (i + 1 < n)
    tail = n - i - 1
    be.tally("scal", int(tail[live].sum()), calls=int(live.sum()))
    g = live & (i + 1 < bf)
    be.tally("ger", int((2 * tail[g] * (bf[g] - i[g] - 1)).sum()), calls=int(g.sum()))
    if blocked:
        for kb in range(0, n, b):
            bf_ = min(kb + b, n)
            if bf_ < n:
                w = bf_ - kb
                be.tally("trsm", w * (w - 1) * (n - bf_))
                be.tally("gemm", 2 * (n - bf_) * (n - bf_) * w)


def _factor(A, b: int, backend, blocked: bool) -> LuFactors:
    be = as_b200(backend)
    n = check_square(A)
    check_precision(A)
    counting = be  # the caller's backend receives the counter tallies
    if isinstance(be, ShardedB200Backend) and be.nshards == 1:
        # one shard owns every column block: the single-GPU factorization (look-ahead panel
        # stream, TMA-fed trailing GEMM) on that shard's device
        be = B200Backend(device=be.devices[0])
    if isinstance(be, ShardedB200Backend) and not is_device(A):
        # columns dealt to the shards in NB-wide blocks (1-D block-cyclic, sharded.py)
        packed, piv, singular = lu_factor_block_cyclic_api(A, max(b, 1), be)
        zero = np.zeros(max(n, 1), dtype=np.int8)
        zero[:n] = np.diagonal(packed) == 0
        _tally_lu(counting, n, max(b, 1), zero, blocked)
        return LuFactors(packed=packed, pivots=piv.astype(np.intp), singular=singular)
    ctx = be.ctx
    src = to_device(A, ctx)
    W = src.copy() if is_device(A) else src  # never mutate the caller's A (direct.py:61)
    piv = np.empty(n, dtype=np.intp)
    zero = np.zeros(max(n, 1), dtype=np.int8)
    sing = c_int32(0)
    _lib.check(ctx.lib.ds_lu_factor(ctx.handle, W.dcode, n, c_void_p(W.ptr), W.ld, max(b, 1),
                                    piv.ctypes.data_as(c_void_p), zero.ctypes.data_as(c_void_p),
                                    ctypes.byref(sing)))
    _tally_lu(counting, n, max(b, 1), zero, blocked)
    packed = W if is_device(A) else W.to_host()
    return LuFactors(packed=packed, pivots=piv, singular=bool(sing.value), device=W)


def lu_factor_unblocked(A, backend=None) -> LuFactors:
    """Right-looking LU, rank-1 update per column (one panel spanning the matrix)."""
    n = check_square(A)
    return _factor(A, max(n, 1), backend, blocked=False)


def lu_factor_blocked(A, b: int, backend=None) -> LuFactors:
    """Blocked right-looking LU: panel, full-row swaps, TRSM, DMMA trailing GEMM."""
    n = check_square(A)
    check_precision(A)
    if b < 1:
        raise ValueError("block size must be >= 1")
    if b > n:
        warnings.warn(f"block size {b} exceeds n={n}; clamping to n")
        b = n
    return _factor(A, b, backend, blocked=True)


def _solve_ctx(*arrays):
    for a in arrays:
        if is_device(a):
            return a.ctx
    return _lib.context()


def forward_substitution(L, b, unit_diagonal: bool = False):
    """Solve L y = b by a blocked device forward sweep over the lower triangle."""
    n = check_square(L)
    if tuple(b.shape) != (n,):
        raise DimensionError(f"rhs shape {tuple(b.shape)} does not conform to {n}x{n}")
    check_precision(L, b)
    ctx = _solve_ctx(L, b)
    dL, db = to_device(L, ctx), to_device(b, ctx)
    dy = DeviceArray(ctx, (n,), dL.dtype)
    bad = c_int64(-1)
    st = ctx.lib.ds_forward_substitution(ctx.handle, dL.dcode, n, c_void_p(dL.ptr), dL.ld,
                                         c_void_p(db.ptr), c_void_p(dy.ptr), 1 if unit_diagonal else 0,
                                         ctypes.byref(bad))
    _lib.check(st)
    return dy if is_device(b) else dy.to_host()


def backward_substitution(U, y):
    """Solve U x = y by a blocked device backward sweep over the upper triangle."""
    n = check_square(U)
    if tuple(y.shape) != (n,):
        raise DimensionError(f"rhs shape {tuple(y.shape)} does not conform to {n}x{n}")
    check_precision(U, y)
    ctx = _solve_ctx(U, y)
    dU, dy = to_device(U, ctx), to_device(y, ctx)
    dx = DeviceArray(ctx, (n,), dU.dtype)
    bad = c_int64(-1)
    st = ctx.lib.ds_backward_substitution(ctx.handle, dU.dcode, n, c_void_p(dU.ptr), dU.ld,
                                          c_void_p(dy.ptr), c_void_p(dx.ptr), ctypes.byref(bad))
    _lib.check(st)
    return dx if is_device(y) else dx.to_host()


def lu_solve(f: LuFactors, b):
    """x = U^-1 L^-1 P b from packed factors, entirely on the device."""
    if f.singular:
        raise SingularMatrixError("LU factors are flagged singular")
    if tuple(b.shape) != (f.n,):
        raise DimensionError(f"rhs shape {tuple(b.shape)} does not conform to n={f.n}")
    check_precision(f.packed, b)
    dLU = f.device if isinstance(f.device, DeviceArray) else None
    ctx = dLU.ctx if dLU is not None else _solve_ctx(f.packed, b)
    if dLU is None:
        dLU = to_device(f.packed, ctx)
    db = to_device(b, ctx)
    dx = DeviceArray(ctx, (f.n,), dLU.dtype)
    piv = np.ascontiguousarray(np.asarray(f.pivots, dtype=np.int64))
    _lib.check(ctx.lib.ds_lu_solve(ctx.handle, dLU.dcode, f.n, c_void_p(dLU.ptr), dLU.ld,
                                   piv.ctypes.data_as(c_void_p), c_void_p(db.ptr), c_void_p(dx.ptr)))
    return dx if is_device(b) else dx.to_host()


def _tally_cholesky(be, n: int, b: int):
    """direct.py:103-119 counter tallies: scal per column, ger inside the panel, one gemm per panel."""
    i = np.arange(n, dtype=np.int64)
    bf = np.minimum((i // b + 1) * b, n)
    tail = n - i - 1
    live = tail > 0
    be.tally("scal", int(tail[live].sum()), calls=int(live.sum()))
    g = i + 1 < bf
    be.tally("ger", int((2 * tail[g] * (bf[g] - i[g] - 1)).sum()), calls=int(g.sum()))
    for kb in range(0, n, b):
        bf_ = min(kb + b, n)
        if bf_ < n:
            be.tally("gemm", 2 * (n - bf_) * (n - bf_) * (bf_ - kb))


def cholesky_factor(A, b: int, backend=None) -> CholeskyFactor:
    """Blocked right-looking Cholesky: exact panel kernels (diagonal block + per-row column
    sweep) and a lower-tile FP64 DMMA SYRK for the trailing update."""
    be = as_b200(backend)
    n = check_square(A)
    check_precision(A)
    if b < 1:
        raise ValueError("block size must be >= 1")
    b = min(b, n)
    ctx = be.ctx
    src = to_device(A, ctx)
    W = src.copy() if is_device(A) else src  # never mutate the caller's A (direct.py:102)
    bad = c_int64(-1)
    st = ctx.lib.ds_cholesky_factor(ctx.handle, W.dcode, n, c_void_p(W.ptr), W.ld, max(b, 1),
                                    ctypes.byref(bad))
    if st == _lib.DS_ENOTSPD:
        idx = int(bad.value)
        raise NotSpdError(_lib.last_error(), index=None if idx < 0 else idx)
    _lib.check(st)
    _tally_cholesky(be, n, max(b, 1))
    return CholeskyFactor(l=W if is_device(A) else W.to_host(), device=W)


def cholesky_solve(f: CholeskyFactor, b):
    """Solve L y = b then L^T x = y (the transposed sweep reads L in place)."""
    if tuple(b.shape) != (f.n,):
        raise DimensionError(f"rhs shape {tuple(b.shape)} does not conform to n={f.n}")
    check_precision(f.l, b)
    dL = f.device if isinstance(f.device, DeviceArray) else None
    ctx = dL.ctx if dL is not None else _solve_ctx(f.l, b)
    if dL is None:
        dL = to_device(f.l, ctx)
    db = to_device(b, ctx)
    dx = DeviceArray(ctx, (f.n,), dL.dtype)
    bad = c_int64(-1)
    _lib.check(ctx.lib.ds_cholesky_solve(ctx.handle, dL.dcode, f.n, c_void_p(dL.ptr), dL.ld,
                                         c_void_p(db.ptr), c_void_p(dx.ptr), ctypes.byref(bad)))
    return dx if is_device(b) else dx.to_host()
