"""The B200 compute backend: the reference's Backend op contract on sm_100a.

Mirrors densolve.backends (/root/reference/pkg/src/densolve/backends.py):
``BackendCounters`` (:30-63) with the same per-op call/flop tallies, the
``Backend`` op set (:76-200: axpy, dot, nrm2, scal, iamax, gemv, ger, gemm,
trsm_lower_unit, trsm_upper) with the same shape/precision errors, the
staging seam (:94-100), and the ``get_backend`` registry (:255-264) with the
name ``"b200"``.

Every op runs on the device through the C ABI.  Host NumPy operands are
staged per call and results come back as new host arrays (the reference's
value semantics); ``DeviceArray`` operands stay on the device.  The fused
solvers (krylov.py / direct.py of this package) do not call these ops one by
one but tally the same logical counters, so the reference's
counter laws still hold.
"""

from __future__ import annotations

import ctypes
from ctypes import c_double, c_int64, c_void_p
from dataclasses import dataclass, fields

import numpy as np

from . import _lib
from .core import DimensionError, check_precision
from .device import DeviceArray, is_device, to_device

_COUNTED_OPS = ("axpy", "dot", "nrm2", "scal", "gemv", "ger", "gemm", "trsm", "iamax")


@dataclass
class BackendCounters:
    axpy_calls: int = 0
    dot_calls: int = 0
    nrm2_calls: int = 0
    scal_calls: int = 0
    gemv_calls: int = 0
    ger_calls: int = 0
    gemm_calls: int = 0
    trsm_calls: int = 0
    iamax_calls: int = 0

    axpy_flops: float = 0.0
    dot_flops: float = 0.0
    nrm2_flops: float = 0.0
    scal_flops: float = 0.0
    gemv_flops: float = 0.0
    ger_flops: float = 0.0
    gemm_flops: float = 0.0
    trsm_flops: float = 0.0
    iamax_flops: float = 0.0

    def reset(self):
        for f in fields(self):
            setattr(self, f.name, 0 if f.name.endswith("_calls") else 0.0)

    def total_calls(self) -> int:
        return sum(getattr(self, f"{op}_calls") for op in _COUNTED_OPS)

    def total_flops(self) -> float:
        return sum(getattr(self, f"{op}_flops") for op in _COUNTED_OPS)

    def snapshot(self) -> "BackendCounters":
        return BackendCounters(**{f.name: getattr(self, f.name) for f in fields(self)})


def _check_vectors(*vs):
    lens = {v.shape[0] for v in vs}
    if len(lens) != 1:
        raise DimensionError(f"vector lengths differ: {sorted(lens)}")
    for v in vs:
        if len(v.shape) != 1:
            raise DimensionError(f"expected 1-d vector, got ndim={len(v.shape)}")
    check_precision(*vs)


class Backend:
    """Operation contract (backends.py:76-200), executed on one B200."""

    name = "abstract"

    def __init__(self):
        self.counters = BackendCounters()

    def tally(self, op: str, flops: float, calls: int = 1):
        c = self.counters
        setattr(c, f"{op}_calls", getattr(c, f"{op}_calls") + calls)
        setattr(c, f"{op}_flops", getattr(c, f"{op}_flops") + flops)

    _tally = tally


class B200Backend(Backend):
    """sm_100a backend; ``device`` selects the GPU (default: $DENSOLVE_B200_DEVICE or 0)."""

    name = "b200"

    def __init__(self, device: int | None = None):
        super().__init__()
        self._device = device
        self._ctx = None

    @property
    def ctx(self) -> _lib.Context:
        if self._ctx is None:
            self._ctx = _lib.context(self._device)
        return self._ctx

    # -- staging seam (backends.py:94-100) -------------------------------------------------
    def stage_in(self, *arrays):
        out = tuple(to_device(a, self.ctx) for a in arrays)
        return out if len(out) != 1 else out[0]

    def stage_in_async(self, *arrays, out=None):
        """Asynchronous stage_in: copies on the context's copy stream (pinned host arrays
        overlap a running solve); a solver consuming the handles waits for the copies.
        ``out`` reuses existing DeviceArrays (e.g. double buffers) instead of allocating."""
        if out is None:
            out = tuple(DeviceArray(self.ctx, np.asarray(a).shape, np.asarray(a).dtype) for a in arrays)
        elif isinstance(out, DeviceArray):
            out = (out,)
        for d, a in zip(out, arrays):
            d.upload_async(a)
        return out if len(out) != 1 else out[0]

    def stage_out(self, *arrays):
        out = tuple(a.to_host() if is_device(a) else a for a in arrays)
        return out if len(out) != 1 else out[0]

    def _out(self, d: DeviceArray, keep_device: bool):
        return d if keep_device else d.to_host()

    # -- level 1 (backends.py:104-132) -----------------------------------------------------
    def axpy(self, alpha: float, x, y):
        _check_vectors(x, y)
        self.tally("axpy", 2 * x.shape[0])
        dx, dy = to_device(x, self.ctx), to_device(y, self.ctx)
        out = DeviceArray(self.ctx, dy.shape, dy.dtype)
        _lib.check(self.ctx.lib.ds_axpy(self.ctx.handle, dx.dcode, dx.shape[0], float(alpha),
                                        c_void_p(dx.ptr), c_void_p(dy.ptr), c_void_p(out.ptr)))
        return self._out(out, is_device(y))

    def dot(self, x, y) -> float:
        _check_vectors(x, y)
        self.tally("dot", 2 * x.shape[0])
        dx, dy = to_device(x, self.ctx), to_device(y, self.ctx)
        r = c_double(0.0)
        _lib.check(self.ctx.lib.ds_dot(self.ctx.handle, dx.dcode, dx.shape[0], c_void_p(dx.ptr),
                                       c_void_p(dy.ptr), ctypes.byref(r)))
        return float(r.value)

    def nrm2(self, x) -> float:
        self.tally("nrm2", 2 * x.shape[0])
        if x.shape[0] == 0:
            return 0.0
        dx = to_device(x, self.ctx)
        r = c_double(0.0)
        _lib.check(self.ctx.lib.ds_nrm2(self.ctx.handle, dx.dcode, dx.shape[0], c_void_p(dx.ptr),
                                        ctypes.byref(r)))
        return float(r.value)

    def scal(self, alpha: float, x):
        self.tally("scal", x.shape[0])
        dx = to_device(x, self.ctx)
        out = DeviceArray(self.ctx, dx.shape, dx.dtype)
        _lib.check(self.ctx.lib.ds_scal(self.ctx.handle, dx.dcode, dx.shape[0], float(alpha),
                                        c_void_p(dx.ptr), c_void_p(out.ptr)))
        return self._out(out, is_device(x))

    def iamax(self, x) -> int:
        if x.shape[0] == 0:
            raise DimensionError("iamax of empty vector")
        self.tally("iamax", 0)
        dx = to_device(x, self.ctx)
        r = c_int64(0)
        _lib.check(self.ctx.lib.ds_iamax(self.ctx.handle, dx.dcode, dx.shape[0], c_void_p(dx.ptr),
                                         ctypes.byref(r)))
        return int(r.value)

    # -- level 2 (backends.py:136-156) -----------------------------------------------------
    def gemv(self, A, x):
        if len(A.shape) != 2 or len(x.shape) != 1 or A.shape[1] != x.shape[0]:
            raise DimensionError(f"gemv shapes {tuple(A.shape)} x {tuple(x.shape)}")
        check_precision(A, x)
        m, n = A.shape
        self.tally("gemv", 2 * m * n)
        dA, dx = to_device(A, self.ctx), to_device(x, self.ctx)
        out = DeviceArray(self.ctx, (m,), dA.dtype)
        _lib.check(self.ctx.lib.ds_gemv(self.ctx.handle, dA.dcode, m, n, c_void_p(dA.ptr), dA.ld,
                                        c_void_p(dx.ptr), c_void_p(out.ptr)))
        return self._out(out, is_device(x))

    def ger(self, A, alpha: float, x, y, out=None):
        m, n = A.shape
        if tuple(x.shape) != (m,) or tuple(y.shape) != (n,):
            raise DimensionError(f"ger shapes {tuple(A.shape)}, x {tuple(x.shape)}, y {tuple(y.shape)}")
        check_precision(A, x, y)
        self.tally("ger", 2 * m * n)
        dA = to_device(A, self.ctx)
        dx, dy = to_device(x, self.ctx), to_device(y, self.ctx)
        dres = dA if (is_device(A) and out is A) else DeviceArray(self.ctx, (m, n), dA.dtype)
        _lib.check(self.ctx.lib.ds_ger(self.ctx.handle, dA.dcode, m, n, c_void_p(dA.ptr), dA.ld,
                                       float(alpha), c_void_p(dx.ptr), c_void_p(dy.ptr),
                                       c_void_p(dres.ptr), dres.ld))
        if out is None:
            return self._out(dres, is_device(A))
        if is_device(out):
            if out is not dres:
                raise ValueError("device ger: out must be A or None")
            return out
        out[...] = dres.to_host()
        return out

    # -- level 3 (backends.py:160-200) -----------------------------------------------------
    def _check_gemm(self, A, B, C):
        if len(A.shape) != 2 or len(B.shape) != 2 or len(C.shape) != 2:
            raise DimensionError("gemm operands must be 2-d")
        m, k = A.shape
        k2, n = B.shape
        if k != k2 or tuple(C.shape) != (m, n):
            raise DimensionError(f"gemm shapes {tuple(A.shape)} @ {tuple(B.shape)} -> {tuple(C.shape)}")
        check_precision(A, B, C)
        self.tally("gemm", 2 * m * n * k)
        return m, n, k

    def gemm(self, alpha: float, A, B, beta: float, C, out=None):
        """alpha * A @ B + beta * C (DMMA tensor-core path for fp64)."""
        m, n, k = self._check_gemm(A, B, C)
        dA, dB, dC = to_device(A, self.ctx), to_device(B, self.ctx), to_device(C, self.ctx)
        dres = dC if (is_device(C) and out is C) else DeviceArray(self.ctx, (m, n), dC.dtype)
        _lib.check(self.ctx.lib.ds_gemm(self.ctx.handle, dA.dcode, m, n, k, float(alpha),
                                        c_void_p(dA.ptr), dA.ld, c_void_p(dB.ptr), dB.ld, float(beta),
                                        c_void_p(dC.ptr), dC.ld, c_void_p(dres.ptr), dres.ld))
        if out is None:
            return self._out(dres, is_device(C))
        if is_device(out):
            if out is not dres:
                raise ValueError("device gemm: out must be C or None")
            return out
        out[...] = dres.to_host()
        return out

    def trsm_lower_unit(self, L, B):
        b = L.shape[0]
        if tuple(L.shape) != (b, b) or len(B.shape) != 2 or B.shape[0] != b:
            raise DimensionError(f"trsm shapes {tuple(L.shape)}, {tuple(B.shape)}")
        check_precision(L, B)
        self.tally("trsm", b * (b - 1) * B.shape[1])
        dL, dB = to_device(L, self.ctx), to_device(B, self.ctx)
        dZ = DeviceArray(self.ctx, tuple(B.shape), dB.dtype)
        _lib.check(self.ctx.lib.ds_trsm_lower_unit(self.ctx.handle, dL.dcode, b, B.shape[1],
                                                   c_void_p(dL.ptr), dL.ld, c_void_p(dB.ptr), dB.ld,
                                                   c_void_p(dZ.ptr), dZ.ld))
        return self._out(dZ, is_device(B))

    def trsm_upper(self, U, B):
        b = U.shape[0]
        if tuple(U.shape) != (b, b) or len(B.shape) != 2 or B.shape[0] != b:
            raise DimensionError(f"trsm shapes {tuple(U.shape)}, {tuple(B.shape)}")
        check_precision(U, B)
        self.tally("trsm", b * b * B.shape[1])
        dU, dB = to_device(U, self.ctx), to_device(B, self.ctx)
        dZ = DeviceArray(self.ctx, tuple(B.shape), dB.dtype)
        _lib.check(self.ctx.lib.ds_trsm_upper(self.ctx.handle, dU.dcode, b, B.shape[1],
                                              c_void_p(dU.ptr), dU.ld, c_void_p(dB.ptr), dB.ld,
                                              c_void_p(dZ.ptr), dZ.ld))
        return self._out(dZ, is_device(B))


BACKEND_NAMES = ("b200",)


def get_backend(name: str = "b200", **kwargs) -> Backend:
    """Construct a backend by name (backends.py:258-264).  Only ``"b200"`` exists:
    the reference's CPU backends are not part of this package (no CPU fallback).
    ``devices=[...]`` (one process, several GPUs) or ``distributed=True`` (one process
    per GPU under torch.distributed) return the sharded backend (sharded.py)."""
    if name == "b200":
        if kwargs.get("devices") is not None or kwargs.get("distributed"):
            from .sharded import ShardedB200Backend
            return ShardedB200Backend(**kwargs)
        kwargs.pop("devices", None)
        kwargs.pop("distributed", None)
        return B200Backend(**kwargs)
    raise ValueError(f"unknown backend {name!r}; expected one of {BACKEND_NAMES}")


def as_b200(backend) -> B200Backend:
    """Accept a B200Backend instance, a backend name, or None (default device)."""
    if backend is None:
        return B200Backend()
    if isinstance(backend, str):
        return get_backend(backend)
    if isinstance(backend, B200Backend):
        return backend
    raise TypeError(f"backend {backend!r} is not a B200Backend; this package has no CPU backends")
