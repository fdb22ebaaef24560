"""Device-resident operands: the staging seam of the Backend contract.

The reference keeps ``Backend.stage_in`` / ``stage_out`` as identity hooks
"preserved for a future accelerator backend" (backends.py:94-100);
here they are real host<->device transfers.  ``DeviceArray`` is a column-major
(F-order) device buffer with a leading dimension padded to a multiple of 4
elements so every column starts 32-byte aligned (128-bit vector loads in the
GEMV, 16-byte cp.async in the GEMM).  Solver entry points accept either NumPy
arrays (uploaded per call, like the reference's per-call arrays) or
``DeviceArray`` handles (no transfer).
"""

from __future__ import annotations

import ctypes
import weakref
from ctypes import c_double, c_int64, c_void_p

import numpy as np

from . import _lib, core

LD_ALIGN = 4


def _release_device(lib, handle, ptr, inflight, ctx=None):
    # ctx: held by the finalizer so the context outlives every buffer allocated on it
    """Finalizer of a DeviceArray: the context stream first waits for a still pending
    asynchronous upload into the buffer (copy stream), then frees it stream-ordered."""
    if inflight[0] is not None:
        lib.ds_wait_event(handle, inflight[0])
        lib.ds_event_destroy(inflight[0])
        inflight[0] = inflight[1] = None
    lib.ds_free(handle, c_void_p(ptr))


def _padded_ld(rows: int) -> int:
    return max(LD_ALIGN, (rows + LD_ALIGN - 1) // LD_ALIGN * LD_ALIGN)


class DeviceArray:
    """A 1-d vector or 2-d column-major matrix in device memory."""

    __slots__ = ("ctx", "shape", "dtype", "ld", "ptr", "_fin", "_inflight", "__weakref__")

    def __init__(self, ctx: _lib.Context, shape, dtype, ld: int | None = None):
        self.ctx = ctx
        self.shape = tuple(int(s) for s in shape)
        self.dtype = np.dtype(dtype)
        _lib.dtype_code(self.dtype)
        if len(self.shape) == 1:
            self.ld = max(self.shape[0], 1)
            nbytes = self.shape[0] * self.dtype.itemsize
        elif len(self.shape) == 2:
            self.ld = ld if ld is not None else _padded_ld(self.shape[0])
            nbytes = self.ld * max(self.shape[1], 1) * self.dtype.itemsize
        else:
            raise core.DimensionError(f"device arrays are 1-d or 2-d, got shape {self.shape}")
        p = c_void_p()
        _lib.check(ctx.lib.ds_malloc(ctx.handle, max(nbytes, 16), ctypes.byref(p)))
        self.ptr = p.value
        # [event, host array] of an in-flight asynchronous upload (upload_async); shared with
        # the finalizer so a handle dropped before its copy finished is freed only after it
        self._inflight = [None, None]
        self._fin = weakref.finalize(self, _release_device, ctx.lib, ctx.handle, self.ptr, self._inflight, ctx)

    # -- numpy-like metadata used by the validators -------------------------------------
    @property
    def ndim(self) -> int:
        return len(self.shape)

    @property
    def nbytes(self) -> int:
        if self.ndim == 1:
            return self.shape[0] * self.dtype.itemsize
        return self.ld * self.shape[1] * self.dtype.itemsize

    @property
    def dcode(self) -> int:
        return _lib.dtype_code(self.dtype)

    @property
    def __cuda_array_interface__(self):
        """Zero-copy view for CUDA-aware consumers (e.g. ``torch.as_tensor(d, device="cuda")``):
        a 2-d array is column-major with the padded leading dimension.  No stream is named;
        the consumer orders its work after the library's stream itself."""
        it = self.dtype.itemsize
        strides = None if self.ndim == 1 else (it, self.ld * it)
        return {"shape": self.shape, "typestr": self.dtype.str, "data": (self.ptr, False),
                "strides": strides, "version": 2}

    def free(self):
        self._fin()

    def __repr__(self):
        return f"DeviceArray(shape={self.shape}, dtype={self.dtype}, ld={self.ld}, device={self.ctx.device})"

    # -- transfers -------------------------------------------------------------------------
    @classmethod
    def empty(cls, shape, dtype, ctx: _lib.Context | None = None):
        return cls(ctx or _lib.context(), shape, dtype)

    @classmethod
    def from_host(cls, a, ctx: _lib.Context | None = None):
        ctx = ctx or _lib.context()
        a = np.asarray(a)
        _lib.dtype_code(a.dtype)
        out = cls(ctx, a.shape, a.dtype)
        out.upload(a)
        return out

    def upload(self, a):
        a = np.asarray(a)
        if a.shape != self.shape or a.dtype != self.dtype:
            raise core.DimensionError(f"upload of {a.shape}/{a.dtype} into {self.shape}/{self.dtype}")
        self.settle()
        lib, h = self.ctx.lib, self.ctx.handle
        if self.ndim == 1:
            a = np.ascontiguousarray(a)
            _lib.check(lib.ds_memcpy_h2d(h, c_void_p(self.ptr), a.ctypes.data_as(c_void_p), a.nbytes))
            return
        rows, cols = self.shape
        if a.flags.f_contiguous:
            order, ld_host = 0, rows
        elif a.flags.c_contiguous:
            order, ld_host = 1, cols
        else:
            a = np.asfortranarray(a)
            order, ld_host = 0, rows
        _lib.check(lib.ds_upload_matrix(h, self.dcode, a.ctypes.data_as(c_void_p), rows, cols,
                                        max(ld_host, 1), order, c_void_p(self.ptr), self.ld))

    def upload_async(self, a):
        """Stage a host array (F-order or 1-d; pinned for a true async copy) on the context's
        copy stream; the next solver call on this array waits for it (pipelined solves)."""
        a = np.asarray(a)
        if a.shape != self.shape or a.dtype != self.dtype:
            raise core.DimensionError(f"upload of {a.shape}/{a.dtype} into {self.shape}/{self.dtype}")
        if self.ndim == 2 and not a.flags.f_contiguous:
            raise ValueError("upload_async needs an F-order (column-major) host matrix")
        self.settle()
        rows, cols = (self.shape[0], 1) if self.ndim == 1 else self.shape
        ev = c_void_p()
        _lib.check(self.ctx.lib.ds_upload_async(self.ctx.handle, self.dcode, a.ctypes.data_as(c_void_p), rows, cols,
                                                max(rows, 1), c_void_p(self.ptr), self.ld if self.ndim == 2
                                                else max(rows, 1), ctypes.byref(ev)))
        self._inflight[0], self._inflight[1] = ev, a
        return self

    def settle(self):
        """Order the context stream after a pending asynchronous upload into this array."""
        if self._inflight[0] is not None:
            _lib.check(self.ctx.lib.ds_wait_event(self.ctx.handle, self._inflight[0]))
            self.ctx.lib.ds_event_destroy(self._inflight[0])
            self._inflight[0] = self._inflight[1] = None

    def to_host(self, out: np.ndarray | None = None) -> np.ndarray:
        self.settle()
        lib, h = self.ctx.lib, self.ctx.handle
        if self.ndim == 1:
            if out is None:
                out = np.empty(self.shape, dtype=self.dtype)
            _lib.check(lib.ds_memcpy_d2h(h, out.ctypes.data_as(c_void_p), c_void_p(self.ptr), out.nbytes))
            return out
        rows, cols = self.shape
        if out is None:
            out = np.empty((rows, cols), dtype=self.dtype, order="F")
        assert out.flags.f_contiguous
        _lib.check(lib.ds_download_matrix(h, self.dcode, c_void_p(self.ptr), rows, cols, self.ld,
                                          out.ctypes.data_as(c_void_p), max(rows, 1)))
        return out

    def copy(self) -> "DeviceArray":
        self.settle()
        out = DeviceArray(self.ctx, self.shape, self.dtype, ld=self.ld)
        _lib.check(self.ctx.lib.ds_memcpy_d2d(self.ctx.handle, c_void_p(out.ptr), c_void_p(self.ptr),
                                              self.nbytes))
        return out

    def col_ptr(self, j: int) -> int:
        return self.ptr + j * self.ld * self.dtype.itemsize


def to_device(a, ctx: _lib.Context | None = None) -> DeviceArray:
    """Stage a host operand (no-op for a DeviceArray on the same context)."""
    ctx = ctx or _lib.context()
    if isinstance(a, DeviceArray):
        if a.ctx is not ctx:
            raise ValueError("operand lives on another device context")
        a.settle()
        return a
    return DeviceArray.from_host(a, ctx)


def is_device(a) -> bool:
    return isinstance(a, DeviceArray)


# ---- pinned host memory (for end-to-end transfers at full PCIe rate) ---------------------
class _PinnedOwner:
    """Owns a page-locked allocation and exposes it through the array interface, so every
    NumPy array or view made from it keeps it (and the allocation) alive."""

    def __init__(self, ptr, nbytes, lib):
        self.ptr = ptr
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
        self._fin = weakref.finalize(self, lib.ds_host_free, c_void_p(ptr))


def pinned_empty(shape, dtype, order="F") -> np.ndarray:
    """A NumPy array backed by page-locked host memory (freed when the last array or view
    that refers to it goes away)."""
    lib = _lib.load_library()
    dt = np.dtype(dtype)
    count = int(np.prod(shape))
    nbytes = max(count * dt.itemsize, 16)
    p = c_void_p()
    _lib.check(lib.ds_host_alloc(nbytes, ctypes.byref(p)))
    raw = np.asarray(_PinnedOwner(p.value, nbytes, lib))  # base chain ends at the owner
    return raw[: count * dt.itemsize].view(dt).reshape(shape, order=order)


def relative_residual_device(A, x, b) -> float:
    ctx = A.ctx if isinstance(A, DeviceArray) else _lib.context()
    dA, dx, db = to_device(A, ctx), to_device(x, ctx), to_device(b, ctx)
    out = c_double(0.0)
    _lib.check(ctx.lib.ds_relative_residual(ctx.handle, dA.dcode, dA.shape[0], c_void_p(dA.ptr), dA.ld,
                                            c_void_p(dx.ptr), c_void_p(db.ptr), ctypes.byref(out)))
    return float(out.value)


def launches(ctx: _lib.Context | None = None) -> int:
    return (ctx or _lib.context()).launches()


__all__ = ["DeviceArray", "to_device", "is_device", "pinned_empty", "relative_residual_device",
           "launches", "c_int64"]
