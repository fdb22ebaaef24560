"""ctypes binding of ``libdensolve_b200.so`` (the C ABI in include/densolve_b200.h).

This is the only module that touches the shared library.  Every public entry
point of the package goes through it; there is no CPU fallback: if the library
is missing or no CUDA device is visible, calls raise ``RuntimeError``.

Status codes map 1:1 onto the reference exceptions (core.py:17-42 of
/root/reference/pkg/src/densolve).
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref
from ctypes import (POINTER, c_char_p, c_double, c_int, c_int8, c_int32, c_int64, c_size_t, c_uint64,
                    c_void_p)

import numpy as np

from . import core

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdensolve_b200.so")

(DS_OK, DS_EDIM, DS_EPREC, DS_EDEGRHS, DS_ESINGULAR, DS_ENOTSPD, DS_EINVAL, DS_ECUDA, DS_ENOMEM, DS_EMM,
 DS_ENOFILE) = range(11)
DS_F32, DS_F64 = 0, 1
DS_ORTH_MODIFIED, DS_ORTH_CLASSICAL = 0, 1
DS_BREAKDOWN_NONE, DS_BREAKDOWN_HAPPY, DS_BREAKDOWN_RHO, DS_BREAKDOWN_OMEGA = 0, 1, 2, 3


class SolveInfo(ctypes.Structure):
    _fields_ = [
        ("converged", c_int32),
        ("breakdown", c_int32),
        ("iterations", c_int64),
        ("final_relative_residual", c_double),
        ("history_len", c_int64),
        ("cycles_len", c_int64),
        ("error_index", c_int64),
        ("error_value", c_double),
        ("kernel_launches", c_int64),
        ("residual_evals", c_int64),
    ]


SINK_FN = ctypes.CFUNCTYPE(None, c_void_p, c_void_p, c_void_p, c_int64, c_double)

# name -> (restype, argtypes); the exported symbol set of include/densolve_b200.h
_SIGNATURES = {
    "ds_last_error": (c_char_p, []),
    "ds_version": (c_char_p, []),
    "ds_device_count": (c_int, [POINTER(c_int)]),
    "ds_ctx_create": (c_int, [c_int, POINTER(c_void_p)]),
    "ds_ctx_destroy": (c_int, [c_void_p]),
    "ds_ctx_set_stream": (c_int, [c_void_p, c_void_p]),
    "ds_ctx_synchronize": (c_int, [c_void_p]),
    "ds_ctx_kernel_launches": (c_int, [c_void_p, POINTER(c_int64)]),
    "ds_malloc": (c_int, [c_void_p, c_size_t, POINTER(c_void_p)]),
    "ds_free": (c_int, [c_void_p, c_void_p]),
    "ds_host_alloc": (c_int, [c_size_t, POINTER(c_void_p)]),
    "ds_host_free": (c_int, [c_void_p]),
    "ds_host_register": (c_int, [c_void_p, c_size_t]),
    "ds_host_unregister": (c_int, [c_void_p]),
    "ds_memcpy_h2d": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t]),
    "ds_memcpy_d2h": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t]),
    "ds_memcpy_d2d": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t]),
    "ds_memset": (c_int, [c_void_p, c_void_p, c_int, c_size_t]),
    "ds_upload_matrix": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64, c_int,
                                 c_void_p, c_int64]),
    "ds_download_matrix": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64,
                                   c_void_p, c_int64]),
    "ds_axpy": (c_int, [c_void_p, c_int, c_int64, c_double, c_void_p, c_void_p, c_void_p]),
    "ds_dot": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_void_p, POINTER(c_double)]),
    "ds_nrm2": (c_int, [c_void_p, c_int, c_int64, c_void_p, POINTER(c_double)]),
    "ds_scal": (c_int, [c_void_p, c_int, c_int64, c_double, c_void_p, c_void_p]),
    "ds_iamax": (c_int, [c_void_p, c_int, c_int64, c_void_p, POINTER(c_int64)]),
    "ds_gemv": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p]),
    "ds_ger": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64, c_double, c_void_p,
                       c_void_p, c_void_p, c_int64]),
    "ds_gemm": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int64, c_double, c_void_p, c_int64,
                        c_void_p, c_int64, c_double, c_void_p, c_int64, c_void_p, c_int64]),
    "ds_trsm_lower_unit": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64,
                                   c_void_p, c_int64, c_void_p, c_int64]),
    "ds_trsm_upper": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                              c_int64, c_void_p, c_int64]),
    "ds_cg": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                      c_double, c_int64, c_int, c_void_p, c_int64, POINTER(SolveInfo)]),
    "ds_gmres": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                         c_void_p, c_double, c_int64, c_int64, c_int, c_void_p, c_int64,
                         c_void_p, c_int64, SINK_FN, c_void_p, POINTER(SolveInfo)]),
    "ds_bicgstab": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                            c_double, c_int64, c_void_p, c_int64, POINTER(SolveInfo)]),
    "ds_lu_factor": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_int64, c_void_p,
                             c_void_p, POINTER(c_int32)]),
    "ds_lu_factor_dev": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_int64,
                                 c_void_p, POINTER(c_int32)]),
    "ds_upload_async": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64,
                                POINTER(c_void_p)]),
    "ds_wait_event": (c_int, [c_void_p, c_void_p]),
    "ds_event_destroy": (c_int, [c_void_p]),
    # row-sharded CG over peer memory (ds_shard.cu)
    "ds_shardset_create": (c_int, [c_int, c_void_p, c_void_p, c_int, c_int, c_int64, c_int64, POINTER(c_void_p)]),
    "ds_shardset_info": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int64)]),
    "ds_shardset_connect_local": (c_int, [c_void_p]),
    "ds_shardset_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "ds_shardset_connect_ipc": (c_int, [c_void_p, c_void_p]),
    "ds_shardset_destroy": (c_int, [c_void_p]),
    "ds_shardset_gather": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "ds_lu_block_cyclic": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int64, c_void_p, POINTER(c_int32)]),
    "ds_gmres_sharded": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_double, c_int64,
                                 c_int64, c_int, c_void_p, c_int64, c_void_p, c_int64, POINTER(SolveInfo)]),
    "ds_cg_sharded": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_double, c_int64,
                              c_int, c_void_p, c_int64, POINTER(SolveInfo)]),
    "ds_mm_read": (c_int, [c_char_p, c_void_p, c_int64, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
    "ds_mm_last_error": (c_char_p, []),
    "ds_cholesky_factor": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_int64, POINTER(c_int64)]),
    "ds_cholesky_solve": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                                  POINTER(c_int64)]),
    "ds_lu_solve": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                            c_void_p]),
    "ds_forward_substitution": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_void_p,
                                        c_void_p, c_int, POINTER(c_int64)]),
    "ds_backward_substitution": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_void_p,
                                         c_void_p, POINTER(c_int64)]),
    "ds_relative_residual": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_void_p,
                                     c_void_p, POINTER(c_double)]),
    "ds_symmetry_check": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, POINTER(c_double),
                                  POINTER(c_double)]),
    # seeded generators at config scale (ds_gen.cu)
    "ds_rng_uniform": (c_int, [c_void_p, c_int, c_void_p, c_uint64, c_int64, c_int64, c_double, c_double, c_int,
                               c_void_p, c_int64]),
    "ds_generate": (c_int, [c_void_p, c_int, c_int, c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    # multi-GPU building blocks
    "ds_vec_parts": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_void_p]),
    "ds_dot_dev": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_void_p, c_void_p]),
    "ds_gemv_acc": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p]),
    "ds_resid_parts": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                               c_void_p, c_void_p]),
    "ds_cg_shard_init": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_double, c_int64]),
    "ds_cg_shard_update": (c_int, [c_void_p, c_int, c_int64, c_int, c_void_p, c_void_p, c_int64, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p]),
    "ds_cg_shard_finish": (c_int, [c_void_p, c_int, c_int64, c_int, c_void_p, c_void_p, c_int64, c_void_p,
                                   c_void_p, c_void_p, c_double, c_int64]),
    "ds_multidot_dev": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "ds_cgs_update_shard": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_int, c_void_p, c_int,
                                    c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_int64]),
    "ds_gmres_shard_start": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                                     c_void_p]),
    "ds_gmres_shard_step": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                    c_int64, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_double,
                                    c_int64, c_int64]),
    "ds_gmres_lsq": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_void_p, c_int, c_void_p, c_void_p]),
    "ds_absdiff_transposed": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_int64,
                                      c_void_p]),
    "ds_lu_panel": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "ds_laswp": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str | None = None):
    """Load (once) and type the shared library.  Raises RuntimeError if absent."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = path or os.environ.get("DENSOLVE_B200_LIB", LIB_PATH)
        if not os.path.exists(p):
            raise RuntimeError(
                f"libdensolve_b200.so not found at {p}: build it with "
                f"`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        lib = ctypes.CDLL(p)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    msg = load_library().ds_last_error()
    return msg.decode() if msg else ""


def check(status: int, *, index=None):
    """Raise the reference exception class matching a C status code."""
    if status == DS_OK:
        return
    msg = last_error()
    if status == DS_EDIM:
        raise core.DimensionError(msg)
    if status == DS_EPREC:
        raise core.PrecisionError(msg)
    if status == DS_EDEGRHS:
        raise core.DegenerateRhsError(msg)
    if status == DS_ESINGULAR:
        raise core.SingularMatrixError(msg)
    if status == DS_ENOTSPD:
        raise core.NotSpdError(msg, index=index)
    if status == DS_EINVAL:
        raise ValueError(msg)
    if status == DS_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"densolve_b200: {msg} (status {status})")


def dtype_code(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return DS_F64
    if dt == np.float32:
        return DS_F32
    raise core.PrecisionError(f"unsupported scalar type {dt}")


class Context:
    """One CUDA device context (stream + scratch) of the library."""

    def __init__(self, device: int = 0, owned: bool = False):
        """owned=True: a private context (e.g. one per shard of a sharded backend) that is
        destroyed with this object; the per-device defaults of context() live for the process."""
        self.lib = load_library()
        n = c_int(0)
        self.lib.ds_device_count(ctypes.byref(n))
        if n.value == 0:
            raise RuntimeError("densolve_b200 requires a CUDA (sm_100a) device; none is visible "
                               "and there is no CPU fallback")
        h = c_void_p()
        check(self.lib.ds_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.device = device
        if owned:  # device arrays keep their context alive (DeviceArray finalizer), so this runs last
            weakref.finalize(self, self.lib.ds_ctx_destroy, h)

    def launches(self) -> int:
        v = c_int64(0)
        check(self.lib.ds_ctx_kernel_launches(self.handle, ctypes.byref(v)))
        return v.value

    def synchronize(self):
        check(self.lib.ds_ctx_synchronize(self.handle))

    def set_stream(self, stream_ptr: int | None):
        check(self.lib.ds_ctx_set_stream(self.handle, c_void_p(stream_ptr or 0)))


_contexts: dict[int, Context] = {}
_ctx_lock = threading.Lock()


def context(device: int | None = None) -> Context:
    if device is None:
        device = int(os.environ.get("DENSOLVE_B200_DEVICE", "0"))
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx


def device_count() -> int:
    try:
        lib = load_library()
    except RuntimeError:
        return 0
    n = c_int(0)
    lib.ds_device_count(ctypes.byref(n))
    return n.value
