"""Multi-GPU behind the reference API: ``get_backend("b200", devices=[...])``.

The reference selects a backend by name with keyword arguments
(``get_backend(name, **kwargs)``, /root/reference/pkg/src/densolve/backends.py:258-264).
Here ``devices=[d0, d1, ...]`` makes a backend whose solves shard the system over
those GPUs from ONE process, and ``distributed=True`` makes one whose solves shard
over the ranks of ``torch.distributed`` (one process per GPU, launched by torchrun,
every rank calling the solver with the same host arrays).  The solver entry points
are unchanged: ``cg_solve(A, b, x0, cfg, backend)`` (krylov.py:36-72) detects the
sharded backend, splits A by rows (shard q owns rows [q*n_loc, (q+1)*n_loc)),
uploads each row block to its GPU and runs ``ds_cg_sharded`` — the whole iteration
loop in the library, the all-gathers fused into the kernels over NVLink peer
memory.  x comes back whole, the report is the reference's.

Device-resident repeated solves (the bench's ``value``): ``backend.stage_in(A)``
returns a :class:`ShardedMatrix`, ``backend.stage_in(b)`` a :class:`ShardedVector`;
``cg_solve`` accepts them and returns a ShardedVector when x0 is one.
"""

from __future__ import annotations

import ctypes
import weakref
from ctypes import c_int, c_int64, c_void_p

import numpy as np

from . import _lib
from .backends import B200Backend
from .core import DimensionError, check_precision
from .device import DeviceArray, _padded_ld


def _ptr_array(ptrs):
    return (c_void_p * len(ptrs))(*[c_void_p(p) for p in ptrs])


def _destroy_shardset(lib, handle, ctxs):
    # ctxs: held until here so the shard contexts outlive the exchange regions
    lib.ds_shardset_destroy(handle)


class ShardSet:
    """One ds_shardset: the exchange regions of the local shards for a system of size n."""

    def __init__(self, backend: "ShardedB200Backend", n: int, dtype, xbytes: int | None = None):
        self.lib = _lib.load_library()
        self.n = int(n)
        self.dtype = np.dtype(dtype)
        self.dcode = _lib.dtype_code(self.dtype)
        self.G = backend.nshards
        self.ranks = backend.local_ranks
        self.ctxs = backend.shard_contexts
        n_loc = -(-self.n // self.G)
        if xbytes is None:  # the symmetry gate's transposed blocks (row-sharded Krylov)
            xbytes = n_loc * n_loc * self.dtype.itemsize
        xbytes = xbytes if self.G > 1 else 0
        h = c_void_p()
        arr = (c_void_p * len(self.ctxs))(*[c.handle for c in self.ctxs])
        ranks = (c_int * len(self.ranks))(*self.ranks)
        _lib.check(self.lib.ds_shardset_create(len(self.ctxs), arr, ranks, self.G, self.dcode, self.n, xbytes,
                                               ctypes.byref(h)))
        self.handle = h
        # destroyed before its contexts: the finalizer holds them
        self._fin = weakref.finalize(self, _destroy_shardset, self.lib, h, tuple(self.ctxs))
        a, b = c_int64(0), c_int64(0)
        _lib.check(self.lib.ds_shardset_info(h, ctypes.byref(a), ctypes.byref(b)))
        self.n_loc, self.N = a.value, b.value
        if backend.distributed:
            self._connect_ipc(backend)
        else:
            _lib.check(self.lib.ds_shardset_connect_local(h))

    def _connect_ipc(self, backend):
        import torch.distributed as dist

        buf = (ctypes.c_ubyte * 64)()
        _lib.check(self.lib.ds_shardset_ipc_handle(self.handle, ctypes.cast(buf, c_void_p)))
        allh = [None] * self.G
        dist.all_gather_object(allh, bytes(buf), group=backend.group)
        flat = (ctypes.c_ubyte * (64 * self.G)).from_buffer_copy(b"".join(allh))
        _lib.check(self.lib.ds_shardset_connect_ipc(self.handle, ctypes.cast(flat, c_void_p)))

    def rows(self, q: int) -> tuple[int, int]:
        r0 = q * self.n_loc
        return r0, max(r0, min(self.n, r0 + self.n_loc))

    def gather(self, vecs: list[DeviceArray]) -> np.ndarray:
        out = np.empty(self.n, dtype=self.dtype)
        _lib.check(self.lib.ds_shardset_gather(self.handle, self.dcode, _ptr_array([v.ptr for v in vecs]),
                                               out.ctypes.data_as(c_void_p)))
        return out

    def close(self):
        self._fin()
        self.handle = None


class ShardedMatrix:
    """Row blocks of an n x n matrix: blocks[i] is the n_loc x n column-major block of
    local shard i (rows past n zero)."""

    def __init__(self, sset: ShardSet, blocks: list[DeviceArray]):
        self.sset, self.blocks = sset, blocks
        self.shape = (sset.n, sset.n)
        self.dtype = sset.dtype
        self.ndim = 2


class ShardedVector:
    """Row slices of an n-vector: parts[i] holds the n_loc entries of local shard i."""

    def __init__(self, sset: ShardSet, parts: list[DeviceArray]):
        self.sset, self.parts = sset, parts
        self.shape = (sset.n,)
        self.dtype = sset.dtype
        self.ndim = 1

    def to_host(self) -> np.ndarray:
        return self.sset.gather(self.parts)


def is_sharded(a) -> bool:
    return isinstance(a, (ShardedMatrix, ShardedVector))


class ShardedB200Backend(B200Backend):
    """The B200 backend sharded over several GPUs.

    ``devices``: CUDA ordinals, one row shard each, all driven from this process (a
    device may repeat: its shards then share the GPU — used to test the exchange on a
    one-GPU box; shards sharing a GPU need their own hardware work queues, so set
    CUDA_DEVICE_MAX_CONNECTIONS=32 before CUDA initialises).  ``distributed=True``: one shard per torch.distributed rank, on
    ``device`` (default: LOCAL_RANK).  The op contract (axpy, gemv, ...) runs on the
    first local device; the solvers shard.
    """

    name = "b200"

    def __init__(self, devices=None, distributed: bool = False, device: int | None = None, group=None):
        import os

        if distributed:
            import torch.distributed as dist

            if not dist.is_initialized():
                raise RuntimeError("get_backend('b200', distributed=True) needs an initialised torch.distributed "
                                   "process group (launch with torchrun)")
            self.group = group
            rank, size = dist.get_rank(group), dist.get_world_size(group)
            dev = device if device is not None else int(os.environ.get("LOCAL_RANK", rank))
            self.devices = [dev]
            self.local_ranks = [rank]
            self.nshards = size
        else:
            if not devices:
                raise ValueError("devices must list at least one CUDA device")
            self.group = None
            self.devices = [int(d) for d in devices]
            self.local_ranks = list(range(len(self.devices)))
            self.nshards = len(self.devices)
        if self.nshards > 16:
            raise ValueError(f"at most 16 shards, got {self.nshards}")
        self.distributed = bool(distributed)
        super().__init__(device=self.devices[0])
        self._shard_ctxs = None
        self._sets: dict[tuple[int, str], ShardSet] = {}

    @property
    def shard_contexts(self) -> list[_lib.Context]:
        # private contexts (own streams and workspaces), so shards sharing a GPU run concurrently
        if self._shard_ctxs is None:
            self._shard_ctxs = [_lib.Context(d, owned=True) for d in self.devices]
        return self._shard_ctxs

    def shardset(self, n: int, dtype, kind: str = "rows", nb: int = 0) -> ShardSet:
        """The exchange regions for systems of size n: "rows" (row-sharded Krylov) or "lu"
        (block-cyclic LU with nb-wide column blocks: two panel slots of n x nb)."""
        key = (int(n), np.dtype(dtype).str, kind, int(nb))
        s = self._sets.get(key)
        if s is None:
            xb = None
            if kind == "lu":
                r256 = lambda v: -(-v // 256) * 256  # noqa: E731
                xb = 2 * (r256(n * nb * np.dtype(dtype).itemsize) + r256(nb * 8) + r256(nb))
            s = ShardSet(self, n, dtype, xbytes=xb)
            self._sets[key] = s
        return s

    # -- staging (backends.py:94-100) for device-resident sharded solves -------------------
    def stage_in(self, *arrays):
        out = tuple(self._stage(a) for a in arrays)
        return out if len(out) != 1 else out[0]

    def _stage(self, a):
        if is_sharded(a):
            return a
        a = np.asarray(a)
        check_precision(a)
        if a.ndim == 2:
            if a.shape[0] != a.shape[1]:
                raise DimensionError(f"matrix must be square, got shape {a.shape}")
            return self.shard_matrix(a)
        if a.ndim == 1:
            return self.shard_vector(a)
        raise DimensionError(f"expected a 1-d or 2-d array, got ndim={a.ndim}")

    def stage_out(self, *arrays):
        out = tuple(a.to_host() if is_sharded(a) else a for a in arrays)
        return out if len(out) != 1 else out[0]

    def shard_matrix(self, A: np.ndarray) -> ShardedMatrix:
        n = A.shape[0]
        ss = self.shardset(n, A.dtype)
        if not (A.flags.f_contiguous or A.flags.c_contiguous):
            A = np.asfortranarray(A)
        it = A.dtype.itemsize
        blocks = []
        for ctx, q in zip(ss.ctxs, ss.ranks):
            r0, r1 = ss.rows(q)
            d = DeviceArray(ctx, (ss.n_loc, n), A.dtype, ld=_padded_ld(ss.n_loc))
            lib, h = ctx.lib, ctx.handle
            if r1 - r0 < ss.n_loc:
                _lib.check(lib.ds_memset(h, c_void_p(d.ptr), 0, d.nbytes))
            if r1 > r0:
                if A.flags.f_contiguous:  # rows r0:r1 of an F-order matrix: column stride n
                    src, order, ld_host = A.ctypes.data + r0 * it, 0, n
                else:                     # C-order: rows are contiguous, row stride n
                    src, order, ld_host = A.ctypes.data + r0 * n * it, 1, n
                _lib.check(lib.ds_upload_matrix(h, d.dcode, c_void_p(src), r1 - r0, n, ld_host, order,
                                                c_void_p(d.ptr), d.ld))
            blocks.append(d)
        return ShardedMatrix(ss, blocks)

    def shard_vector(self, v: np.ndarray, ss: ShardSet | None = None) -> ShardedVector:
        ss = ss or self.shardset(v.shape[0], v.dtype)
        v = np.ascontiguousarray(v)
        parts = []
        for ctx, q in zip(ss.ctxs, ss.ranks):
            r0, r1 = ss.rows(q)
            d = DeviceArray(ctx, (ss.n_loc,), v.dtype)
            if r1 - r0 < ss.n_loc:
                _lib.check(ctx.lib.ds_memset(ctx.handle, c_void_p(d.ptr), 0, d.nbytes))
            if r1 > r0:
                _lib.check(ctx.lib.ds_memcpy_h2d(ctx.handle, c_void_p(d.ptr), c_void_p(v.ctypes.data + r0 * v.itemsize),
                                                 (r1 - r0) * v.itemsize))
            parts.append(d)
        return ShardedVector(ss, parts)

    def empty_vector(self, ss: ShardSet) -> ShardedVector:
        return ShardedVector(ss, [DeviceArray(c, (ss.n_loc,), ss.dtype) for c in ss.ctxs])

    def close(self):
        for s in self._sets.values():
            s.close()
        self._sets.clear()


def cg_solve_sharded(A, b, x0, cfg, be: ShardedB200Backend):
    """krylov.cg_solve (krylov.py:36-72) over the backend's shards; see ds_cg_sharded."""
    from .core import NotSpdError, SolveReport

    n = A.shape[0]
    dA = be._stage(A)
    ss = dA.sset
    db = b if is_sharded(b) else be.shard_vector(np.asarray(b), ss)
    dx0 = x0 if is_sharded(x0) else be.shard_vector(np.asarray(x0), ss)
    for v in (db, dx0):
        if v.sset is not ss:
            raise ValueError("sharded operands belong to different shard sets")
    dx = be.empty_vector(ss)
    cap = int(cfg.iteration_cap(n))
    hist = np.empty(cap + 1, dtype=np.float64)
    info = _lib.SolveInfo()
    st = be.ctx.lib.ds_cg_sharded(ss.handle, ss.dcode, _ptr_array([d.ptr for d in dA.blocks]), dA.blocks[0].ld,
                                  _ptr_array([d.ptr for d in db.parts]), _ptr_array([d.ptr for d in dx0.parts]),
                                  _ptr_array([d.ptr for d in dx.parts]), float(cfg.tolerance), cap, 1,
                                  hist.ctypes.data_as(c_void_p), cap + 1, ctypes.byref(info))
    if st == _lib.DS_ENOTSPD:
        raise NotSpdError(_lib.last_error(), index=None)
    _lib.check(st)
    report = SolveReport(converged=bool(info.converged), iterations=int(info.iterations),
                         final_relative_residual=float(info.final_relative_residual),
                         residual_history=hist[: info.history_len].tolist())
    report.kernel_launches = int(info.kernel_launches)
    x = dx if is_sharded(x0) else dx.to_host()
    return x, report, info


# ---------------------------------------------------------------------------
# GMRES(m) and block-cyclic LU over the backend's shards
# ---------------------------------------------------------------------------
def gmres_solve_rows(A, b, x0, cfg, be: ShardedB200Backend):
    """krylov.gmres_solve (krylov.py:75-182) with A split by rows over the backend's shards:
    ds_gmres_sharded runs the restarted Arnoldi loop in the library (the v_k slices, the
    multi-dot records of each CGS pass and the norm records all-gathered over peer memory)."""
    from .core import SingularMatrixError, SolveReport

    n = A.shape[0]
    m = int(cfg.restart_m)
    if m > 63 and be.nshards > 1:
        raise ValueError(f"restart_m = {m} exceeds the sharded GMRES limit of 63 (use the single-GPU backend)")
    dA = be._stage(A)
    ss = dA.sset
    db = b if is_sharded(b) else be.shard_vector(np.asarray(b), ss)
    dx0 = x0 if is_sharded(x0) else be.shard_vector(np.asarray(x0), ss)
    for v in (db, dx0):
        if v.sset is not ss:
            raise ValueError("sharded operands belong to different shard sets")
    dx = be.empty_vector(ss)
    cap = int(cfg.iteration_cap(n))
    hist = np.empty(cap + 2, dtype=np.float64)
    cycles = np.empty(cap + 2, dtype=np.int64)
    info = _lib.SolveInfo()
    orth = _lib.DS_ORTH_CLASSICAL if cfg.orthogonalization == "classical" else _lib.DS_ORTH_MODIFIED
    st = be.ctx.lib.ds_gmres_sharded(ss.handle, ss.dcode, _ptr_array([d.ptr for d in dA.blocks]), dA.blocks[0].ld,
                                     _ptr_array([d.ptr for d in db.parts]), _ptr_array([d.ptr for d in dx0.parts]),
                                     _ptr_array([d.ptr for d in dx.parts]), float(cfg.tolerance), cap, m, orth,
                                     hist.ctypes.data_as(c_void_p), cap + 2, cycles.ctypes.data_as(c_void_p),
                                     cap + 2, ctypes.byref(info))
    if st == _lib.DS_ESINGULAR:
        raise SingularMatrixError(_lib.last_error())
    _lib.check(st)
    report = SolveReport(converged=bool(info.converged), iterations=int(info.iterations),
                         final_relative_residual=float(info.final_relative_residual),
                         residual_history=hist[: info.history_len].tolist(),
                         breakdown="happy-breakdown" if info.breakdown == _lib.DS_BREAKDOWN_HAPPY else None,
                         restart_cycles=cycles[: info.cycles_len].tolist())
    report.kernel_launches = int(info.kernel_launches)
    x = dx if is_sharded(x0) else dx.to_host()
    return x, report, info


def lu_factor_block_cyclic_api(A, b: int, be: ShardedB200Backend):
    """direct.lu_factor_blocked (direct.py:50-84) with the columns dealt to the backend's
    shards in NB-wide blocks, round-robin: ds_lu_block_cyclic factors them in the library
    (panels broadcast over the peer-memory regions, look-ahead on the next panel's owner).
    Returns (packed F-order host factors, pivots, singular)."""
    from . import distributed as D

    A = np.asarray(A)
    n = A.shape[0]
    NB = D.outer_block(b, n)
    ss = be.shardset(n, A.dtype, kind="lu", nb=NB)
    G = be.nshards
    nblocks = -(-n // NB)
    ld = _padded_ld(n)
    blocks, cols = [], []
    for ctx, q in zip(ss.ctxs, ss.ranks):
        mine = D.local_blocks(nblocks, q, G)
        idx = np.concatenate([np.arange(k * NB, min((k + 1) * NB, n)) for k in mine]) if mine else np.zeros(0, np.int64)
        d = DeviceArray(ctx, (n, max(len(idx), 1)), A.dtype, ld=ld)
        if len(idx):
            d.upload(np.asfortranarray(A[:, idx]))
        blocks.append(d)
        cols.append(idx)
    piv, singular = lu_block_cyclic_device(be, blocks, n, b, A.dtype)
    packed = np.empty((n, n), dtype=A.dtype, order="F")
    local = [(idx, d.to_host()[:, : len(idx)]) for idx, d in zip(cols, blocks) if len(idx)]
    if be.distributed:  # every rank returns the whole factorization
        import torch.distributed as dist

        allp = [None] * G
        dist.all_gather_object(allp, local, group=be.group)
        local = [item for part in allp for item in part]
    for idx, c in local:
        packed[:, idx] = c
    return packed, piv, singular


def lu_block_cyclic_device(be: ShardedB200Backend, blocks, n: int, b: int, dtype):
    """Factor device-resident block-cyclic column blocks in place (blocks[i]: the n x cols
    DeviceArray of local shard i, NB = distributed.outer_block(b, n) wide blocks in
    increasing global order).  Returns (pivots, singular)."""
    from . import distributed as D

    NB = D.outer_block(b, n)
    ss = be.shardset(n, dtype, kind="lu", nb=NB)
    piv = np.empty(n, dtype=np.int64)
    sing = ctypes.c_int32(0)
    _lib.check(be.ctx.lib.ds_lu_block_cyclic(ss.handle, ss.dcode, _ptr_array([d.ptr for d in blocks]),
                                             blocks[0].ld, NB, max(int(b), 1), piv.ctypes.data_as(c_void_p),
                                             ctypes.byref(sing)))
    return piv, bool(sing.value)
