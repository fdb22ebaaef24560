"""Multi-GPU drivers: one process per GPU, torch.distributed.

* Row-sharded CG (config C4) and GMRES(m) (config C5): rank q owns rows
  [q*n_loc, (q+1)*n_loc) of A (an n_loc x n column-major block; n padded to
  G*n_loc with zero rows) and of every vector.  Per iteration the exchanges are
  an all-gather of the GEMV input (p or v_k) and all-gathers of 3-double
  reduction records; every rank combines the records IN RANK ORDER on the
  device, so all ranks hold bitwise-identical scalars (alpha, beta, Givens
  rotations, residual estimates) and stop on the same iteration.
* 1-D block-cyclic LU (config C5): column blocks of width NB (the internal outer
  block of the single-GPU LU) are dealt round-robin; the owner of block k
  factors its tall panel (ds_lu_panel, the reference's b-blocking), broadcasts
  the panel and its pivots, and every rank applies the swaps, the blocked TRSM
  and the K = NB DMMA trailing GEMM to the columns it owns.

The drivers are written against two small interfaces so the host logic runs
unchanged on CPU with the gloo backend in tests: ``comm`` (collectives) and
``ops`` (per-rank compute).  ``CudaShardOps`` is the product implementation:
every method is one C-ABI call into libdensolve_b200.so on device tensors.
"""

from __future__ import annotations

import math
import time
from ctypes import c_double, c_void_p

import numpy as np

from . import _lib
from .core import (DegenerateRhsError, NotSpdError, SingularMatrixError, SolveReport, SolverConfig,
                   unit_roundoff)


# ---------------------------------------------------------------------------
# partitioning
# ---------------------------------------------------------------------------
def row_partition(n: int, nranks: int) -> tuple[int, int]:
    """Equal row shards: (n_loc, N) with N = nranks * n_loc >= n (zero padding)."""
    n_loc = max(1, -(-n // nranks))
    return n_loc, n_loc * nranks


def block_owner(k: int, nranks: int) -> int:
    """Owner of column block k in the 1-D block-cyclic layout."""
    return k % nranks


def local_blocks(nblocks: int, rank: int, nranks: int) -> list[int]:
    return list(range(rank, nblocks, nranks))


def combine3_host(parts: np.ndarray) -> tuple[float, float]:
    """Rank-ordered combination of (sum x^2, scale, ssq) records, bit-identical to
    the device combine3 (ds_dist.cu): returns (sum x^2, overflow-safe norm)."""
    s2, scale, ssq = 0.0, 0.0, 0.0
    for q in range(parts.shape[0] // 3):
        s2 += float(parts[3 * q])
        bs, bq = float(parts[3 * q + 1]), float(parts[3 * q + 2])
        if scale != scale:
            continue
        if bs != bs:
            scale, ssq = bs, bq
            continue
        if math.isinf(scale) or math.isinf(bs):
            scale, ssq = math.inf, 1.0
            continue
        if bs == 0.0:
            continue
        if scale == 0.0:
            scale, ssq = bs, bq
            continue
        if scale >= bs:
            r = bs / scale
            ssq = ssq + bq * r * r
        else:
            r = scale / bs
            scale, ssq = bs, bq + ssq * r * r
    if scale == 0.0 or not (scale - scale == 0.0):
        return s2, scale
    return s2, scale * math.sqrt(ssq)


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------
class TorchComm:
    """torch.distributed collectives (NCCL on CUDA tensors, gloo on CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allgather(self, out, inp):
        self.dist.all_gather_into_tensor(out, inp.contiguous(), group=self.group)

    def broadcast(self, t, src: int):
        self.dist.broadcast(t, src, group=self.group)

    def allreduce_max(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)

    def alltoall(self, out, inp):
        self.dist.all_to_all_single(out, inp.contiguous(), group=self.group)

    def barrier(self):
        self.dist.barrier(group=self.group)


# ---------------------------------------------------------------------------
# per-rank compute on the device (product implementation)
# ---------------------------------------------------------------------------
def _p(t) -> c_void_p:
    return c_void_p(t.data_ptr())


class CudaShardOps:
    """Per-rank kernels through the C ABI.  Matrices are torch tensors holding the
    column-major data: an m x n block is a row-major tensor of shape (n, ld)."""

    def __init__(self, ctx: _lib.Context | None = None):
        self.ctx = ctx or _lib.context()
        self.lib, self.h = self.ctx.lib, self.ctx.handle

    @staticmethod
    def code(t) -> int:
        import torch
        return _lib.DS_F64 if t.dtype == torch.float64 else _lib.DS_F32

    def bind_current_stream(self):
        import torch
        s = torch.cuda.current_stream()
        if s.cuda_stream == 0:
            s = torch.cuda.Stream()
            torch.cuda.set_stream(s)
        self.ctx.set_stream(s.cuda_stream)

    def sync(self):
        self.ctx.synchronize()

    def vec_parts(self, x, out3):
        _lib.check(self.lib.ds_vec_parts(self.h, self.code(x), x.numel(), _p(x), _p(out3)))

    def resid_parts(self, A, lda, m, n, x_full, b, r, out3):
        _lib.check(self.lib.ds_resid_parts(self.h, self.code(b), m, n, _p(A), lda, _p(x_full), _p(b), _p(r),
                                           _p(out3)))

    def gemv(self, A, lda, m, n, x, y):
        _lib.check(self.lib.ds_gemv(self.h, self.code(y), m, n, _p(A), lda, _p(x), _p(y)))

    def gemv_acc(self, A, lda, m, n, x, y):
        _lib.check(self.lib.ds_gemv_acc(self.h, self.code(y), m, n, _p(A), lda, _p(x), _p(y)))

    def dot_dev(self, x, y, out1):
        _lib.check(self.lib.ds_dot_dev(self.h, self.code(x), x.numel(), _p(x), _p(y), _p(out1)))

    def cg_init(self, bparts, rparts, nranks, state, hist, tol, cap):
        _lib.check(self.lib.ds_cg_shard_init(self.h, _p(bparts), _p(rparts), nranks, _p(state), _p(hist),
                                             float(tol), int(cap)))

    def cg_update(self, nranks, pap_all, state, k, x, r, p, Ap, out3):
        _lib.check(self.lib.ds_cg_shard_update(self.h, self.code(x), x.numel(), nranks, _p(pap_all), _p(state),
                                               k, _p(x), _p(r), _p(p), _p(Ap), _p(out3)))

    def cg_finish(self, nranks, parts_all, state, k, r, p, hist, tol, cap):
        _lib.check(self.lib.ds_cg_shard_finish(self.h, self.code(r), r.numel(), nranks, _p(parts_all), _p(state),
                                               k, _p(r), _p(p), _p(hist), float(tol), int(cap)))

    def absdiff_t(self, A, lda, m, n, B, ldb):
        out = (c_double * 2)()
        _lib.check(self.lib.ds_absdiff_transposed(self.h, self.code(A), m, n, _p(A), lda, _p(B), ldb, out))
        return float(out[0]), float(out[1])

    # GMRES
    def multidot(self, V, ldv, n_loc, kc, w, out):
        _lib.check(self.lib.ds_multidot_dev(self.h, self.code(w), n_loc, _p(V), ldv, kc, _p(w), _p(out)))

    def cgs_update(self, V, ldv, n_loc, kc, w, nranks, parts_all, Hcol, hsave, ps, out3, state, k):
        _lib.check(self.lib.ds_cgs_update_shard(self.h, self.code(w), n_loc, _p(V), ldv, kc, _p(w), nranks,
                                                _p(parts_all), _p(Hcol), _p(hsave), ps, _p(out3), _p(state), k))

    def gm_start(self, r, v0, nranks, parts_all, g, state):
        _lib.check(self.lib.ds_gmres_shard_start(self.h, self.code(r), r.numel(), _p(r), _p(v0), nranks,
                                                 _p(parts_all), _p(g), _p(state)))

    def gm_step(self, w, nranks, parts_all, H, Hraw, ldh, g, cs, sn, k, est, state, tol, total_before, cap):
        _lib.check(self.lib.ds_gmres_shard_step(self.h, self.code(w), w.numel(), _p(w), nranks, _p(parts_all),
                                                _p(H), _p(Hraw), ldh, _p(g), _p(cs), _p(sn), k, _p(est),
                                                _p(state), float(tol), int(total_before), int(cap)))

    def gm_lsq(self, H, ldh, g, inner, y, state):
        _lib.check(self.lib.ds_gmres_lsq(self.h, self.code(H), _p(H), ldh, _p(g), inner, _p(y), _p(state)))

    # LU
    def lu_panel(self, P, ldp, m, w, b, piv, zero):
        _lib.check(self.lib.ds_lu_panel(self.h, self.code(P), m, w, _p(P), ldp, b, _p(piv), _p(zero)))

    def laswp(self, A, lda, ncols, k0, k1, piv):
        _lib.check(self.lib.ds_laswp(self.h, self.code(A), ncols, _p(A), lda, k0, k1, _p(piv)))

    def trsm_lower_unit(self, b, m, L, ldl, B, ldb):
        _lib.check(self.lib.ds_trsm_lower_unit(self.h, self.code(B), b, m, _p(L), ldl, _p(B), ldb, _p(B), ldb))

    def gemm_sub(self, m, n, k, A, lda, B, ldb, C, ldc):
        """C -= A B"""
        _lib.check(self.lib.ds_gemm(self.h, self.code(C), m, n, k, -1.0, _p(A), lda, _p(B), ldb, 1.0, _p(C), ldc,
                                    _p(C), ldc))


# ---------------------------------------------------------------------------
# views into column-major storage held by row-major torch tensors
# ---------------------------------------------------------------------------
def col(t2d, j):
    """Column j of a column-major matrix stored as a (cols, ld) tensor."""
    return t2d[j]


def offset_view(t2d, row0: int, col0: int):
    """Flat view starting at element (row0, col0) of a column-major (cols, ld) tensor
    (pass with the same ld)."""
    return t2d.reshape(-1)[col0 * t2d.shape[1] + row0:]


# ---------------------------------------------------------------------------
# row-sharded CG  (krylov.cg_solve, krylov.py:36-72)
# ---------------------------------------------------------------------------
def _symmetry_gate(A_blk, n, n_loc, comm, ops, dtype):
    """max|A - A^T| <= 10 u max|A| over the row-sharded matrix (krylov.py:41-44):
    rank q sends its block A[rows q, cols r] to rank r (all-to-all) and compares
    it against the transpose of its own A[rows r, cols q]."""
    import torch

    G = comm.size
    N = G * n_loc
    # send buffer: for each destination r, our block rows(q) x cols(r), column-major.  The
    # row block is stored as a torch (n, n_loc) tensor (column-major n_loc x n, ld n_loc);
    # when n == N (n divisible by G) its G column groups are already contiguous blocks: a
    # view, no copy of the local matrix.  Otherwise (or for any other shape) the blocks are
    # copied into a zeroed buffer, so padding never enters the comparison.
    if A_blk.is_contiguous() and tuple(A_blk.shape) == (n, n_loc) and n == N:
        send = A_blk.view(G, n_loc, n_loc)
    else:
        send = torch.zeros((G, n_loc, n_loc), dtype=A_blk.dtype, device=A_blk.device)
        for r in range(G):
            c0, c1 = r * n_loc, min(n, (r + 1) * n_loc)
            if c1 > c0:
                send[r, : c1 - c0, :] = A_blk[c0:c1, :]
    if G == 1:
        recv = send
    else:
        recv = torch.empty_like(send)
        comm.alltoall(recv.reshape(-1), send.reshape(-1))
    md, am = 0.0, 0.0
    for r in range(G):
        c0, c1 = r * n_loc, min(n, (r + 1) * n_loc)
        if c1 <= c0:
            continue
        mine = send[r]          # A[rows q, cols r]  (n_loc x n_loc column-major, ld n_loc)
        theirs = recv[r]        # A[rows r, cols q]
        d, a = ops.absdiff_t(mine, n_loc, n_loc, n_loc, theirs, n_loc)
        md, am = max(md, d) if d == d else d, max(am, a) if a == a else a
    t = torch.tensor([md, am], dtype=torch.float64, device=A_blk.device)
    comm.allreduce_max(t)
    md, am = float(t[0]), float(t[1])
    u = unit_roundoff(dtype)
    if md > 10.0 * u * am:
        raise NotSpdError("matrix is not symmetric")
    del N


def cg_solve_sharded(A_blk, b_loc, x0_loc, n: int, cfg: SolverConfig, comm, ops, check_sym: bool = True):
    """CG on a row-sharded system.  A_blk: (n, n_loc) tensor = column-major
    n_loc x n row block (zero rows past n); b_loc, x0_loc: (n_loc,) shards.
    Returns (x_loc, SolveReport) with the replicated history."""
    import torch

    t0 = time.perf_counter()
    G = comm.size
    n_loc = b_loc.numel()
    N = G * n_loc
    dev, dt = b_loc.device, b_loc.dtype
    np_dt = np.float64 if dt == torch.float64 else np.float32
    if check_sym:
        _symmetry_gate(A_blk, n, n_loc, comm, ops, np_dt)
    cap = int(cfg.iteration_cap(n))
    f64 = dict(dtype=torch.float64, device=dev)
    state = torch.zeros(_STATE, **f64)
    hist = torch.zeros(cap + 2, **f64)
    parts = torch.zeros(3, **f64)
    bparts = torch.zeros(3 * G, **f64)
    rparts = torch.zeros(3 * G, **f64)
    pap = torch.zeros(1, **f64)
    pap_all = torch.zeros(G, **f64)
    x = x0_loc.clone()
    r = torch.empty_like(b_loc)
    Ap = torch.empty_like(b_loc)
    full = torch.empty(N, dtype=dt, device=dev)

    ops.vec_parts(b_loc, parts)
    comm.allgather(bparts, parts)
    comm.allgather(full, x)
    ops.resid_parts(A_blk, n_loc, n_loc, n, full, b_loc, r, parts)
    comm.allgather(rparts, parts)
    ops.cg_init(bparts, rparts, G, state, hist, cfg.tolerance, cap)
    st = state.cpu().numpy()
    if st[1] == 0.0:
        raise DegenerateRhsError("||b|| = 0")
    p = r.clone()
    k, chunk = 0, 2
    while True:
        st = state.cpu().numpy()
        if st[3] <= k or k >= cap or st[2] != 0:
            break
        kend = min(cap, k + chunk)
        while k < kend:
            comm.allgather(full, p)
            ops.gemv(A_blk, n_loc, n_loc, n, full, Ap)
            ops.dot_dev(p, Ap, pap)
            comm.allgather(pap_all, pap)
            ops.cg_update(G, pap_all, state, k, x, r, p, Ap, parts)
            comm.allgather(rparts, parts)
            ops.cg_finish(G, rparts, state, k, r, p, hist, cfg.tolerance, cap)
            k += 1
        chunk = min(2 * chunk, 64)
    st = state.cpu().numpy()
    if st[2] == _lib.DS_ENOTSPD:
        raise NotSpdError(f"p'Ap = {st[4]} <= 0: matrix is not positive definite")
    iters = int(min(st[3], cap))
    h = hist[: iters + 1].cpu().numpy().tolist()
    rep = SolveReport(converged=bool(h[-1] <= cfg.tolerance), iterations=iters, final_relative_residual=h[-1],
                      residual_history=h, wall_time=time.perf_counter() - t0)
    return x, rep


_STATE = 16  # the shard kernels keep an int64 mirror of the stop word at slot 8


# ---------------------------------------------------------------------------
# row-sharded GMRES(m)  (krylov.gmres_solve, krylov.py:75-182)
# ---------------------------------------------------------------------------
def gmres_solve_sharded(A_blk, b_loc, x0_loc, n: int, cfg: SolverConfig, comm, ops):
    import torch

    t0 = time.perf_counter()
    G = comm.size
    n_loc = b_loc.numel()
    N = G * n_loc
    dev, dt = b_loc.device, b_loc.dtype
    np_dt = np.float64 if dt == torch.float64 else np.float32
    u = unit_roundoff(np_dt)
    m = int(cfg.restart_m)
    if m > 62:
        raise ValueError(f"restart_m = {m} exceeds the device limit of 62")
    cap = int(cfg.iteration_cap(n))
    f64 = dict(dtype=torch.float64, device=dev)
    tdt = dict(dtype=dt, device=dev)
    state = torch.zeros(_STATE, **f64)
    parts = torch.zeros(3, **f64)
    parts_all = torch.zeros(3 * G, **f64)
    mparts = torch.zeros(64, **f64)
    mparts_all = torch.zeros(64 * G, **f64)
    hsave = torch.zeros(64, **f64)
    est = torch.zeros(64, **f64)
    V = torch.zeros((m + 1, n_loc), **tdt)           # column-major n_loc x (m+1)
    H = torch.zeros((m, m + 1), **tdt)               # column-major (m+1) x m
    Hraw = torch.zeros((m, m + 1), **tdt)
    g = torch.zeros(m + 2, **tdt)
    cs = torch.zeros(m + 2, **tdt)
    sn = torch.zeros(m + 2, **tdt)
    y = torch.zeros(64, **tdt)
    x = x0_loc.clone()
    r = torch.empty_like(b_loc)
    full = torch.empty(N, **tdt)
    orth_passes = 1 if cfg.orthogonalization == "classical" else 2

    ops.vec_parts(b_loc, parts)
    comm.allgather(parts_all, parts)
    s2b, bnorm = combine3_host(parts_all.cpu().numpy())
    bnorm_plain = math.sqrt(s2b)
    if bnorm == 0.0:
        raise DegenerateRhsError("||b|| = 0")
    state[1] = bnorm

    history: list[float] = []
    cycles: list[int] = []
    total = 0
    breakdown = None
    converged = False
    while True:
        comm.allgather(full, x)
        ops.resid_parts(A_blk, n_loc, n_loc, n, full, b_loc, r, parts)
        comm.allgather(parts_all, parts)
        _, beta = combine3_host(parts_all.cpu().numpy())
        relres = beta / bnorm
        if total == 0:
            history.append(relres)
        if relres <= cfg.tolerance:
            converged = True
            break
        if total >= cap:
            break
        cycles.append(total)
        start_res = relres
        V.zero_()
        H.zero_()
        Hraw.zero_()
        g.zero_()
        cs.zero_()
        sn.zero_()
        state[2] = 0.0
        state[3] = float(m)
        state[4] = 0.0
        ops.gm_start(r, V[0], G, parts_all, g, state)
        k, chunk = 0, 4
        while True:
            if k > 0:
                stop = float(state[3].item())
                if stop <= k or k >= m:
                    break
            kend = min(m, k + chunk)
            while k < kend:
                comm.allgather(full, V[k])
                w = V[k + 1]
                ops.gemv(A_blk, n_loc, n_loc, n, full, w)
                kc = k + 1
                for ps in range(orth_passes):
                    ops.multidot(V, n_loc, n_loc, kc, w, mparts)
                    # rank-major (G x kc) records of the partial dots
                    comm.allgather(mparts_all[: G * kc], mparts[:kc])
                    ops.cgs_update(V, n_loc, n_loc, kc, w, G, mparts_all[: G * kc], H[k], hsave, ps, parts,
                                   state, k)
                comm.allgather(parts_all, parts)
                ops.gm_step(w, G, parts_all, H, Hraw, m + 1, g, cs, sn, k, est, state, cfg.tolerance, total, cap)
                k += 1
            chunk = min(2 * chunk, 32)
        st = state.cpu().numpy()
        inner = int(min(st[3], m))
        happy = st[4] != 0.0
        history.extend(est[:inner].cpu().numpy().tolist())
        total += inner
        ops.gm_lsq(H, m + 1, g, inner, y, state)
        st = state.cpu().numpy()
        if st[2] == _lib.DS_ESINGULAR:
            raise SingularMatrixError(f"zero diagonal at row {int(st[5])}")
        ops.gemv_acc(V, n_loc, n_loc, inner, y, x)
        comm.allgather(full, x)
        ops.resid_parts(A_blk, n_loc, n_loc, n, full, b_loc, r, parts)
        comm.allgather(parts_all, parts)
        s2r, _ = combine3_host(parts_all.cpu().numpy())
        true_res = math.sqrt(s2r) / bnorm_plain
        if happy or history[-1] <= cfg.tolerance or true_res <= cfg.tolerance:
            history[-1] = true_res
            if true_res <= cfg.tolerance or happy:
                converged = True
                breakdown = "happy-breakdown" if happy else None
                break
        if total >= cap:
            history[-1] = true_res
            break
        if inner == m and true_res >= start_res * (1.0 - u):
            history[-1] = true_res
            break
    rep = SolveReport(converged=converged, iterations=total, final_relative_residual=history[-1],
                      residual_history=history, breakdown=breakdown, restart_cycles=cycles,
                      wall_time=time.perf_counter() - t0)
    return x, rep


# ---------------------------------------------------------------------------
# 1-D block-cyclic LU  (direct.lu_factor_blocked, direct.py:50-84)
# ---------------------------------------------------------------------------
def outer_block(b: int, n: int) -> int:
    """Column-block width of the 1-D block-cyclic layout: 256 (b * floor(256/b)); narrower
    than the single-GPU outer block (512) so 8 ranks still own 16 blocks each at n=32768."""
    if b >= 256 or b >= n:
        return min(b, n)
    return min(n, b * max(1, 256 // b))


def lu_factor_block_cyclic(W_loc, n: int, b: int, comm, ops, nb_outer: int | None = None):
    """Factor the block-cyclic matrix in place.  W_loc: (n_loc_cols, n) tensor =
    column-major n x n_loc_cols holding this rank's column blocks (block k at
    local position (k // G) * NB).  Returns (pivots int64 tensor (n,), singular).

    Look-ahead: after receiving panel k, the owner of block k+1 first applies the
    swaps and the update of step k to that block and factors it, and only then
    updates its other blocks -- so panel k+1 is ready (and broadcast) while the
    other ranks are still running their step-k trailing GEMMs."""
    import torch

    G, q = comm.size, comm.rank
    NB = nb_outer or outer_block(b, n)
    nblocks = -(-n // NB)
    dev = W_loc.device
    piv = torch.zeros(n, dtype=torch.int64, device=dev)
    zero = torch.zeros(n, dtype=torch.int8, device=dev)
    mine = local_blocks(nblocks, q, G)
    lcol = {k: i * NB for i, k in enumerate(mine)}   # local column offset of block k

    def factor_own(k):
        """Owner of block k: factor its (already updated) panel; return (panel, pv, zf)."""
        kb, bf = k * NB, min((k + 1) * NB, n)
        w = bf - kb
        c0 = lcol[k]
        pv = torch.empty(w, dtype=torch.int64, device=dev)
        zf = torch.zeros(w, dtype=torch.int8, device=dev)
        ops.lu_panel(offset_view(W_loc, kb, c0), n, n - kb, w, b, pv, zf)  # pivots relative to row kb
        pv += kb
        panel = W_loc[c0:c0 + w, kb:].clone()  # column-major (n-kb) x w
        return panel, pv, zf

    def update_blocks(k, L00, blocks_):
        """TRSM of the U block row + trailing GEMM of step k on the given local blocks
        (contiguous ascending run)."""
        if not blocks_:
            return
        kb, bf = k * NB, min((k + 1) * NB, n)
        w = bf - kb
        c0 = lcol[blocks_[0]]
        cw = sum(min(NB, n - kk * NB) for kk in blocks_)
        for ib in range(0, w, b):
            ibf = min(ib + b, w)
            ops.trsm_lower_unit(ibf - ib, cw, offset_view(L00, ib, ib), n - kb, offset_view(W_loc, kb + ib, c0), n)
            if ibf < w:
                ops.gemm_sub(w - ibf, cw, ibf - ib, offset_view(L00, ibf, ib), n - kb,
                             offset_view(W_loc, kb + ib, c0), n, offset_view(W_loc, kb + ibf, c0), n)
        if bf < n:
            ops.gemm_sub(n - bf, cw, w, offset_view(L00, w, 0), n - kb, offset_view(W_loc, kb, c0), n,
                         offset_view(W_loc, bf, c0), n)

    ready = factor_own(0) if block_owner(0, G) == q else None
    for k in range(nblocks):
        kb, bf = k * NB, min((k + 1) * NB, n)
        w = bf - kb
        owner = block_owner(k, G)
        if q == owner:
            panel, pv, zf = ready
        else:
            panel = torch.empty((w, n - kb), dtype=W_loc.dtype, device=dev)
            pv = torch.empty(w, dtype=torch.int64, device=dev)
            zf = torch.zeros(w, dtype=torch.int8, device=dev)
        comm.broadcast(panel, owner)
        comm.broadcast(pv, owner)
        comm.broadcast(zf, owner)
        piv[kb:bf] = pv
        zero[kb:bf] = zf
        # swaps on every local column outside block k (the owner's block k is done)
        for kk in mine:
            if kk == k:
                continue
            ops.laswp(offset_view(W_loc, 0, lcol[kk]), n, min(NB, n - kk * NB), kb, bf, piv)
        right = [kk for kk in mine if kk > k]
        if k + 1 < nblocks and block_owner(k + 1, G) == q:
            update_blocks(k, panel, [k + 1])  # look-ahead block first
            ready = factor_own(k + 1)
            right = [kk for kk in right if kk != k + 1]
        update_blocks(k, panel, right)
    return piv, bool(zero.any().item())


def scatter_block_cyclic(A: np.ndarray, n: int, b: int, rank: int, nranks: int, torch, device, dtype,
                         nb_outer: int | None = None):
    """This rank's column blocks of a host F-order matrix, as a (cols, n) tensor."""
    NB = nb_outer or outer_block(b, n)
    blocks = local_blocks(-(-n // NB), rank, nranks)
    cols = [np.arange(k * NB, min((k + 1) * NB, n)) for k in blocks]
    idx = np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)
    host = np.ascontiguousarray(np.asarray(A)[:, idx].T)  # (cols, n) = column-major block
    return torch.from_numpy(host).to(device=device, dtype=dtype), idx


def gather_block_cyclic(W_loc, idx, n: int, comm):
    """All-gather the distributed packed factors into a full F-order host array."""
    import torch

    G = comm.size
    counts = torch.tensor([W_loc.shape[0]], dtype=torch.int64, device=W_loc.device)
    all_counts = torch.zeros(G, dtype=torch.int64, device=W_loc.device)
    comm.allgather(all_counts, counts)
    mx = int(all_counts.max().item())
    pad = torch.zeros((mx, n), dtype=W_loc.dtype, device=W_loc.device)
    pad[: W_loc.shape[0]] = W_loc
    out = torch.empty((G * mx, n), dtype=W_loc.dtype, device=W_loc.device)
    comm.allgather(out.reshape(-1), pad.reshape(-1))
    ipad = torch.full((mx,), -1, dtype=torch.int64, device=W_loc.device)
    ipad[: len(idx)] = torch.as_tensor(idx, dtype=torch.int64, device=W_loc.device)
    iall = torch.empty(G * mx, dtype=torch.int64, device=W_loc.device)
    comm.allgather(iall, ipad)
    full = np.empty((n, n), order="F", dtype=out.cpu().numpy().dtype)
    o, ii = out.cpu().numpy(), iall.cpu().numpy()
    for j in range(G * mx):
        if ii[j] >= 0:
            full[:, ii[j]] = o[j]
    return full


# ---------------------------------------------------------------------------
# benchmark entry (C4 on N GPUs)
# ---------------------------------------------------------------------------
def spd_block_device(n: int, r0: int, r1: int, torch, device, seed: int = 0):
    """Rows [r0, r1) of the synthetic symmetric matrix A = S + 1.5 sqrt(n) I, S[i,j] =
    u(min(i,j), max(i,j)) with u a counter-based hash in [-1, 1) (symmetric by
    construction, generated independently on every rank).  S has a semicircle
    spectrum of radius 2 sqrt(n/3) = 1.15 sqrt(n), so A is SPD with kappa ~ 7.6.  Returned as a
    column-major (n, r1-r0) tensor (= A[r0:r1, :]^T row-major)."""
    rows = torch.arange(r0, r1, device=device, dtype=torch.int64)
    out = torch.empty((n, r1 - r0), dtype=torch.float64, device=device)
    cols_chunk = 4096
    mask = (1 << 62) - 1
    for c0 in range(0, n, cols_chunk):
        cols = torch.arange(c0, min(n, c0 + cols_chunk), device=device, dtype=torch.int64)
        i = torch.minimum(rows[None, :], cols[:, None])
        j = torch.maximum(rows[None, :], cols[:, None])
        h = (i * n + j + seed * 0x9E3779B97F4A7C15) & mask
        h = (h ^ (h >> 31)) * 0x5851F42D4C957F2D & mask
        h = (h ^ (h >> 29)) * 0x2545F4914F6CDD1D & mask
        h = h ^ (h >> 32)
        v = (h & ((1 << 52) - 1)).to(torch.float64) * (2.0 / float(1 << 52)) - 1.0
        v = torch.where(i == j, v + 1.5 * math.sqrt(n), v)
        out[c0:c0 + cols.numel()] = v
    return out
