"""CPU ORACLE — test infrastructure only, never the product path.

A NumPy restatement of the reference algorithms on the B200 hot path
(/root/reference/pkg/src/densolve, cited file:line per function).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference/CPU
baseline leg may import this module, and only as the checker / the timed CPU
baseline.  The shipped package (paper_1511_07207_b200) never imports it.

Parity pinning: tests/test_oracle_golden.py checks this restatement against
golden vectors produced by running the reference itself in the build
container (tests/golden/make_golden.py -> tests/golden/golden.npz): iteration
counts, residual histories, pivots, packed factors and generator outputs.

The arithmetic lives in NumPy (reference pyproject.toml:10 pins only
``numpy>=1.24``; the container has numpy 2.3.5 / OpenBLAS 0.3.30).  Every
elementwise update below is written with the same NumPy expression as the
reference so rounding is identical; BLAS reductions (dot/gemv/gemm) are the
same library calls.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

PROBLEM_KINDS = ("identity", "diag_dominant", "spd", "general_nonsymmetric", "from_file")


class OracleError(Exception):
    pass


class NotSpd(OracleError):
    pass


class Singular(OracleError):
    pass


class Degenerate(OracleError):
    pass


def unit_roundoff(dtype) -> float:
    """core.py:45-47"""
    return float(np.finfo(np.dtype(dtype)).eps) / 2.0


# ---------------------------------------------------------------------------
# generators (harness.py:73-123)
# ---------------------------------------------------------------------------
def generate_problem(kind: str, n: int, seed: int = 0, precision: str = "f64"):
    """harness.py:77-105 — seeded (A, b, x_true)."""
    rng = np.random.default_rng([seed, n, PROBLEM_KINDS.index(kind)])
    if kind == "identity":
        A = np.eye(n)
    elif kind == "diag_dominant":
        A = rng.uniform(-1.0, 1.0, size=(n, n))
        np.fill_diagonal(A, 0.0)
        np.fill_diagonal(A, 4.0 * np.sum(np.abs(A), axis=1))
    elif kind == "spd":
        M = rng.uniform(-1.0, 1.0, size=(n, n))
        A = M.T @ M + n * np.eye(n)
        A = np.tril(A) + np.tril(A, -1).T
    elif kind == "general_nonsymmetric":
        E = rng.uniform(-1.0, 1.0, size=(n, n))
        np.fill_diagonal(E, 0.0)
        R = rng.uniform(-1.0, 1.0, size=(n, n))
        A = E + 0.5 * (R - R.T)
        np.fill_diagonal(A, 0.0)
        np.fill_diagonal(A, 4.0 * np.sum(np.abs(A), axis=1))
    else:
        raise ValueError(kind)
    x_true = rng.uniform(-1.0, 1.0, size=n)
    dt = np.float32 if precision == "f32" else np.float64
    A = np.asfortranarray(A, dtype=dt)
    x_true = x_true.astype(dt)
    return A, A @ x_true, x_true


def generate_well_separated(n: int, seed: int = 0, dtype=np.float64):
    """harness.py:114-123"""
    rng = np.random.default_rng([seed, n, 97])
    A = np.empty((n, n), order="F")
    for j in range(n):
        mags = 1.002 ** rng.permutation(n)
        signs = rng.choice([-1.0, 1.0], size=n)
        A[:, j] = signs * mags
    return np.asfortranarray(A, dtype=dtype)


# ---------------------------------------------------------------------------
# the op contract (backends.py:104-252) — Blocked flavour (threads = all cores)
# ---------------------------------------------------------------------------
class Ops:
    def __init__(self, tile: int = 64, threads: int | None = None):
        self.tile = tile
        self.threads = threads if threads is not None else (os.cpu_count() or 1)

    @staticmethod
    def axpy(alpha, x, y):  # backends.py:104-107
        return y + alpha * x

    @staticmethod
    def dot(x, y):  # backends.py:109-112
        return float(np.dot(x, y))

    @staticmethod
    def nrm2(x):  # backends.py:114-122 (scaled two-pass form)
        if x.shape[0] == 0:
            return 0.0
        m = float(np.max(np.abs(x)))
        if m == 0.0 or not np.isfinite(m):
            return m
        return m * float(np.sqrt(np.dot(x / m, x / m)))

    @staticmethod
    def scal(alpha, x):  # backends.py:124-126
        return alpha * x

    @staticmethod
    def iamax(x):  # backends.py:128-132
        return int(np.argmax(np.abs(x)))

    @staticmethod
    def gemv(A, x):  # backends.py:136-142
        return A @ x

    @staticmethod
    def ger_inplace(out, alpha, x, y):  # backends.py:152-155 (out aliases A)
        out += alpha * np.outer(x, y)
        return out

    def gemm_inplace(self, alpha, A, B, beta, C):
        """backends.py:234-252: 64x64 output tiles, thread pool above 2**24 flops."""
        m, k = A.shape
        n = B.shape[1]
        t = self.tile
        tiles = [(i, min(i + t, m), j, min(j + t, n)) for j in range(0, n, t) for i in range(0, m, t)]

        def run(tile):
            i0, i1, j0, j1 = tile
            C[i0:i1, j0:j1] = beta * C[i0:i1, j0:j1] + alpha * np.dot(A[i0:i1, :], B[:, j0:j1])

        if self.threads > 1 and len(tiles) > 1 and 2 * m * n * k >= (1 << 24):
            with ThreadPoolExecutor(max_workers=self.threads) as pool:
                list(pool.map(run, tiles))
        else:
            for tl in tiles:
                run(tl)
        return C

    @staticmethod
    def trsm_lower_unit(L, B):  # backends.py:176-186
        b = L.shape[0]
        Z = np.array(B, order="F", copy=True)
        for i in range(1, b):
            Z[i, :] -= L[i, :i] @ Z[:i, :]
        return Z


# ---------------------------------------------------------------------------
# CG (krylov.py:36-72)
# ---------------------------------------------------------------------------
def cg(A, b, x0, tol: float, max_it: int | None = None, ops: Ops | None = None):
    ops = ops or Ops()
    n = A.shape[0]
    cap = max_it if max_it is not None else 10 * n
    u = unit_roundoff(A.dtype)
    amax = float(np.max(np.abs(A)))
    if float(np.max(np.abs(A - A.T))) > 10.0 * u * amax:  # krylov.py:41-44
        raise NotSpd("matrix is not symmetric")
    bnorm = ops.nrm2(b)
    if bnorm == 0.0:
        raise Degenerate("||b|| = 0")
    x = x0.copy()
    r = ops.axpy(-1.0, ops.gemv(A, x), b)
    res = ops.nrm2(r) / bnorm
    hist = [res]
    p = r.copy()
    rs = ops.dot(r, r)
    it = 0
    while res > tol and it < cap:  # krylov.py:54-67
        Ap = ops.gemv(A, p)
        pAp = ops.dot(p, Ap)
        if pAp <= 0.0:
            raise NotSpd(f"p'Ap = {pAp}")
        alpha = rs / pAp
        x = ops.axpy(alpha, p, x)
        r = ops.axpy(-alpha, Ap, r)
        rs_new = ops.dot(r, r)
        p = ops.axpy(rs_new / rs, p, r)
        rs = rs_new
        res = ops.nrm2(r) / bnorm
        hist.append(res)
        it += 1
    return x, {"converged": res <= tol, "iterations": it, "final": float(res), "history": hist}


# ---------------------------------------------------------------------------
# substitution (direct.py:123-152)
# ---------------------------------------------------------------------------
def forward_substitution(L, b, unit_diagonal=False):
    n = L.shape[0]
    y = b.copy()
    for i in range(n):
        y[i] -= L[i, :i] @ y[:i]
        if not unit_diagonal:
            if L[i, i] == 0.0:
                raise Singular(f"zero diagonal at row {i}")
            y[i] /= L[i, i]
    return y


def backward_substitution(U, y):
    n = U.shape[0]
    x = y.copy()
    for i in range(n - 1, -1, -1):
        if i + 1 < n:
            x[i] -= U[i, i + 1:] @ x[i + 1:]
        if U[i, i] == 0.0:
            raise Singular(f"zero diagonal at row {i}")
        x[i] /= U[i, i]
    return x


def relative_residual(A, x, b):
    """core.py:204-210"""
    bn = np.linalg.norm(b)
    if bn == 0.0:
        raise Degenerate("||b|| = 0")
    return float(np.linalg.norm(b - A @ x) / bn)


# ---------------------------------------------------------------------------
# GMRES(m) (krylov.py:75-182); orth "modified" = MGS, "classical" = CGS
# ---------------------------------------------------------------------------
def gmres(A, b, x0, tol: float, restart_m: int = 35, max_it: int | None = None,
          orth: str = "modified", ops: Ops | None = None, sink: list | None = None):
    ops = ops or Ops()
    n = A.shape[0]
    m = restart_m
    u = unit_roundoff(A.dtype)
    bnorm = ops.nrm2(b)
    if bnorm == 0.0:
        raise Degenerate("||b|| = 0")
    x = x0.copy()
    cap = max_it if max_it is not None else 10 * n
    total = 0
    hist: list = []
    cycles: list = []

    def done(conv, bd=None):
        return x, {"converged": conv, "iterations": total, "final": hist[-1], "history": hist,
                   "cycles": cycles, "breakdown": bd}

    while True:
        r = ops.axpy(-1.0, ops.gemv(A, x), b)
        beta = ops.nrm2(r)
        relres = beta / bnorm
        if total == 0:
            hist.append(relres)
        if relres <= tol:
            return done(True)
        if total >= cap:
            return done(False)
        cycles.append(total)
        start_res = relres
        V = np.zeros((n, m + 1), dtype=A.dtype, order="F")
        H = np.zeros((m + 1, m), dtype=A.dtype, order="F")
        Hraw = np.zeros((m + 1, m), dtype=A.dtype, order="F")
        g = np.zeros(m + 1, dtype=A.dtype)
        cs = np.zeros(m, dtype=A.dtype)
        sn = np.zeros(m, dtype=A.dtype)
        g[0] = beta
        V[:, 0] = ops.scal(1.0 / beta, r)
        inner = 0
        happy = False
        for k in range(m):
            w = ops.gemv(A, V[:, k])
            if orth == "modified":
                for j in range(k + 1):
                    h = ops.dot(V[:, j], w)
                    w = ops.axpy(-h, V[:, j], w)
                    H[j, k] = h
            else:
                coeffs = [ops.dot(V[:, j], w) for j in range(k + 1)]
                for j, h in enumerate(coeffs):
                    w = ops.axpy(-h, V[:, j], w)
                    H[j, k] = h
            hk1 = ops.nrm2(w)
            H[k + 1, k] = hk1
            Hraw[:, k] = H[:, k]
            happy = hk1 == 0.0
            if not happy:
                V[:, k + 1] = ops.scal(1.0 / hk1, w)
            for j in range(k):  # krylov.py:147-150
                t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
                H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
                H[j, k] = t
            denom = np.hypot(H[k, k], H[k + 1, k])
            cs[k], sn[k] = H[k, k] / denom, H[k + 1, k] / denom
            H[k, k] = denom
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            total += 1
            inner = k + 1
            est = abs(float(g[k + 1])) / bnorm
            hist.append(est)
            if happy or est <= tol or total >= cap:
                break
        y = backward_substitution(np.asfortranarray(H[:inner, :inner]), g[:inner].copy())
        x = ops.axpy(1.0, ops.gemv(V[:, :inner], y), x)
        if sink is not None:
            sink.append({"V": V, "H": Hraw, "inner": inner, "beta": beta})
        true_res = relative_residual(A, x, b)
        if happy or hist[-1] <= tol or true_res <= tol:
            hist[-1] = true_res
            if true_res <= tol or happy:
                return done(True, "happy-breakdown" if happy else None)
        if total >= cap:
            hist[-1] = true_res
            return done(False)
        if inner == m and true_res >= start_res * (1.0 - u):
            hist[-1] = true_res
            return done(False)


# ---------------------------------------------------------------------------
# LU (direct.py:25-84, 155-163) and pivots (core.py:94-100)
# ---------------------------------------------------------------------------
def lu_factor_blocked(A, b: int, ops: Ops | None = None):
    """direct.py:50-84 — returns (packed, pivots, singular)."""
    ops = ops or Ops()
    n = A.shape[0]
    b = min(b, n)
    W = np.array(A, order="F", copy=True)
    piv = np.empty(n, dtype=np.intp)
    singular = False
    for kb in range(0, n, b):
        bf = min(kb + b, n)
        for i in range(kb, bf):
            v = i + ops.iamax(W[i:, i])
            piv[i] = v
            if v != i:
                W[[i, v], :] = W[[v, i], :]
            aii = W[i, i]
            if aii == 0.0:
                singular = True
                continue
            if i + 1 < n:
                W[i + 1:, i] = ops.scal(1.0 / aii, W[i + 1:, i])
                if i + 1 < bf:
                    ops.ger_inplace(W[i + 1:, i + 1:bf], -1.0, W[i + 1:, i], W[i, i + 1:bf])
        if bf < n:
            W[kb:bf, bf:] = ops.trsm_lower_unit(W[kb:bf, kb:bf], W[kb:bf, bf:])
            ops.gemm_inplace(-1.0, W[bf:, kb:bf], W[kb:bf, bf:], 1.0, W[bf:, bf:])
    return W, piv, singular


def lu_factor_unblocked(A, ops: Ops | None = None):
    """direct.py:25-47"""
    ops = ops or Ops()
    n = A.shape[0]
    W = np.array(A, order="F", copy=True)
    piv = np.empty(n, dtype=np.intp)
    singular = False
    for k in range(n):
        v = k + ops.iamax(W[k:, k])
        piv[k] = v
        if v != k:
            W[[k, v], :] = W[[v, k], :]
        akk = W[k, k]
        if akk == 0.0:
            singular = True
            continue
        if k + 1 < n:
            W[k + 1:, k] = ops.scal(1.0 / akk, W[k + 1:, k])
            ops.ger_inplace(W[k + 1:, k + 1:], -1.0, W[k + 1:, k], W[k, k + 1:])
    return W, piv, singular


def apply_pivots(pivots, v):
    """core.py:94-100"""
    out = v.copy()
    for k, p in enumerate(pivots):
        if p != k:
            out[[k, p]] = out[[p, k]]
    return out


def lu_solve(packed, pivots, b):
    """direct.py:155-163 (singular check left to the caller)."""
    pb = apply_pivots(pivots, b)
    y = forward_substitution(packed, pb, unit_diagonal=True)
    return backward_substitution(packed, y)


def permutation_matrix(pivots, n, dtype=np.float64):
    """core.py:113-116"""
    return np.asfortranarray(apply_pivots(pivots, np.eye(n, dtype=dtype, order="F")))


def lu_backward_error(A, packed, pivots):
    """||PA - LU||_F (test_direct.py:24-27)."""
    n = A.shape[0]
    P = permutation_matrix(pivots, n)
    L = np.tril(packed, -1).astype(np.float64)
    np.fill_diagonal(L, 1.0)
    U = np.triu(packed).astype(np.float64)
    return float(np.linalg.norm(P @ A.astype(np.float64) - L @ U))


# ---------------------------------------------------------------------------
# BiCGSTAB (krylov.py:185-253)
# ---------------------------------------------------------------------------
def bicgstab(A, b, x0, tol: float, max_it: int | None = None, ops: Ops | None = None):
    ops = ops or Ops()
    n = A.shape[0]
    cap = max_it if max_it is not None else 10 * n
    u = unit_roundoff(A.dtype)
    bnorm = ops.nrm2(b)  # _rhs_norm (krylov.py:29-33)
    if bnorm == 0.0:
        raise Degenerate("||b|| = 0")
    x = x0.copy()
    r = ops.axpy(-1.0, ops.gemv(A, x), b)
    r0hat = r.copy()
    r0hat_norm = float(np.linalg.norm(r0hat))
    rho_prev, alpha, omega = 1.0, 1.0, 1.0
    rho = ops.dot(r0hat, r)
    p = np.zeros_like(b)
    v = np.zeros_like(b)
    res = ops.nrm2(r) / bnorm
    hist = [res]
    rnorm = res * bnorm
    it = 0
    breakdown = None
    while res > tol and it < cap:  # krylov.py:212-245
        if abs(rho) < u * r0hat_norm * rnorm:
            breakdown = "rho-breakdown"
            break
        beta = (rho / rho_prev) * (alpha / omega)
        p = ops.axpy(beta, ops.axpy(-omega, v, p), r)
        v = ops.gemv(A, p)
        rv = ops.dot(r0hat, v)
        if rv == 0.0:
            breakdown = "rho-breakdown"
            break
        alpha = rho / rv
        s = ops.axpy(-alpha, v, r)
        snorm = ops.nrm2(s)
        if snorm / bnorm <= tol:
            x = ops.axpy(alpha, p, x)
            r = s
            res = snorm / bnorm
            hist.append(res)
            it += 1
            break
        t = ops.gemv(A, s)
        ts = ops.dot(t, s)
        tt = ops.dot(t, t)
        if tt == 0.0:
            breakdown = "omega-breakdown"
            break
        omega = ts / tt
        if abs(omega) < u:
            breakdown = "omega-breakdown"
            break
        x = ops.axpy(omega, s, ops.axpy(alpha, p, x))
        r = ops.axpy(-omega, t, s)
        rho_prev, rho = rho, ops.dot(r0hat, r)
        rnorm = ops.nrm2(r)
        res = rnorm / bnorm
        hist.append(res)
        it += 1
    return x, {"converged": res <= tol and breakdown is None, "iterations": it, "final": float(res),
               "history": hist, "breakdown": breakdown}


# ---------------------------------------------------------------------------
# Cholesky (direct.py:87-120, 166-171)
# ---------------------------------------------------------------------------
def cholesky_factor(A, b: int, ops: Ops | None = None):
    """Returns tril(W) (CholeskyFactor.l); raises NotSpd with .index on a bad pivot."""
    ops = ops or Ops()
    n = A.shape[0]
    b = min(b, n)
    u = unit_roundoff(A.dtype)
    amax = float(np.max(np.abs(A))) if n else 0.0
    if float(np.max(np.abs(A - A.T))) > 10.0 * u * amax:
        raise NotSpd("matrix is not symmetric")
    W = np.array(A, order="F", copy=True)
    for kb in range(0, n, b):
        bf = min(kb + b, n)
        for i in range(kb, bf):
            aii = W[i, i]
            if not (aii > 0.0) or not np.isfinite(aii):
                e = NotSpd(f"nonpositive pivot {aii} at index {i}")
                e.index = i
                raise e
            W[i, i] = np.sqrt(aii)
            if i + 1 < n:
                W[i + 1:, i] = ops.scal(1.0 / W[i, i], W[i + 1:, i])
                if i + 1 < bf:
                    ops.ger_inplace(W[i + 1:, i + 1:bf], -1.0, W[i + 1:, i], W[i + 1:bf, i])
        if bf < n:
            L10 = W[bf:, kb:bf]
            ops.gemm_inplace(-1.0, L10, np.asfortranarray(L10.T), 1.0, W[bf:, bf:])
    return np.asfortranarray(np.tril(W))


def cholesky_solve(L, b):  # direct.py:166-171
    y = forward_substitution(L, b, unit_diagonal=False)
    return backward_substitution(np.asfortranarray(L.T), y)
