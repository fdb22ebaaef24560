"""CPU test double of distributed.CudaShardOps (test infrastructure only).

Implements the per-rank compute of the multi-GPU drivers with NumPy on torch CPU
tensors so the host logic (sharding, collectives, rank-ordered reductions,
stopping, block-cyclic LU) runs under torch.distributed/gloo on a CPU box.  The
kernels' contracts (ds_dist.cu) are mirrored: (sum x^2, scale, ssq) records,
rank-ordered combination, state words, NumPy rounding of elementwise updates.
"""
import math

import numpy as np

from paper_1511_07207_b200.distributed import combine3_host

ST_RS, ST_BNORM, ST_STATUS, ST_STOP, ST_BAD, ST_RES = range(6)


def vec(t):
    return t.numpy()


def mat(flat, ld, rows, cols):
    a = flat.reshape(-1).numpy()
    return np.lib.stride_tricks.as_strided(a, shape=(rows, cols), strides=(a.itemsize, ld * a.itemsize))


def parts3(x):
    x = np.asarray(x, dtype=np.float64)
    s2 = float(np.dot(x, x))
    m = float(np.max(np.abs(x))) if x.size else 0.0
    if m == 0.0 or not np.isfinite(m):
        return [s2, m, 1.0 if m != 0.0 else 0.0]
    return [s2, m, float(np.dot(x / m, x / m))]


class NumpyShardOps:
    def sync(self):
        pass

    def vec_parts(self, x, out3):
        out3.numpy()[:] = parts3(vec(x))

    def resid_parts(self, A, lda, m, n, x_full, b, r, out3):
        Am = mat(A, lda, m, n)
        rv = vec(r)
        rv[:] = vec(b) + -1.0 * (Am @ vec(x_full)[:n])
        out3.numpy()[:] = parts3(rv)

    def gemv(self, A, lda, m, n, x, y):
        vec(y)[:] = mat(A, lda, m, n) @ vec(x)[:n]

    def gemv_acc(self, A, lda, m, n, x, y):
        vec(y)[:] = vec(y) + 1.0 * (mat(A, lda, m, n) @ vec(x)[:n])

    def dot_dev(self, x, y, out1):
        out1.numpy()[0] = float(np.dot(vec(x).astype(np.float64), vec(y).astype(np.float64)))

    def cg_init(self, bparts, rparts, G, state, hist, tol, cap):
        st = state.numpy()
        _, bn = combine3_host(bparts.numpy())
        rs, rn = combine3_host(rparts.numpy())
        res = rn / bn if bn != 0 else math.inf
        st[ST_RS], st[ST_BNORM], st[ST_STATUS], st[ST_RES] = rs, bn, 0.0, res
        st[ST_STOP] = float(cap) if (res > tol and cap > 0) else 0.0
        hist.numpy()[0] = res

    def cg_update(self, G, pap_all, state, k, x, r, p, Ap, out3):
        st = state.numpy()
        if st[ST_STOP] <= k:
            return
        pAp = 0.0
        for v in pap_all.numpy():
            pAp += float(v)
        if pAp <= 0.0:
            st[ST_STATUS], st[ST_BAD] = 5.0, pAp
            return
        alpha = st[ST_RS] / pAp
        xv, rv = vec(x), vec(r)
        xv[:] = xv + alpha * vec(p)
        rv[:] = rv + (-alpha) * vec(Ap)
        out3.numpy()[:] = parts3(rv)

    def cg_finish(self, G, parts_all, state, k, r, p, hist, tol, cap):
        st = state.numpy()
        if st[ST_STOP] <= k or st[ST_STATUS] != 0.0:
            if st[ST_STATUS] != 0.0 and st[ST_STOP] > k:
                st[ST_STOP] = float(k)
            return
        rs_new, nrm = combine3_host(parts_all.numpy())
        beta = rs_new / st[ST_RS]
        pv = vec(p)
        pv[:] = vec(r) + beta * pv
        res = nrm / st[ST_BNORM]
        st[ST_RS], st[ST_RES] = rs_new, res
        hist.numpy()[k + 1] = res
        if not (res > tol) or k + 1 >= cap:
            st[ST_STOP] = float(k + 1)

    def absdiff_t(self, A, lda, m, n, B, ldb):
        Am, Bm = mat(A, lda, m, n), mat(B, ldb, n, m)
        return float(np.max(np.abs(Am - Bm.T))), float(np.max(np.abs(Am)))

    # GMRES
    def multidot(self, V, ldv, n_loc, kc, w, out):
        Vm = mat(V, ldv, n_loc, kc)
        out.numpy()[:kc] = Vm.T.astype(np.float64) @ vec(w).astype(np.float64)

    def cgs_update(self, V, ldv, n_loc, kc, w, G, parts_all, Hcol, hsave, ps, out3, state, k):
        st = state.numpy()
        if st[ST_STOP] <= k:
            return
        pa = parts_all.numpy().reshape(G, kc)
        h = [sum(float(pa[q, j]) for q in range(G)) for j in range(kc)]
        hv, Hc = hsave.numpy(), vec(Hcol)
        for j in range(kc):
            if ps == 0:
                hv[j] = h[j]
                Hc[j] = h[j]
            else:
                Hc[j] = hv[j] + h[j]
        wv = vec(w)
        Vm = mat(V, ldv, n_loc, kc)
        for j in range(kc):
            wv[:] = wv + (-h[j]) * Vm[:, j]
        out3.numpy()[:] = parts3(wv)

    def gm_start(self, r, v0, G, parts_all, g, state):
        _, beta = combine3_host(parts_all.numpy())
        vec(v0)[:] = (1.0 / beta) * vec(r)
        vec(g)[0] = beta

    def gm_step(self, w, G, parts_all, H, Hraw, ldh, g, cs, sn, k, est, state, tol, total_before, cap):
        st = state.numpy()
        if st[ST_STOP] <= k:
            return
        _, hk1 = combine3_host(parts_all.numpy())
        happy = hk1 == 0.0
        wv = vec(w)
        if not happy:
            wv[:] = (1.0 / hk1) * wv
        Hm = mat(H, ldh, ldh, ldh - 1)
        Hr = mat(Hraw, ldh, ldh, ldh - 1)
        gv, c, s = vec(g), vec(cs), vec(sn)
        Hm[k + 1, k] = hk1
        Hr[:, k] = Hm[:, k]
        for j in range(k):
            t = c[j] * Hm[j, k] + s[j] * Hm[j + 1, k]
            Hm[j + 1, k] = -s[j] * Hm[j, k] + c[j] * Hm[j + 1, k]
            Hm[j, k] = t
        denom = np.hypot(Hm[k, k], Hm[k + 1, k])
        c[k], s[k] = Hm[k, k] / denom, Hm[k + 1, k] / denom
        Hm[k, k] = denom
        Hm[k + 1, k] = 0.0
        gv[k + 1] = -s[k] * gv[k]
        gv[k] = c[k] * gv[k]
        e = abs(float(gv[k + 1])) / st[ST_BNORM]
        est.numpy()[k] = e
        if happy:
            st[ST_BAD] = 1.0
        if happy or e <= tol or total_before + k + 1 >= cap:
            st[ST_STOP] = float(k + 1)

    def gm_lsq(self, H, ldh, g, inner, y, state):
        Hm = mat(H, ldh, ldh, ldh - 1)
        yv, gv = vec(y), vec(g)
        yv[:inner] = gv[:inner]
        for i in range(inner - 1, -1, -1):
            if i + 1 < inner:
                yv[i] -= Hm[i, i + 1:inner] @ yv[i + 1:inner]
            if Hm[i, i] == 0.0:
                state.numpy()[ST_STATUS] = 4.0
                state.numpy()[ST_RES] = float(i)
                return
            yv[i] /= Hm[i, i]

    # LU
    def lu_panel(self, P, ldp, m, w, b, piv, zero):
        W = mat(P, ldp, m, w)
        pv, zf = vec(piv), vec(zero)
        b = min(b, w)
        for kb in range(0, w, b):
            bf = min(kb + b, w)
            for i in range(kb, bf):
                v = i + int(np.argmax(np.abs(W[i:, i])))
                pv[i] = v
                if v != i:
                    W[[i, v], :] = W[[v, i], :]
                aii = W[i, i]
                if aii == 0.0:
                    zf[i] = 1
                    continue
                if i + 1 < m:
                    W[i + 1:, i] = (1.0 / aii) * W[i + 1:, i]
                    if i + 1 < bf:
                        W[i + 1:, i + 1:bf] += -1.0 * np.outer(W[i + 1:, i], W[i, i + 1:bf])
            if bf < w:
                Z = W[kb:bf, bf:].copy()
                for i in range(1, bf - kb):
                    Z[i, :] -= W[kb + i, kb:kb + i] @ Z[:i, :]
                W[kb:bf, bf:] = Z
                W[bf:, bf:] = W[bf:, bf:] - W[bf:, kb:bf] @ W[kb:bf, bf:]

    def laswp(self, A, lda, ncols, k0, k1, piv):
        Am = mat(A, lda, lda, ncols)
        pv = vec(piv)
        for k in range(k0, k1):
            p = int(pv[k])
            if p != k:
                Am[[k, p], :] = Am[[p, k], :]

    def trsm_lower_unit(self, b, m, L, ldl, B, ldb):
        Lm, Bm = mat(L, ldl, b, b), mat(B, ldb, b, m)
        for i in range(1, b):
            Bm[i, :] -= Lm[i, :i] @ Bm[:i, :]

    def gemm_sub(self, m, n, k, A, lda, B, ldb, C, ldc):
        Cm = mat(C, ldc, m, n)
        Cm[:, :] = Cm - mat(A, lda, m, k) @ mat(B, ldb, k, n)
