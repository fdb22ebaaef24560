// ds_krylov.cu — CG and restarted GMRES(m) with device-side convergence control.
//
// CG  restates krylov.cg_solve    (/root/reference/pkg/src/densolve/krylov.py:36-72)
// GMRES restates krylov.gmres_solve (krylov.py:75-182)
//
// Every iteration is a short fixed sequence of kernels; all scalars (alpha,
// beta, rho, Givens rotations, residual estimates, stop decisions) live on the
// device.  Kernels of iteration k are gated on a device word `stop_it`
// (Gate{stop_it, k}) so the host enqueues iterations speculatively in growing
// chunks and synchronises only once per chunk — never once per dot product as
// the reference's Python loop does.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

constexpr int kT = 256;  // threads per block of the vector kernels

// ============================================================================
// CG
// ============================================================================
struct CgDev {
  int64_t stop_it;  // number of completed iterations at which the loop stops
  int32_t status;   // DS_OK or DS_ENOTSPD
  int32_t pad;
  double bad_val;   // offending p'Ap
  double bnorm;
};

// r0 = b - A x0 was produced by gemv EPI_RESID; finish the setup of krylov.py:47-52
__global__ void cg_init_kernel(const double* red, int nblk, CgDev* st, double* rs_hist,
                               double* hist, double tol, int64_t cap) {
  __shared__ double sm[64];
  Ssq q{0.0, 0.0};
  double s2 = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    q = ssq_merge(q, Ssq{red[2 * i], red[2 * i + 1]});
    s2 += red[2 * nblk + i];
  }
  q = block_ssq(q, sm);
  s2 = block_sum(s2, sm);
  if (threadIdx.x == 0) {
    const double res = ssq_norm(q.scale, q.ssq) / st->bnorm;  // nrm2(r)/bnorm (krylov.py:48)
    hist[0] = res;
    rs_hist[0] = s2;  // rs = dot(r, r) (krylov.py:52)
    st->stop_it = (res > tol && 0 < cap) ? cap : 0;
    st->status = DS_OK;
  }
}

// alpha = rs/pAp ; x += alpha p ; r -= alpha Ap ; partials of r.r and ssq(r)
template <typename T>
__global__ void __launch_bounds__(kT)
    cg_update_kernel(int64_t n, T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p,
                     const T* __restrict__ Ap, const double* __restrict__ red_pap, int nblk_pap,
                     const double* __restrict__ rs_hist, CgDev* st, double* __restrict__ red_out,
                     Gate gate) {
  if (gated(gate)) return;
  __shared__ double sm[64];
  const double pAp = reduce_sum_partials(red_pap, nblk_pap, sm);  // same order in every block
  if (pAp <= 0.0) {  // krylov.py:57-58
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->status = DS_ENOTSPD;
      st->bad_val = pAp;
      st->stop_it = gate.k;
    }
    return;
  }
  const double alpha = rs_hist[gate.k] / pAp;  // krylov.py:59
  const T a = (T)alpha, na = (T)(-alpha);
  Ssq q{0.0, 0.0};
  double s2 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = add_rn(x[i], mul_rn(a, p[i]));              // x = axpy(alpha, p, x)
    const T ri = add_rn(r[i], mul_rn(na, Ap[i]));      // r = axpy(-alpha, Ap, r)
    r[i] = ri;
    const double rd = (double)ri;
    s2 = fma(rd, rd, s2);
    q = ssq_add(q, rd);
  }
  q = block_ssq(q, sm);
  s2 = block_sum(s2, sm);
  if (threadIdx.x == 0) {
    red_out[blockIdx.x] = s2;
    red_out[gridDim.x + 2 * blockIdx.x] = q.scale;
    red_out[gridDim.x + 2 * blockIdx.x + 1] = q.ssq;
  }
}

// beta = rs_new/rs ; p = r + beta p ; history, stop decision (krylov.py:62-67)
template <typename T>
__global__ void __launch_bounds__(kT)
    cg_finish_kernel(int64_t n, const T* __restrict__ r, T* __restrict__ p,
                     const double* __restrict__ red, int nblk, double* rs_hist, double* hist,
                     CgDev* st, double tol, int64_t cap, Gate gate) {
  if (gated(gate)) return;
  __shared__ double sm[64];
  double s2 = 0.0;
  Ssq q{0.0, 0.0};
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    s2 += red[i];
    q = ssq_merge(q, Ssq{red[nblk + 2 * i], red[nblk + 2 * i + 1]});
  }
  s2 = block_sum(s2, sm);
  q = block_ssq(q, sm);
  const int64_t k = gate.k;
  const double beta = s2 / rs_hist[k];
  const T bt = (T)beta;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = add_rn(r[i], mul_rn(bt, p[i]));  // p = axpy(rs_new/rs, p, r)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double res = ssq_norm(q.scale, q.ssq) / st->bnorm;
    rs_hist[k + 1] = s2;
    hist[k + 1] = res;
    if (!(res > tol) || k + 1 >= cap) st->stop_it = k + 1;
  }
}

__global__ void set_bnorm_kernel(const double* norm, CgDev* st) {
  if (threadIdx.x == 0) st->bnorm = norm[0];
}

static int vec_grid(ds_ctx* ctx, int64_t n) {
  int64_t want = ceil_div(std::max<int64_t>(n, 1), kT);
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->num_sms * 2));
}


template <typename T>
int cg_impl(ds_ctx* ctx, int64_t n, const T* A, int64_t lda, const T* b, const T* x0, T* x,
            double tol, int64_t cap, int check_sym, double* h_hist, int64_t hist_cap,
            ds_solve_info* info) {
  const int64_t launches0 = ctx->launches;
  const double u = (sizeof(T) == 8 ? 1.1102230246251565e-16 : 5.960464477539063e-08);
  if (check_sym) {
    double md = 0, am = 0;
    DS_TRY(ds_symmetry_check(ctx, sizeof(T) == 8 ? DS_F64 : DS_F32, n, A, lda, &md, &am));
    if (md > 10.0 * u * am) {  // krylov.py:42-44
      set_error("matrix is not symmetric");
      info->error_index = -1;
      return DS_ENOTSPD;
    }
  }
  const GemvPlan gp = gemv_plan(ctx, n, n, sizeof(T));
  const int rblocks = (int)ceil_div(std::max<int64_t>(n, 1), 256);
  const int vg = vec_grid(ctx, n);
  // workspace
  size_t need = 0;
  {
    need += gp.part_bytes + 256;
    need += (size_t)n * sizeof(T) * 3 + 3 * 256;                    // r, p, Ap
    need += ((size_t)rblocks * 3 + (size_t)vg * 3 + 64) * sizeof(double) * 2 + 4 * 256;
    need += (size_t)(cap + 2) * sizeof(double) * 2 + 2 * 256;       // rs_hist, hist
    need += sizeof(CgDev) + 256 + 64;
  }
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, need, &ws));
  Carver cv{(char*)ws};
  double* part = cv.take<double>(gp.part_bytes);
  T* r = cv.take<T>((size_t)n * sizeof(T));
  T* p = cv.take<T>((size_t)n * sizeof(T));
  T* Ap = cv.take<T>((size_t)n * sizeof(T));
  double* red_a = cv.take<double>(((size_t)rblocks * 3 + 64) * sizeof(double));
  double* red_b = cv.take<double>(((size_t)vg * 3 + 64) * sizeof(double));
  double* rs_hist = cv.take<double>((size_t)(cap + 2) * sizeof(double));
  double* hist = cv.take<double>((size_t)(cap + 2) * sizeof(double));
  CgDev* st = cv.take<CgDev>(sizeof(CgDev));
  double* scal = cv.take<double>(64);

  // ||b|| = nrm2(b) (krylov.py:45 -> _rhs_norm :29-33)
  int nb = 0;
  DS_TRY(ssq_launch<T>(ctx, n, b, red_b, &nb));
  DS_TRY(finish_ssq(ctx, red_b, nb, scal));
  double bnorm = 0;
  DS_CUDA(cudaMemcpyAsync(&bnorm, scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (bnorm == 0.0) {
    set_error("||b|| = 0");
    return DS_EDEGRHS;
  }
  set_bnorm_kernel<<<1, 32, 0, ctx->stream>>>(scal, st);
  count_launch(ctx);
  // x = x0.copy(); r = b - A x; res; p = r; rs = r.r   (krylov.py:46-52)
  if (x != x0) DS_CUDA(cudaMemcpyAsync(x, x0, n * sizeof(T), cudaMemcpyDeviceToDevice, ctx->stream));
  int rb = 0;
  DS_TRY(gemv_launch<T>(ctx, gp, A, lda, x, r, part, EPI_RESID, b, red_a, &rb));
  cg_init_kernel<<<1, 256, 0, ctx->stream>>>(red_a, rb, st, rs_hist, hist, tol, cap);
  count_launch(ctx);
  DS_CUDA(cudaMemcpyAsync(p, r, n * sizeof(T), cudaMemcpyDeviceToDevice, ctx->stream));
  DS_CHECK_LAUNCH();

  // hot loop (krylov.py:54-67), enqueued in growing chunks
  int64_t* h_stop = nullptr;
  DS_TRY(ctx_hostbuf(ctx, 64, (void**)&h_stop));
  int64_t k = 0, chunk = 2;
  int64_t stop_it = cap;
  while (true) {
    // read the stop word produced so far
    DS_CUDA(cudaMemcpyAsync(h_stop, &st->stop_it, sizeof(int64_t), cudaMemcpyDeviceToHost,
                            ctx->stream));
    DS_CUDA(cudaStreamSynchronize(ctx->stream));
    stop_it = *h_stop;
    if (stop_it <= k || k >= cap) break;
    const int64_t kend = std::min<int64_t>(cap, k + chunk);
    for (; k < kend; ++k) {
      const Gate g{&st->stop_it, k};
      int rb2 = 0;
      DS_TRY(gemv_launch<T>(ctx, gp, A, lda, p, Ap, part, EPI_DOT, p, red_a, &rb2, g));
      cg_update_kernel<T><<<vg, kT, 0, ctx->stream>>>(n, x, r, p, Ap, red_a, rb2, rs_hist, st,
                                                      red_b, g);
      cg_finish_kernel<T><<<vg, kT, 0, ctx->stream>>>(n, r, p, red_b, vg, rs_hist, hist, st, tol,
                                                      cap, g);
      count_launch(ctx, 2);
    }
    DS_CHECK_LAUNCH();
    chunk = std::min<int64_t>(chunk * 2, 64);
  }
  // results
  CgDev hst;
  DS_CUDA(cudaMemcpyAsync(&hst, st, sizeof(CgDev), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hst.status == DS_ENOTSPD) {
    set_error("p'Ap = %.17g <= 0: matrix is not positive definite", hst.bad_val);
    info->error_value = hst.bad_val;
    info->error_index = hst.stop_it;
    return DS_ENOTSPD;
  }
  const int64_t iters = std::min<int64_t>(hst.stop_it, cap);
  const int64_t hl = std::min<int64_t>(iters + 1, hist_cap);
  if (h_hist && hl > 0)
    DS_CUDA(cudaMemcpyAsync(h_hist, hist, hl * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
  double res = 0;
  DS_CUDA(cudaMemcpyAsync(&res, hist + iters, sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  info->iterations = iters;
  info->history_len = hl;
  info->final_relative_residual = res;
  info->converged = res <= tol;  // krylov.py:68
  info->breakdown = DS_BREAKDOWN_NONE;
  info->kernel_launches = ctx->launches - launches0;
  return DS_OK;
}

// ============================================================================
// GMRES(m)
// ============================================================================
struct GmDev {
  int64_t stop_k;  // inner step at which the cycle stops (m if it runs full)
  int32_t happy;
  int32_t status;  // DS_OK / DS_ESINGULAR (LS solve)
  int64_t bad_row;
  double beta;     // ||r0|| of the cycle
  double bnorm;    // nrm2(b)
  int64_t givens_done;  // cluster path with deferred Givens: columns rotated so far
};

// multi-dot  h_j = V[:,j] . w  for j < kc (one pass over V, w kept in registers)
template <typename T>
__global__ void __launch_bounds__(kT)
    multidot_kernel(int64_t n, const T* __restrict__ V, int64_t ldv, int kc,
                    const T* __restrict__ w, double* __restrict__ part, int ldp, Gate gate) {
  if (gated(gate)) return;
  __shared__ double sm[kT / 32][64];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double wi = i < n ? (double)w[i] : 0.0;
  for (int c0 = 0; c0 < kc; c0 += 64) {  // columns in chunks of 64 (restart_m > 62)
    const int cn = min(64, kc - c0);
    if (c0 > 0) __syncthreads();
    for (int j = 0; j < cn; ++j) {
      double s = i < n ? (double)V[i + (int64_t)(c0 + j) * ldv] * wi : 0.0;
      s = warp_sum(s);
      if (lane == 0) sm[wid][j] = s;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cn; j += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < kT / 32; ++q) s += sm[q][j];
      part[(int64_t)blockIdx.x * ldp + c0 + j] = s;
    }
  }
}

// w -= sum_j h_j V[:,j] (sequential axpys, krylov.py:136-138); optionally emits
// ssq partials of the updated w; block 0 records the coefficients.
//   pass 0: H[j,k] = h_j, hsave = h      pass 1 (reorth): H[j,k] = hsave + h
template <typename T>
__global__ void __launch_bounds__(kT)
    cgs_update_kernel(int64_t n, const T* __restrict__ V, int64_t ldv, int kc, T* __restrict__ w,
                      const double* __restrict__ part, int ldp, int nparts, T* Hcol,
                      double* hsave, int pass, double* red_ssq, Gate gate) {
  if (gated(gate)) return;
  extern __shared__ double hs[];  // kc coefficients (dynamic: restart_m > 62)
  __shared__ double sm[64];
  for (int j = threadIdx.x; j < kc; j += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += part[(int64_t)b * ldp + j];
    hs[j] = s;
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    for (int j = threadIdx.x; j < kc; j += blockDim.x) {
      if (pass == 0) {
        hsave[j] = hs[j];
        Hcol[j] = (T)hs[j];
      } else {
        Hcol[j] = (T)(hsave[j] + hs[j]);
      }
    }
  }
  Ssq q{0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    T wi = w[i];
    int j = 0;
    for (; j + 8 <= kc; j += 8) {
      T vv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) vv[u] = V[i + (int64_t)(j + u) * ldv];
#pragma unroll
      for (int u = 0; u < 8; ++u) wi = add_rn(wi, mul_rn((T)(-hs[j + u]), vv[u]));
    }
    for (; j < kc; ++j) wi = add_rn(wi, mul_rn((T)(-hs[j]), V[i + (int64_t)j * ldv]));
    w[i] = wi;
    q = ssq_add(q, (double)wi);
  }
  if (red_ssq) {
    q = block_ssq(q, sm);
    if (threadIdx.x == 0) {
      red_ssq[2 * blockIdx.x] = q.scale;
      red_ssq[2 * blockIdx.x + 1] = q.ssq;
    }
  }
}

// h_{k+1,k} = ||w|| ; v_{k+1} = w / h ; Givens rotation ; LS estimate ; stop gate
// (krylov.py:139-163)
template <typename T>
__global__ void __launch_bounds__(kT)
    gm_step_finish_kernel(int64_t n, T* __restrict__ w /* = V[:,k+1] */, const double* red_ssq,
                          int nblk, T* H, T* Hraw, int64_t ldh, T* g, T* cs, T* sn, int k,
                          double* est_out, GmDev* st, double tol, int64_t total_before,
                          int64_t cap, Gate gate) {
  if (gated(gate)) return;
  __shared__ double sm[64];
  Ssq q{0.0, 0.0};
  for (int i = threadIdx.x; i < nblk; i += blockDim.x)
    q = ssq_merge(q, Ssq{red_ssq[2 * i], red_ssq[2 * i + 1]});
  q = block_ssq(q, sm);
  const double hk1 = ssq_norm(q.scale, q.ssq);
  const bool happy = hk1 == 0.0;
  if (!happy) {
    const T s = (T)(1.0 / hk1);  // scal(1.0/hk1, w) (krylov.py:143-144)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
      w[i] = mul_rn(s, w[i]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    T* Hk = H + (int64_t)k * ldh;
    T* Hr = Hraw + (int64_t)k * ldh;
    Hk[k + 1] = (T)hk1;
    for (int j = 0; j <= k + 1; ++j) Hr[j] = Hk[j];  // Hraw[:,k] = H[:,k] (krylov.py:141)
    for (int j = 0; j < k; ++j) {                     // krylov.py:147-150
      const T t = add_rn(mul_rn(cs[j], Hk[j]), mul_rn(sn[j], Hk[j + 1]));
      Hk[j + 1] = add_rn(mul_rn(-sn[j], Hk[j]), mul_rn(cs[j], Hk[j + 1]));
      Hk[j] = t;
    }
    const T denom = sizeof(T) == 8 ? (T)hypot((double)Hk[k], (double)Hk[k + 1])
                                   : (T)hypotf((float)Hk[k], (float)Hk[k + 1]);  // np.hypot
    cs[k] = div_rn(Hk[k], denom);
    sn[k] = div_rn(Hk[k + 1], denom);
    Hk[k] = denom;
    Hk[k + 1] = T(0);
    g[k + 1] = mul_rn(-sn[k], g[k]);
    g[k] = mul_rn(cs[k], g[k]);
    const double est = fabs((double)g[k + 1]) / st->bnorm;  // krylov.py:160
    est_out[k] = est;
    const int64_t total = total_before + k + 1;
    if (happy) st->happy = 1;
    if (happy || est <= tol || total >= cap) st->stop_k = k + 1;  // krylov.py:162-163
  }
}

// ============================================================================
// Fused Arnoldi step for small / medium n (latency-bound sizes such as C2, n=4096):
// ONE kernel per inner step instead of ~7 launches.  Each CTA owns a contiguous
// block of rows: w = A v_k for its rows (row-split GEMV: no cross-CTA reduction),
// then every CGS pass is a local partial multi-dot, one grid-wide LL exchange of
// the (k+1)-vectors of partials (32-bit data + epoch flag words, summed in fixed
// CTA order by every CTA => identical h everywhere) and a local update; the norm
// is one more exchange of (scale, ssq) records.  CTA 0 records H / Hraw and runs
// the Givens / estimate / stop logic of gm_step_finish_kernel.
// ============================================================================
constexpr int kArnThreads = 512;
constexpr int kArnMaxRows = 128;  // rows per CTA (n <= 148 * 128)

struct ArnArgs {
  int64_t n, lda, ldv, ldh, total_before, cap;
  int k, passes, per;
  unsigned seq;
  double tol;
  uint64_t* ll;  // [2][grid][64 * 2] exchange words
  double* est;
  GmDev* st;
  unsigned long long* trace;  // optional per-CTA phase cycle accumulators (DENSOLVE_GMRES_TRACE)
};

__device__ __forceinline__ void arn_store(uint64_t* p, uint32_t data, uint32_t flag) {
  const uint64_t w = ((uint64_t)flag << 32) | data;
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;\n" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ uint64_t arn_load(const uint64_t* p) {
  uint64_t w;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ void arn_put(uint64_t* p, double v, uint32_t f) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  arn_store(p, (uint32_t)b, f);
  arn_store(p + 1, (uint32_t)(b >> 32), f);
}
// poll one double published with flag f
__device__ __forceinline__ double arn_get(const uint64_t* p, uint32_t f) {
  uint64_t a, b;
  while (true) {
    a = arn_load(p);
    b = arn_load(p + 1);
    if ((uint32_t)(a >> 32) == f && (uint32_t)(b >> 32) == f) break;
  }
  return __longlong_as_double((long long)((a & 0xffffffffull) | (b << 32)));
}

template <typename T, int RCH /* 32-row chunks per CTA: 1, 2 or 4 */>
__global__ void __launch_bounds__(kArnThreads)
    arnoldi_step_kernel(const T* __restrict__ A, T* V, T* H, T* Hraw, T* g, T* cs, T* sn, ArnArgs a,
                        Gate gate) {
  if (gated(gate)) return;
  extern __shared__ __align__(16) unsigned char arn_smem[];
  T* Vb = reinterpret_cast<T*>(arn_smem);  // [kc][nr]: my rows of V[:, 0..k] (staged once)
  __shared__ double wv[kArnMaxRows];      // w for my rows (fp64 copy of the T values)
  __shared__ double red[kArnThreads / 32][kArnMaxRows];
  __shared__ double hs[64], hsave[64], sm[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kArnThreads / 32;
  const unsigned G = gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * a.per;
  const int nr = (int)max((int64_t)0, min((int64_t)a.per, a.n - r0));
  const int k = a.k, kc = k + 1;
  const T* vk = V + (int64_t)k * a.ldv;
  uint32_t round = 0;
  long long tt[8];
  int nt_ = 0;
  tt[nt_++] = clock64();

  // ---- w = A v_k for my rows: warps split the columns, lanes the rows (RCH chunks
  // of 32); U columns per warp in flight per step (RCH * U = 16 loads per thread)
  {
    constexpr int U = 16 / RCH;
    double acc[RCH];
#pragma unroll
    for (int q = 0; q < RCH; ++q) acc[q] = 0.0;
    int64_t c = warp;
    for (; c + (U - 1) * nw < a.n; c += U * nw) {
      T av[U][RCH];
      double xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        xv[u] = (double)__ldg(vk + c + u * nw);
#pragma unroll
        for (int q = 0; q < RCH; ++q) {
          const int r = q * 32 + lane;
          av[u][q] = r < nr ? __ldg(A + (r0 + r) + (c + u * nw) * a.lda) : T(0);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < RCH; ++q) acc[q] = fma((double)av[u][q], xv[u], acc[q]);
    }
    for (; c < a.n; c += nw) {
      const double xv = (double)__ldg(vk + c);
#pragma unroll
      for (int q = 0; q < RCH; ++q) {
        const int r = q * 32 + lane;
        if (r < nr) acc[q] = fma((double)__ldg(A + (r0 + r) + c * a.lda), xv, acc[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < RCH; ++q) red[warp][q * 32 + lane] = acc[q];
    __syncthreads();
    for (int r = tid; r < nr; r += blockDim.x) {
      double s = 0.0;
      for (int w2 = 0; w2 < nw; ++w2) s += red[w2][r];
      wv[r] = (double)(T)s;  // the GEMV result in the array dtype
    }
    __syncthreads();
  }
  tt[nt_++] = clock64();  // after GEMV
  // stage my rows of the basis (L2-resident) once: coalesced, all loads in flight
  for (int e0 = 0; e0 < kc * nr; e0 += (int)blockDim.x * 8) {
    T tv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + tid + u * (int)blockDim.x;
      tv[u] = e < kc * nr ? V[(r0 + e % nr) + (int64_t)(e / nr) * a.ldv] : T(0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + tid + u * (int)blockDim.x;
      if (e < kc * nr) Vb[e] = tv[u];
    }
  }
  __syncthreads();
  tt[nt_++] = clock64();  // after V staging
  // ---- CGS passes (krylov.py:134-138; pass 2 = re-orthogonalisation)
  for (int ps = 0; ps < a.passes; ++ps) {
    // partial h_j over my rows: warp per j, lanes over rows
    for (int j = warp; j < kc; j += nw) {
      const T* vj = Vb + j * nr;
      double s = 0.0;
      for (int r = lane; r < nr; r += 32) s = fma((double)vj[r], wv[r], s);
      s = warp_sum(s);
      if (lane == 0) sm[j] = s;
    }
    __syncthreads();
    // exchange: CTA j reduces component j over the G partials (fixed order), publishes
    // h_j; every CTA then polls the kc results (two round trips, low contention)
    const uint32_t ep = a.seq * 4u + round + 1u;
    uint64_t* buf = a.ll + (size_t)(round & 1) * G * 128;
    uint64_t* res = a.ll + (size_t)2 * G * 128 + (size_t)(round & 1) * 128;
    for (int j = tid; j < kc; j += blockDim.x) arn_put(buf + ((size_t)blockIdx.x * 128) + 2 * j, sm[j], ep);
    ++round;
    for (int j = (int)blockIdx.x; j < kc; j += (int)G) {
      if (warp == 0) {
        uint64_t wd[5][2];
        while (true) {
          bool ok = true;
#pragma unroll
          for (int u = 0; u < 5; ++u) {
            const unsigned bb = lane + 32u * u;
            if (bb < G) {
              wd[u][0] = arn_load(buf + (size_t)bb * 128 + 2 * j);
              wd[u][1] = arn_load(buf + (size_t)bb * 128 + 2 * j + 1);
              ok = ok && (uint32_t)(wd[u][0] >> 32) == ep && (uint32_t)(wd[u][1] >> 32) == ep;
            }
          }
          if (__all_sync(0xffffffffu, ok)) break;
        }
        double v = 0.0;
#pragma unroll
        for (int u = 0; u < 5; ++u)
          if (lane + 32u * u < G)
            v += __longlong_as_double((long long)((wd[u][0] & 0xffffffffull) | (wd[u][1] << 32)));
        v = warp_sum(v);
        if (lane == 0) arn_put(res + 2 * j, v, ep);
      }
    }
    if (warp == 0) {
      for (int j = lane; j < kc; j += 32) hs[j] = arn_get(res + 2 * j, ep);
    }
    __syncthreads();
    if (blockIdx.x == 0) {
      T* Hcol = H + (int64_t)k * a.ldh;
      for (int j = tid; j < kc; j += blockDim.x) {
        if (ps == 0) {
          hsave[j] = hs[j];
          Hcol[j] = (T)hs[j];
        } else {
          Hcol[j] = (T)(hsave[j] + hs[j]);
        }
      }
    }
    // w -= sum_j h_j V[:, j] for my rows (sequential axpys, krylov.py:136-138)
    for (int r = tid; r < nr; r += blockDim.x) {
      T wi = (T)wv[r];
      for (int j = 0; j < kc; ++j) wi = add_rn(wi, mul_rn((T)(-hs[j]), Vb[j * nr + r]));
      wv[r] = (double)wi;
    }
    __syncthreads();
    tt[nt_++] = clock64();  // after each pass
  }
  // ---- h_{k+1,k} = ||w|| (scaled, Backend.nrm2) across the grid
  Ssq q{0.0, 0.0};
  for (int r = tid; r < nr; r += blockDim.x) q = ssq_add(q, wv[r]);
  q = block_ssq(q, sm);
  {
    const uint32_t ep = a.seq * 4u + round + 1u;
    uint64_t* buf = a.ll + (size_t)(round & 1) * G * 128;
    if (tid == 0) {
      arn_put(buf + (size_t)blockIdx.x * 128, q.scale, ep);
      arn_put(buf + (size_t)blockIdx.x * 128 + 2, q.ssq, ep);
    }
    ++round;
    uint64_t* res = a.ll + (size_t)2 * G * 128 + (size_t)(round & 1) * 128;
    ++round;
    if (blockIdx.x == 0 && warp == 0) {  // CTA 0 merges the G records in fixed order
      uint64_t wd[5][4];
      while (true) {
        bool ok = true;
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          const unsigned bb = lane + 32u * u;
          if (bb < G) {
#pragma unroll
            for (int z = 0; z < 4; ++z) {
              wd[u][z] = arn_load(buf + (size_t)bb * 128 + z);
              ok = ok && (uint32_t)(wd[u][z] >> 32) == ep;
            }
          }
        }
        if (__all_sync(0xffffffffu, ok)) break;
      }
      Ssq m{0.0, 0.0};
#pragma unroll
      for (int u = 0; u < 5; ++u)
        if (lane + 32u * u < G)
          m = ssq_merge(m, Ssq{__longlong_as_double((long long)((wd[u][0] & 0xffffffffull) | (wd[u][1] << 32))),
                               __longlong_as_double((long long)((wd[u][2] & 0xffffffffull) | (wd[u][3] << 32)))});
      m = warp_ssq(m);
      if (lane == 0) {
        arn_put(res, m.scale, ep);
        arn_put(res + 2, m.ssq, ep);
      }
    }
    if (tid == 0) {
      sm[0] = arn_get(res, ep);
      sm[1] = arn_get(res + 2, ep);
    }
    __syncthreads();
  }
  tt[nt_++] = clock64();  // after the norm exchange
  if (a.trace && tid == 0)
    for (int z = 1; z < nt_ && z < 7; ++z) atomicAdd(a.trace + blockIdx.x * 8 + z, (unsigned long long)(tt[z] - tt[z - 1]));
  const double hk1 = ssq_norm(sm[0], sm[1]);
  const bool happy = hk1 == 0.0;
  {
    T* vout = V + (int64_t)(k + 1) * a.ldv + r0;
    const T sc = (T)(1.0 / hk1);
    for (int r = tid; r < nr; r += blockDim.x) vout[r] = happy ? (T)wv[r] : mul_rn(sc, (T)wv[r]);
  }
  if (blockIdx.x == 0 && tid == 0) {  // Givens, estimate, stop (krylov.py:146-163)
    T* Hk = H + (int64_t)k * a.ldh;
    T* Hr = Hraw + (int64_t)k * a.ldh;
    Hk[k + 1] = (T)hk1;
    for (int j = 0; j <= k + 1; ++j) Hr[j] = Hk[j];
    for (int j = 0; j < k; ++j) {
      const T t = add_rn(mul_rn(cs[j], Hk[j]), mul_rn(sn[j], Hk[j + 1]));
      Hk[j + 1] = add_rn(mul_rn(-sn[j], Hk[j]), mul_rn(cs[j], Hk[j + 1]));
      Hk[j] = t;
    }
    const T denom = sizeof(T) == 8 ? (T)hypot((double)Hk[k], (double)Hk[k + 1])
                                   : (T)hypotf((float)Hk[k], (float)Hk[k + 1]);
    cs[k] = div_rn(Hk[k], denom);
    sn[k] = div_rn(Hk[k + 1], denom);
    Hk[k] = denom;
    Hk[k + 1] = T(0);
    g[k + 1] = mul_rn(-sn[k], g[k]);
    g[k] = mul_rn(cs[k], g[k]);
    const double est = fabs((double)g[k + 1]) / a.st->bnorm;
    a.est[k] = est;
    const int64_t total = a.total_before + k + 1;
    if (happy) a.st->happy = 1;
    if (happy || est <= a.tol || total >= a.cap) a.st->stop_k = k + 1;
  }
}

// ============================================================================
// Cluster orthogonalisation (small / medium n): after w = A v_k (the streamed
// GEMV on every SM), ONE thread-block cluster of up to 16 CTAs runs the CGS
// passes, the norm, the normalisation and the Givens step.  Each CTA owns a
// contiguous row block; the three reductions per step go through distributed
// shared memory (partials in each CTA's smem, cluster barrier, every CTA reads the
// CL partials of each component in rank order => identical h everywhere) instead
// of L2 round trips.  CTA rank 0 records H / Hraw and runs the Givens logic.
// ============================================================================
constexpr int kOrthThreads = 512;
constexpr unsigned kOrthMaxCluster = 16;  // the launch uses 16 or 8

// Givens step of column kk (krylov.py:146-163) by ONE thread, from shared-memory copies:
// hc = raw H[0..kk+1, kk], css / sns = the rotations of the earlier columns.  The running
// H[j+1] is carried in a register (no store -> load round trip per rotation).  Writes the
// rotated column, cs / sn[kk], g[kk..kk+1] and est[kk]; returns the estimate.
template <typename T>
__device__ __forceinline__ double gm_givens_apply(int kk, const T* hc, const T* css, const T* sns, T gk, double bnorm,
                                                  T* H, int64_t ldh, T* g, T* cs, T* sn, double* est_out) {
  T* Hk = H + (int64_t)kk * ldh;
  const T col_last = hc[kk + 1];
  T cur = hc[0];
  for (int j = 0; j < kk; ++j) {
    const T nxt = hc[j + 1];
    const T c = css[j], s_ = sns[j];
    const T t = add_rn(mul_rn(c, cur), mul_rn(s_, nxt));
    cur = add_rn(mul_rn(-s_, cur), mul_rn(c, nxt));
    Hk[j] = t;
  }
  // cur = rotated H[kk], col_last = H[kk+1]
  const T denom = sizeof(T) == 8 ? (T)hypot((double)cur, (double)col_last) : (T)hypotf((float)cur, (float)col_last);
  const T ck = div_rn(cur, denom), sk = div_rn(col_last, denom);
  cs[kk] = ck;
  sn[kk] = sk;
  Hk[kk] = denom;
  Hk[kk + 1] = T(0);
  g[kk + 1] = mul_rn(-sk, gk);
  g[kk] = mul_rn(ck, gk);
  const double est = fabs((double)mul_rn(-sk, gk)) / bnorm;
  est_out[kk] = est;
  return est;
}

// one warp stages raw H[:, kk] and the earlier rotations in shared memory; the scalars the
// chain needs at its end (g[kk], ||b||) are loaded in the same round trip
template <typename T>
__device__ __forceinline__ void gm_givens_stage(int kk, const T* Hraw, int64_t ldh, const T* cs, const T* sn, T* hc,
                                                T* css, T* sns, int lane) {
  const T* Hr = Hraw + (int64_t)kk * ldh;
  for (int j = lane; j <= kk + 1; j += 32) hc[j] = Hr[j];
  for (int j = lane; j < kk; j += 32) {
    css[j] = cs[j];
    sns[j] = sn[j];
  }
}

// Cycle tail of the deferred-Givens cluster path: the last executed step's Givens (its
// cluster had no successor, or the successor was gated by a happy / cap stop).
template <typename T>
__global__ void gm_givens_tail_kernel(int64_t kend, const T* Hraw, T* H, int64_t ldh, T* g, T* cs, T* sn,
                                      double* est_out, GmDev* st, double tol) {
  __shared__ T hc[66], css[64], sns[64];
  const int64_t E = min(st->stop_k, kend);
  if (st->givens_done >= E) return;
  const int kk = (int)(E - 1);
  gm_givens_stage<T>(kk, Hraw, ldh, cs, sn, hc, css, sns, (int)threadIdx.x);
  const T gk = g[kk];
  const double bnorm = st->bnorm;
  __syncwarp();
  if (threadIdx.x == 0) {
    const double est = gm_givens_apply<T>(kk, hc, css, sns, gk, bnorm, H, ldh, g, cs, sn, est_out);
    if (est <= tol) st->stop_k = kk + 1;
    st->givens_done = kk + 1;
  }
}

template <typename T>
__global__ void __launch_bounds__(kOrthThreads, 2)
    arnoldi_orth_cluster_kernel(int64_t n, T* V, int64_t ldv, int k, int passes, T* H, T* Hraw, int64_t ldh, T* g,
                                T* cs, T* sn, double* est_out, GmDev* st, double tol, int64_t total_before,
                                int64_t cap, Gate gate, const double* __restrict__ gpart, int64_t nchunks,
                                unsigned long long* trace, int defer) {
  namespace cgr = cooperative_groups;
  pdl_wait();  // the GEMV partials, V and the stop word come from earlier kernels
  if (gated(gate)) return;
  pdl_launch_dependents();
  cgr::cluster_group cluster = cgr::this_cluster();
  const unsigned CL = cluster.num_blocks();
  const unsigned rank = cluster.block_rank();
  // debug (DENSOLVE_ORTH_TRACE): %globaltimer at the phase boundaries, ranks 0 and CL - 1
  auto stamp = [&](int idx) {
    if (trace && threadIdx.x == 0 && (rank == 0 || rank == CL - 1)) {
      unsigned long long tm;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
      trace[((size_t)k * 2 + (rank == 0 ? 0 : 1)) * 16 + idx] = tm;
    }
  };
  stamp(0);
  extern __shared__ __align__(16) unsigned char orth_smem[];
  double* wv = reinterpret_cast<double*>(orth_smem);  // my rows of w (fp64 copy of T values)
  __shared__ double part[2][64];                      // my CGS partials, buffer per pass
  __shared__ double inbox[2][kOrthMaxCluster];        // norm partials pushed by every CTA
  __shared__ double hs[64], hsave[64], sm[64];
  __shared__ T hcol[66], css[64], sns[64];            // rank 0: H[:, k] and the rotations so far
  __shared__ T ghc[66], gcs[64], gsn[64];             // defer: column k-1's Givens inputs
  __shared__ int s_abort;                             // defer (rank 0): column k-1 stopped the cycle
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kOrthThreads / 32;
  const int64_t per = ceil_div(ceil_div(n, (int64_t)CL), 4) * 4;
  const int64_t r0 = (int64_t)rank * per;
  const int nr = (int)max((int64_t)0, min(per, n - r0));
  const int kc = k + 1;
  T* w = V + (int64_t)(k + 1) * ldv;
  // w = A v_k: the GEMV's chunk partials summed here, in chunk order (ds_colstream_reduce_kernel's
  // order, so w is bitwise the EPI_STORE result), up to 32 loads in flight
  for (int r = tid; r < nr; r += blockDim.x) {
    if (gpart == nullptr) {  // w already summed by the GEMV's reduce kernel
      wv[r] = (double)w[r0 + r];
      continue;
    }
    const double* pr = gpart + r0 + r;
    double s = 0.0;
    constexpr int PB = 16;  // partial loads in flight (the 64-register budget of 2 CTAs/SM)
    for (int64_t c0 = 0; c0 < nchunks; c0 += PB) {
      double v[PB];
#pragma unroll
      for (int u = 0; u < PB; ++u) v[u] = c0 + u < nchunks ? pr[(c0 + u) * n] : 0.0;
#pragma unroll
      for (int u = 0; u < PB; ++u)
        if (c0 + u < nchunks) s += v[u];
    }
    wv[r] = (double)(T)s;
  }
  if (defer) {
    // deferred Givens of column k - 1 (the previous step's estimate and stop test), by the last
    // warp of rank 0, which has no rows here (host: rows per CTA <= kOrthThreads - 32), while
    // the CTA sums the partials; its stop aborts this step before it writes anything
    if (rank == 0 && warp == nw - 1) {
      bool stop = false;
      if (k > 0) {
        // every load of the step in one round trip: the staged column and rotations, g[k-1],
        // ||b|| and the done count (a chunked enqueue's tail may have rotated k-1 already)
        gm_givens_stage<T>(k - 1, Hraw, ldh, cs, sn, ghc, gcs, gsn, lane);
        const int64_t done = st->givens_done;
        const T gk = g[k - 1];
        const double bnorm = st->bnorm;
        __syncwarp();
        if (done == k - 1 && lane == 31) {
          const double est = gm_givens_apply<T>(k - 1, ghc, gcs, gsn, gk, bnorm, H, ldh, g, cs, sn, est_out);
          stop = est <= tol;
          if (stop) st->stop_k = k;
          st->givens_done = k;
        }
      }
      if (lane == 31) s_abort = stop ? 1 : 0;
    }
  } else if (rank == 0) {
    for (int j = tid; j < k; j += blockDim.x) {
      css[j] = cs[j];
      sns[j] = sn[j];
    }
  }
  __syncthreads();
  stamp(1);
  for (int ps = 0; ps < passes; ++ps) {
    // partial h_j over my rows: warp per j, lanes over rows (V from L2)
    for (int j = warp; j < kc; j += nw) {
      const T* vj = V + (int64_t)j * ldv + r0;
      double s = 0.0;
#pragma unroll 8
      for (int r = lane; r < nr; r += 32) s = fma((double)vj[r], wv[r], s);
      s = warp_sum(s);
      if (lane == 0) part[ps][j] = s;
    }
    stamp(2 + 4 * ps);
    cluster.sync();
    if (defer && ps == 0 && *cluster.map_shared_rank(&s_abort, 0)) {
      cluster.sync();  // rank 0's flag stays readable until every CTA has seen it
      return;
    }
    stamp(3 + 4 * ps);
    for (int j = tid; j < kc; j += blockDim.x) {  // rank-ordered sum over the cluster (DSMEM)
      double v[kOrthMaxCluster];  // every remote load in flight before the ordered sum
#pragma unroll
      for (unsigned b = 0; b < kOrthMaxCluster; ++b)
        v[b] = b < CL ? cluster.map_shared_rank(&part[ps][0], b)[j] : 0.0;
      double s = 0.0;
#pragma unroll
      for (unsigned b = 0; b < kOrthMaxCluster; ++b)
        if (b < CL) s += v[b];
      hs[j] = s;
    }
    __syncthreads();
    stamp(4 + 4 * ps);
    if (rank == 0) {
      for (int j = tid; j < kc; j += blockDim.x) {
        if (ps == 0) {
          hsave[j] = hs[j];
          hcol[j] = (T)hs[j];
        } else {
          hcol[j] = (T)(hsave[j] + hs[j]);
        }
      }
    }
    // w -= sum_j h_j V[:, j] for my rows (sequential axpys, krylov.py:136-138)
    for (int r = tid; r < nr; r += blockDim.x) {
      T wi = (T)wv[r];
      const T* vr = V + r0 + r;
      constexpr int VB = sizeof(T) == 8 ? 16 : 32;  // basis loads in flight, then the ordered axpys
      for (int j0 = 0; j0 < kc; j0 += VB) {
        T vv[VB];
#pragma unroll
        for (int u = 0; u < VB; ++u) vv[u] = j0 + u < kc ? vr[(int64_t)(j0 + u) * ldv] : T(0);
#pragma unroll
        for (int u = 0; u < VB; ++u)
          if (j0 + u < kc) wi = add_rn(wi, mul_rn((T)(-hs[j0 + u]), vv[u]));
      }
      wv[r] = (double)wi;
    }
    __syncthreads();
    stamp(5 + 4 * ps);
  }
  // h_{k+1,k} = nrm2(w), the reference's two-pass form (backends.py:114-122):
  // m = max|w| (exact, order-free), then m * sqrt(sum (w/m)^2).  Both cluster
  // exchanges PUSH each CTA's partial into every CTA's inbox before the barrier,
  // so afterwards only local shared memory is read (no exit guard needed).
  double mx = 0.0;
  for (int r = tid; r < nr; r += blockDim.x) mx = nan_max(mx, fabs(wv[r]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = nan_max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) sm[warp] = mx;
  __syncthreads();
  if (tid < (int)CL) {
    double cm = 0.0;
    for (int w2 = 0; w2 < nw; ++w2) cm = nan_max(cm, sm[w2]);
    cluster.map_shared_rank(&inbox[0][0], (unsigned)tid)[rank] = cm;
  }
  cluster.sync();
  double m_all = 0.0;
#pragma unroll
  for (unsigned b = 0; b < kOrthMaxCluster; ++b)
    if (b < CL) m_all = nan_max(m_all, inbox[0][b]);
  double hk1 = m_all;
  if (m_all != 0.0 && m_all - m_all == 0.0) {  // finite, nonzero
    double s2 = 0.0;
    for (int r = tid; r < nr; r += blockDim.x) {
      const double t = div_rn(wv[r], m_all);
      s2 = add_rn(s2, mul_rn(t, t));
    }
    s2 = block_sum(s2, sm);
    if (tid < (int)CL) cluster.map_shared_rank(&inbox[1][0], (unsigned)tid)[rank] = s2;
    cluster.sync();
    double tot = 0.0;
#pragma unroll
    for (unsigned b = 0; b < kOrthMaxCluster; ++b)
      if (b < CL) tot += inbox[1][b];
    hk1 = mul_rn(m_all, sqrt(tot));
  }
  stamp(10);
  const bool happy = hk1 == 0.0;
  {
    const T sc = (T)(1.0 / hk1);  // scal(1.0/hk1, w) (krylov.py:143-144)
    for (int r = tid; r < nr; r += blockDim.x) w[r0 + r] = happy ? (T)wv[r] : mul_rn(sc, (T)wv[r]);
  }
  stamp(11);
  if (rank == 0) {  // raw column, then Givens, estimate, stop (krylov.py:146-163)
    T* Hr = Hraw + (int64_t)k * ldh;
    for (int j = tid; j <= k; j += blockDim.x) Hr[j] = hcol[j];
    if (tid == 0) {
      Hr[k + 1] = (T)hk1;
      const int64_t total = total_before + k + 1;
      if (happy) st->happy = 1;
      if (defer) {  // the estimate waits for the next step's cluster (or the cycle tail)
        if (happy || total >= cap) st->stop_k = k + 1;
      } else {
        hcol[k + 1] = (T)hk1;
        const double est = gm_givens_apply<T>(k, hcol, css, sns, g[k], st->bnorm, H, ldh, g, cs, sn, est_out);
        if (happy || est <= tol || total >= cap) st->stop_k = k + 1;
      }
    }
  }
  stamp(12);
}

// y = H[:inner,:inner]^-1 g[:inner] (backward_substitution, direct.py:139-152): the
// block stages the upper triangle in shared memory, then one thread runs the
// dependent recurrence out of shared memory (no global round trip per term)
// inner < 0: the cycle's stop step is read on the device (inner = min(stop_k, -inner)) and
// y is written up to -inner with zeros past it, so the host enqueues the cycle's tail
// without a readback (the x update then runs over -inner columns).
template <typename T>
__global__ void gm_lsq_kernel(const T* H, int64_t ldh, const T* g, int inner, T* y, GmDev* st) {
  __shared__ T Hs[64][65];
  __shared__ T ys[64];
  const int ypad = inner < 0 ? -inner : inner;
  if (inner < 0) {
    inner = (int)min(st->stop_k, (int64_t)ypad);
    for (int i = inner + (int)threadIdx.x; i < ypad; i += blockDim.x) y[i] = T(0);
  }
  for (int idx = threadIdx.x; idx < inner * inner; idx += blockDim.x) {
    const int i = idx % inner, j = idx / inner;
    if (i <= j) Hs[i][j] = H[i + (int64_t)j * ldh];
  }
  for (int i = threadIdx.x; i < inner; i += blockDim.x) ys[i] = g[i];
  __syncthreads();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = inner - 1; i >= 0; --i) {
    T yi = ys[i];
    if (i + 1 < inner) {
      double s = 0.0;
      for (int j = i + 1; j < inner; ++j) s = fma((double)Hs[i][j], (double)ys[j], s);
      yi = sub_rn(yi, (T)s);
    }
    ys[i] = yi;
    const T d = Hs[i][i];
    if (d == T(0)) {
      st->status = DS_ESINGULAR;
      st->bad_row = i;
      for (int k = 0; k < inner; ++k) y[k] = ys[k];
      return;
    }
    ys[i] = div_rn(yi, d);
  }
  for (int k = 0; k < inner; ++k) y[k] = ys[k];
}

// the same recurrence for inner > 64 (restart_m > 62), straight from global memory
template <typename T>
__global__ void gm_lsq_global_kernel(const T* H, int64_t ldh, const T* g, int inner, T* y, GmDev* st) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = 0; i < inner; ++i) y[i] = g[i];
  for (int i = inner - 1; i >= 0; --i) {
    T yi = y[i];
    if (i + 1 < inner) {
      double s = 0.0;
      for (int j = i + 1; j < inner; ++j) s = fma((double)H[i + (int64_t)j * ldh], (double)y[j], s);
      yi = sub_rn(yi, (T)s);
    }
    y[i] = yi;
    const T d = H[i + (int64_t)i * ldh];
    if (d == T(0)) {
      st->status = DS_ESINGULAR;
      st->bad_row = i;
      return;
    }
    y[i] = div_rn(yi, d);
  }
}

// cycle start: V[:,0] = scal(1/beta, r); g = beta e1 (krylov.py:116-123)
// cycle start: V[:,0] = scal(1/beta, r), the rest of V, H, Hraw, g, cs, sn zeroed, g = beta e1
// (krylov.py:116-123), and the device state of the cycle initialised (one launch instead of
// four memsets, a host-to-device copy and the scaling kernel)
template <typename T>
__global__ void gm_cycle_start_kernel(int64_t n, const T* __restrict__ r, T* __restrict__ V, int64_t vlen,
                                      T* __restrict__ H, T* __restrict__ Hraw, int64_t hlen, T* __restrict__ g,
                                      int64_t glen, double* __restrict__ est, double beta, double bnorm, int64_t m,
                                      GmDev* st) {
  const T s = (T)(1.0 / beta);
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = i0; i < vlen; i += step) V[i] = i < n ? mul_rn(s, r[i]) : T(0);
  for (int64_t i = i0; i < hlen; i += step) {
    H[i] = T(0);
    Hraw[i] = T(0);
  }
  for (int64_t i = i0; i < glen; i += step) g[i] = i == 0 ? (T)beta : T(0);
  for (int64_t i = i0; i < m; i += step) est[i] = 0.0;  // read back whole with the device-side tail
  if (i0 == 0) {
    GmDev d{};
    d.stop_k = m;
    d.bad_row = -1;
    d.beta = beta;
    d.bnorm = bnorm;
    *st = d;
  }
}

__global__ void finish_resid_kernel(const double* red, int nblk, double* out) {
  // out[0] = nrm2 (scaled, Backend.nrm2), out[1] = plain sum of squares
  __shared__ double sm[64];
  Ssq q{0.0, 0.0};
  double s2 = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    q = ssq_merge(q, Ssq{red[2 * i], red[2 * i + 1]});
    s2 += red[2 * nblk + i];
  }
  q = block_ssq(q, sm);
  s2 = block_sum(s2, sm);
  if (threadIdx.x == 0) {
    out[0] = ssq_norm(q.scale, q.ssq);
    out[1] = s2;
  }
}

template <typename T>
int gmres_impl(ds_ctx* ctx, int64_t n, const T* A, int64_t lda, const T* b, const T* x0, T* x,
               double tol, int64_t cap, int64_t m, int orth, double* h_hist, int64_t hist_cap,
               int64_t* h_cycles, int64_t cycles_cap, ds_sink_fn sink, void* sink_user,
               ds_solve_info* info) {
  const int64_t launches0 = ctx->launches;
  const double u = (sizeof(T) == 8 ? 1.1102230246251565e-16 : 5.960464477539063e-08);
  // restart_m > 62: the fused step kernel and the cluster kernel keep <= 64 coefficients
  // on chip, so large m runs the split multidot / cgs_update / step_finish kernels
  // (coefficients in dynamic shared / global memory) and the global-memory LS solve.
  const bool big_m = m > 62;
  if (m + 1 > 6144) {  // the CGS coefficients of one step live in <= 48 KB of shared memory
    set_error("restart_m = %lld exceeds the supported maximum of 6143", (long long)m);
    return DS_EINVAL;
  }
  const GemvPlan gp = gemv_plan(ctx, n, n, sizeof(T));
  const int rblocks = (int)ceil_div(std::max<int64_t>(n, 1), 256);
  const int vg = vec_grid(ctx, n);
  const int mdb = (int)ceil_div(std::max<int64_t>(n, 1), kT);  // multidot blocks
  const int64_t ldv = ceil_div(std::max<int64_t>(n, 1), 4) * 4;
  const int64_t ldh = m + 1;
  const int ldp = (int)std::max<int64_t>(64, ceil_div(m + 1, 64) * 64);
  // fused one-kernel Arnoldi step for n <= 148 * 128 (latency-bound sizes, e.g. C2)
  const char* fz = getenv("DENSOLVE_GMRES_FUSED");
  int64_t arn_g = std::min<int64_t>((int64_t)ctx->num_sms, ceil_div(n, 4));
  int64_t arn_per = ceil_div(ceil_div(n, arn_g), 4) * 4;  // 32-byte aligned row blocks
  arn_g = ceil_div(n, arn_per);
  const bool fused = !(fz && fz[0] == '0') && arn_per <= kArnMaxRows && !big_m;
  // cluster orthogonalisation (DENSOLVE_GMRES_ORTH=cluster|grid): the largest cluster
  // (16 non-portable, else 8) that the device can co-schedule; rows per CTA <= 4096
  int orth_cl = 0;
  size_t orth_smem = 0;
  bool orth_fold = true;
  static const bool pdl_on = [] {  // programmatic dependent launch in the cluster path
    const char* e = getenv("DENSOLVE_PDL");
    return !(e && e[0] == '0');
  }();
  unsigned long long* orth_trace = nullptr;
  int orth_defer = 0;
  {
    const char* oe = getenv("DENSOLVE_GMRES_ORTH");
    const bool want = !(oe && strcmp(oe, "grid") == 0) && n <= 16 * 4096 && !big_m;
    if (want) {
      static int best[2] = {-1, -1};
      int& bc = best[sizeof(T) == 8];
      if (bc < 0) {
        bc = 0;
        DS_CUDA(cudaFuncSetAttribute(arnoldi_orth_cluster_kernel<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        DS_CUDA(cudaFuncSetAttribute(arnoldi_orth_cluster_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     4096 * (int)sizeof(double)));
        for (int c : {16, 8}) {
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3((unsigned)c);
          lc.blockDim = dim3(kOrthThreads);
          lc.dynamicSmemBytes = 4096 * sizeof(double);
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = (unsigned)c;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          lc.attrs = at;
          lc.numAttrs = 1;
          int nclusters = 0;
          if (cudaOccupancyMaxActiveClusters(&nclusters, (void*)arnoldi_orth_cluster_kernel<T>, &lc) == cudaSuccess &&
              nclusters >= 1) {
            bc = c;
            break;
          }
          cudaGetLastError();
        }
      }
      if (bc > 0 && ceil_div(ceil_div(n, (int64_t)bc), 4) * 4 <= 4096) {
        if (getenv("DENSOLVE_ORTH_TRACE")) {
          DS_CUDA(cudaMalloc((void**)&orth_trace, sizeof(unsigned long long) * m * 2 * 16));
          DS_CUDA(cudaMemset(orth_trace, 0, sizeof(unsigned long long) * m * 2 * 16));
        }
        orth_cl = bc;
        orth_smem = (size_t)ceil_div(ceil_div(n, (int64_t)bc), 4) * 4 * sizeof(double);
        // the cluster sums the GEMV partials of its rows itself only while that is a small
        // read per CTA (C2: 128 KB); at n = 65536 (1.2 MB per CTA, ~40 us on 16 SMs) the
        // reduce kernel on every SM is faster
        orth_fold = ceil_div(n, (int64_t)bc) * gp.nchunks * (int64_t)sizeof(double) <= 256 * 1024;
        // each step's Givens deferred to the next step's cluster (off the GEMV -> cluster
        // chain) when the last warp of a CTA has no rows and the GEMV writes only its
        // partials (a step that runs past an estimate stop then leaves no trace: the next
        // GEMV writes scratch, the next cluster aborts before writing); DENSOLVE_ORTH_DEFER=0
        // disables
        static const bool defer_env = [] {
          const char* e = getenv("DENSOLVE_ORTH_DEFER");
          return !(e && e[0] == '0');
        }();
        orth_defer = defer_env && orth_fold && ceil_div(ceil_div(n, (int64_t)bc), 4) * 4 <= kOrthThreads - 32 ? 1 : 0;
      }
    }
  }
  // small n (C2): the wide-CTA GEMV (~one CTA per SM, one partial per row per CTA) feeds the
  // cluster, which then sums ~18 instead of ~64 partials per row; DENSOLVE_GEMV_WIDE=0 disables
  static const bool wide_env = [] {
    const char* e = getenv("DENSOLVE_GEMV_WIDE");
    return !(e && e[0] == '0');
  }();
  constexpr int kVecW = sizeof(T) == 8 ? 2 : 4;
  const GemvPlan wp = gemv_wide_plan(ctx, n, n, sizeof(T));
  const bool wide = wide_env && orth_cl > 0 && orth_fold && n <= 8192 && wp.part_bytes <= gp.part_bytes &&
                    reinterpret_cast<uintptr_t>(A) % 16 == 0 && lda % kVecW == 0;
  const int arn_rch = (int)std::min<int64_t>(4, ceil_div(arn_per, 32)) == 3 ? 4
                                                                           : (int)std::min<int64_t>(4, ceil_div(arn_per, 32));
  size_t need = gp.part_bytes + (size_t)ldv * (m + 1) * sizeof(T) + (size_t)n * sizeof(T) +
                (fused ? ((size_t)2 * arn_g * 128 + 256) * sizeof(uint64_t) + 256 : 0) +
                (size_t)(ldh * m * 2 + 3 * (m + 2) + m + 64) * sizeof(T) + (size_t)(2 * m + 2) * sizeof(double) +
                ((size_t)mdb * ldp + (size_t)rblocks * 3 + (size_t)vg * 2 + 512) * sizeof(double) +
                sizeof(GmDev) + 16 * 256;
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, need, &ws));
  Carver cv{(char*)ws};
  double* part = cv.take<double>(gp.part_bytes);
  T* V = cv.take<T>((size_t)ldv * (m + 1) * sizeof(T));
  T* r = cv.take<T>((size_t)n * sizeof(T));
  T* H = cv.take<T>((size_t)ldh * m * sizeof(T));
  T* Hraw = cv.take<T>((size_t)ldh * m * sizeof(T));
  T* g = cv.take<T>((size_t)(m + 2) * sizeof(T));
  T* cs = cv.take<T>((size_t)(m + 2) * sizeof(T));
  T* sn = cv.take<T>((size_t)(m + 2) * sizeof(T));
  T* y = cv.take<T>((size_t)std::max<int64_t>(m, 64) * sizeof(T));
  double* mpart = cv.take<double>((size_t)mdb * ldp * sizeof(double));
  double* red_a = cv.take<double>(((size_t)rblocks * 3 + 64) * sizeof(double));
  double* red_b = cv.take<double>(((size_t)std::max(vg, rblocks) * 2 + 64) * sizeof(double));
  double* hsave = cv.take<double>((size_t)std::max<int64_t>(m + 1, 64) * sizeof(double));
  double* est = cv.take<double>((size_t)std::max<int64_t>(m, 64) * sizeof(double));
  double* scal = cv.take<double>(64 * sizeof(double));
  GmDev* st = cv.take<GmDev>(sizeof(GmDev));
  uint64_t* arn_ll = fused ? cv.take<uint64_t>(((size_t)2 * arn_g * 128 + 256) * sizeof(uint64_t)) : nullptr;
  unsigned long long* arn_trace = nullptr;
  if (fused && getenv("DENSOLVE_GMRES_TRACE")) {
    DS_CUDA(cudaMalloc((void**)&arn_trace, 8 * 8 * arn_g));
    DS_CUDA(cudaMemsetAsync(arn_trace, 0, 8 * 8 * arn_g, ctx->stream));
  }

  double* hbuf = nullptr;
  DS_TRY(ctx_hostbuf(ctx, (size_t)(128 + m + 64) * sizeof(double), (void**)&hbuf));

  // ||b|| via nrm2 (krylov.py:87) and the plain ||b|| of relative_residual (core.py:207)
  // read back together with the first cycle's r = b - A x0 (one host synchronisation)
  int nb = 0;
  DS_TRY(ssq_launch<T>(ctx, n, b, red_b, &nb));
  DS_TRY(finish_ssq(ctx, red_b, nb, scal));
  int nb2 = 0;
  DS_TRY(dot_launch<T>(ctx, n, b, b, red_a, &nb2));
  DS_TRY(finish_sum(ctx, red_a, nb2, scal + 1));
  if (x != x0) DS_CUDA(cudaMemcpyAsync(x, x0, n * sizeof(T), cudaMemcpyDeviceToDevice, ctx->stream));
  {
    int rb = 0;
    DS_TRY(gemv_launch<T>(ctx, gp, A, lda, x, r, part, EPI_RESID, b, red_a, &rb));
    finish_resid_kernel<<<1, 256, 0, ctx->stream>>>(red_a, rb, scal + 2);
    count_launch(ctx);
  }
  DS_CUDA(cudaMemcpyAsync(hbuf, scal, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  const double bnorm = hbuf[0];
  const double bnorm_plain = sqrt(hbuf[1]);
  if (bnorm == 0.0) {
    set_error("||b|| = 0");
    return DS_EDEGRHS;
  }

  std::vector<double> history;
  std::vector<int64_t> cycles;
  int64_t total_it = 0;
  int breakdown = DS_BREAKDOWN_NONE;
  bool converged = false;
  std::vector<T> hV, hH;

  auto finish = [&](bool conv, int bd) {
    converged = conv;
    breakdown = bd;
  };

  int64_t residual_evals = 0;
  // r = b - A x and beta: the first cycle's were computed above with ||b||; every later
  // cycle's are the previous cycle's true residual (same x, same kernels), reused instead of
  // recomputed (still tallied as the reference's evaluation)
  double next_beta = hbuf[2];
  while (true) {
    // r = b - A x ; beta = nrm2(r)   (krylov.py:104-106)
    ++residual_evals;
    const double beta = next_beta;
    const double relres = beta / bnorm;
    if (total_it == 0) history.push_back(relres);
    if (relres <= tol) {
      finish(true, DS_BREAKDOWN_NONE);
      break;
    }
    if (total_it >= cap) {
      finish(false, DS_BREAKDOWN_NONE);
      break;
    }
    cycles.push_back(total_it);
    const double cycle_start_res = relres;

    // fresh cycle state (krylov.py:116-123); g, cs, sn are contiguous
    gm_cycle_start_kernel<T><<<vg, kT, 0, ctx->stream>>>(n, r, V, ldv * (m + 1), H, Hraw, ldh * m, g,
                                                         3 * (m + 2), est, beta, bnorm, m, st);
    count_launch(ctx);
    DS_CHECK_LAUNCH();

    // inner Arnoldi steps, enqueued in chunks behind the device gate
    // all m steps are enqueued at once (gated kernels after a stop are near-free): one
    // host synchronisation per cycle instead of one per chunk
    int64_t k = 0, chunk = m;
    int64_t stop_k = m;
    // one readback per chunk: the device state and the estimates together (pinned)
    GmDev* h_st = reinterpret_cast<GmDev*>(hbuf + 64);
    double* h_est = hbuf + 128;
    static_assert(sizeof(GmDev) <= 64 * sizeof(double), "GmDev staging slot");
    // m <= 64 without a sink: the tail (LS solve, x update, true residual) reads the stop step
    // on the device, so the cycle needs one host synchronisation (after the true residual)
    const bool dev_tail = !sink && m <= 64;
    while (true) {
      if (k > 0 && dev_tail) break;
      if (k > 0) {
        DS_CUDA(cudaMemcpyAsync(h_st, st, sizeof(GmDev), cudaMemcpyDeviceToHost, ctx->stream));
        DS_CUDA(cudaMemcpyAsync(h_est, est, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        DS_CUDA(cudaStreamSynchronize(ctx->stream));
        stop_k = h_st->stop_k;
        if (stop_k <= k || k >= m) break;
      }
      const int64_t kend = std::min<int64_t>(m, k + chunk);
      for (; k < kend; ++k) {
        const Gate gt{&st->stop_k, k};
        T* vk = V + k * ldv;
        T* w = V + (k + 1) * ldv;
        const int kc = (int)k + 1;
        if (orth_cl > 0) {  // streamed GEMV on every SM + one-cluster orthogonalisation
          if (!orth_fold)  // large n: the reduce kernel on every SM writes w
            DS_TRY(gemv_launch<T>(ctx, gp, A, lda, vk, w, part, EPI_STORE, nullptr, nullptr, nullptr, gt));
          else if (pdl_on && wide)
            DS_TRY(gemv_partial_wide_pdl_launch<T>(ctx, wp, A, lda, vk, part, gt));
          else if (pdl_on)
            DS_TRY(gemv_partial_pdl_launch<T>(ctx, gp, A, lda, vk, part, gt));
          else
            DS_TRY(gemv_launch<T>(ctx, gp, A, lda, vk, w, part, EPI_PARTIAL, nullptr, nullptr, nullptr, gt));
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3((unsigned)orth_cl);
          lc.blockDim = dim3(kOrthThreads);
          lc.dynamicSmemBytes = orth_smem;
          lc.stream = ctx->stream;
          cudaLaunchAttribute at[2];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = (unsigned)orth_cl;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[1].val.programmaticStreamSerializationAllowed = 1;
          lc.attrs = at;
          lc.numAttrs = pdl_on ? 2 : 1;
          const int passes = orth == DS_ORTH_CLASSICAL ? 1 : 2;
          DS_CUDA(cudaLaunchKernelEx(&lc, arnoldi_orth_cluster_kernel<T>, n, V, ldv, (int)k, passes, H, Hraw, ldh, g,
                                     cs, sn, est, st, tol, total_it, cap, gt,
                                     orth_fold ? (const double*)part : nullptr,
                                     (int64_t)(pdl_on && wide ? wp.nchunks : gp.nchunks),
                                     orth_trace, orth_defer));
          count_launch(ctx);
          continue;
        }
        if (fused) {
          const size_t arn_smem = (size_t)kc * arn_per * sizeof(T);
          static bool arn_attr[2] = {false, false};
          if (!arn_attr[sizeof(T) == 8]) {
            const int mx = (int)std::min<size_t>(ctx->smem_optin, 200 * 1024);
            DS_CUDA(cudaFuncSetAttribute(arnoldi_step_kernel<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            DS_CUDA(cudaFuncSetAttribute(arnoldi_step_kernel<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            DS_CUDA(cudaFuncSetAttribute(arnoldi_step_kernel<T, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            arn_attr[sizeof(T) == 8] = true;
          }
          ArnArgs aa;
          aa.n = n;
          aa.lda = lda;
          aa.ldv = ldv;
          aa.ldh = ldh;
          aa.total_before = total_it;
          aa.cap = cap;
          aa.k = (int)k;
          aa.passes = orth == DS_ORTH_CLASSICAL ? 1 : 2;
          aa.per = (int)arn_per;
          aa.seq = next_ll_epoch();
          aa.tol = tol;
          aa.ll = arn_ll;
          aa.est = est;
          aa.st = st;
          aa.trace = arn_trace;
          if (arn_rch == 1)
            arnoldi_step_kernel<T, 1><<<(unsigned)arn_g, kArnThreads, arn_smem, ctx->stream>>>(A, V, H, Hraw, g, cs, sn,
                                                                                       aa, gt);
          else if (arn_rch == 2)
            arnoldi_step_kernel<T, 2><<<(unsigned)arn_g, kArnThreads, arn_smem, ctx->stream>>>(A, V, H, Hraw, g, cs, sn,
                                                                                       aa, gt);
          else
            arnoldi_step_kernel<T, 4><<<(unsigned)arn_g, kArnThreads, arn_smem, ctx->stream>>>(A, V, H, Hraw, g, cs, sn,
                                                                                       aa, gt);
          count_launch(ctx);
          (void)vk;
          (void)w;
          (void)kc;
          continue;
        }
        DS_TRY(gemv_launch<T>(ctx, gp, A, lda, vk, w, part, EPI_STORE, nullptr, nullptr, nullptr,
                              gt));
        const int passes = orth == DS_ORTH_CLASSICAL ? 1 : 2;
        for (int ps = 0; ps < passes; ++ps) {
          multidot_kernel<T><<<mdb, kT, 0, ctx->stream>>>(n, V, ldv, kc, w, mpart, ldp, gt);
          cgs_update_kernel<T><<<vg, kT, (size_t)kc * sizeof(double), ctx->stream>>>(
              n, V, ldv, kc, w, mpart, ldp, mdb, H + k * ldh, hsave, ps,
              ps == passes - 1 ? red_b : nullptr, gt);
          count_launch(ctx, 2);
        }
        gm_step_finish_kernel<T><<<vg, kT, 0, ctx->stream>>>(n, w, red_b, vg, H, Hraw, ldh, g, cs,
                                                             sn, (int)k, est, st, tol, total_it,
                                                             cap, gt);
        count_launch(ctx);
      }
      if (orth_cl > 0 && orth_defer) {  // the last executed step's Givens
        gm_givens_tail_kernel<T><<<1, 32, 0, ctx->stream>>>(kend, Hraw, H, ldh, g, cs, sn, est, st, tol);
        count_launch(ctx);
      }
      DS_CHECK_LAUNCH();
      chunk = std::min<int64_t>(chunk * 2, 32);
    }
    int inner = (int)m;
    bool happy = false;
    if (!dev_tail) {
      const GmDev hst = *h_st;  // read by the chunk loop's final readback
      inner = (int)std::min<int64_t>(hst.stop_k, m);
      happy = hst.happy != 0;
      for (int i = 0; i < inner; ++i) history.push_back(h_est[i]);
      total_it += inner;
    }

    // cycle end: y = H^-1 g ; x += V y   (krylov.py:166-167).  dev_tail: the stop step is read
    // on the device and the update runs over all m columns with y = 0 past it (one column
    // chunk for m <= 64, the same order of accumulation)
    if (dev_tail)
      gm_lsq_kernel<T><<<1, 256, 0, ctx->stream>>>(H, ldh, g, -(int)m, y, st);
    else if (inner <= 64)
      gm_lsq_kernel<T><<<1, 256, 0, ctx->stream>>>(H, ldh, g, inner, y, st);
    else
      gm_lsq_global_kernel<T><<<1, 32, 0, ctx->stream>>>(H, ldh, g, inner, y, st);
    count_launch(ctx);
    {
      const GemvPlan gp2 = gemv_plan(ctx, n, inner, sizeof(T));
      if (gp2.part_bytes > gp.part_bytes) {
        set_error("internal: gemv workspace");
        return DS_ECUDA;
      }
      DS_TRY(gemv_launch<T>(ctx, gp2, V, ldv, y, x, part, EPI_AXPY_INTO, nullptr, nullptr,
                            nullptr));
    }
    auto singular_check = [&]() -> int {
      if (h_st->status == DS_ESINGULAR) {
        set_error("zero diagonal at row %lld", (long long)h_st->bad_row);
        info->error_index = h_st->bad_row;
        return DS_ESINGULAR;
      }
      return DS_OK;
    };
    if (sink) {  // the sink sees V / H only for a nonsingular cycle
      DS_CUDA(cudaMemcpyAsync(h_st, st, sizeof(GmDev), cudaMemcpyDeviceToHost, ctx->stream));
      DS_CUDA(cudaStreamSynchronize(ctx->stream));
      DS_TRY(singular_check());
    }
    if (sink) {  // krylov.py:168-169
      hV.resize((size_t)n * (m + 1));
      hH.resize((size_t)ldh * m);
      DS_CUDA(cudaMemcpy2DAsync(hV.data(), n * sizeof(T), V, ldv * sizeof(T), n * sizeof(T), m + 1,
                                cudaMemcpyDeviceToHost, ctx->stream));
      DS_CUDA(cudaMemcpyAsync(hH.data(), Hraw, (size_t)ldh * m * sizeof(T),
                              cudaMemcpyDeviceToHost, ctx->stream));
      DS_CUDA(cudaStreamSynchronize(ctx->stream));
      sink(sink_user, hV.data(), hH.data(), inner, beta);
    }
    // true residual (core.relative_residual, uncounted A @ x; krylov.py:171)
    {
      int rb2 = 0;
      DS_TRY(gemv_launch<T>(ctx, gp, A, lda, x, r, part, EPI_RESID, b, red_a, &rb2));
      finish_resid_kernel<<<1, 256, 0, ctx->stream>>>(red_a, rb2, scal + 4);
      count_launch(ctx);
      DS_CUDA(cudaMemcpyAsync(hbuf, scal + 4, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                              ctx->stream));
      DS_CUDA(cudaMemcpyAsync(h_st, st, sizeof(GmDev), cudaMemcpyDeviceToHost, ctx->stream));
      if (dev_tail)
        DS_CUDA(cudaMemcpyAsync(h_est, est, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      DS_CUDA(cudaStreamSynchronize(ctx->stream));
      if (dev_tail) {
        inner = (int)std::min<int64_t>(h_st->stop_k, m);
        happy = h_st->happy != 0;
        for (int i = 0; i < inner; ++i) history.push_back(h_est[i]);
        total_it += inner;
      }
      DS_TRY(singular_check());  // the least-squares solve's zero-diagonal flag (krylov.py:166)
    }
    next_beta = hbuf[0];
    const double true_res = sqrt(hbuf[1]) / bnorm_plain;
    if (happy || history.back() <= tol || true_res <= tol) {  // krylov.py:172-175
      history.back() = true_res;
      if (true_res <= tol || happy) {
        finish(true, happy ? DS_BREAKDOWN_HAPPY : DS_BREAKDOWN_NONE);
        break;
      }
    }
    if (total_it >= cap) {  // krylov.py:176-178
      history.back() = true_res;
      finish(false, DS_BREAKDOWN_NONE);
      break;
    }
    if (inner == m && true_res >= cycle_start_res * (1.0 - u)) {  // stagnation :180-182
      history.back() = true_res;
      finish(false, DS_BREAKDOWN_NONE);
      break;
    }
  }
  if (orth_trace) {  // last cycle's per-step phase durations (ns), mean over its steps
    std::vector<unsigned long long> h((size_t)m * 2 * 16);
    DS_CUDA(cudaMemcpy(h.data(), orth_trace, h.size() * 8, cudaMemcpyDeviceToHost));
    cudaFree(orth_trace);
    for (int rk = 0; rk < 2; ++rk) {
      double d[13] = {};
      int cnt = 0;
      for (int64_t kk = 0; kk < m; ++kk) {
        const unsigned long long* t = h.data() + ((size_t)kk * 2 + rk) * 16;
        if (t[0] == 0 || t[12] == 0 && rk == 0) continue;
        ++cnt;
        for (int z = 1; z <= (rk == 0 ? 12 : 11); ++z) d[z] += (double)(t[z] - t[z - 1]);
      }
      double period = 0.0, outside = 0.0;
      int np_ = 0;
      for (int64_t kk = 0; kk + 1 < m; ++kk) {
        const unsigned long long* t = h.data() + ((size_t)kk * 2) * 16;
        const unsigned long long* t2 = h.data() + ((size_t)(kk + 1) * 2) * 16;
        if (t[0] == 0 || t2[0] == 0 || t[12] == 0) continue;
        period += (double)(t2[0] - t[0]);
        outside += (double)(t2[0] - t[12]);
        ++np_;
      }
      fprintf(stderr, "[orth trace] %s, %d steps, ns/step: load %.0f | p0 dot %.0f csync %.0f red %.0f upd %.0f | "
              "p1 dot %.0f csync %.0f red %.0f upd %.0f | norm+2 csync %.0f | store %.0f | givens %.0f || step period "
              "%.0f, between orth kernels (GEMV + launch gaps) %.0f\n",
              rk == 0 ? "rank 0" : "last rank", cnt, d[1] / cnt, d[2] / cnt, d[3] / cnt, d[4] / cnt, d[5] / cnt,
              d[6] / cnt, d[7] / cnt, d[8] / cnt, d[9] / cnt, d[10] / cnt, d[11] / cnt, d[12] / cnt,
              np_ ? period / np_ : 0.0, np_ ? outside / np_ : 0.0);
    }
  }
  if (arn_trace) {
    std::vector<unsigned long long> h(8 * arn_g);
    DS_CUDA(cudaMemcpy(h.data(), arn_trace, 8 * 8 * arn_g, cudaMemcpyDeviceToHost));
    cudaFree(arn_trace);
    double mean[8] = {}, mx[8] = {};
    for (int64_t b = 0; b < arn_g; ++b)
      for (int z = 1; z < 7; ++z) {
        mean[z] += (double)h[b * 8 + z] / arn_g / std::max<int64_t>(total_it, 1);
        mx[z] = std::max(mx[z], (double)h[b * 8 + z] / std::max<int64_t>(total_it, 1));
      }
    fprintf(stderr, "[gmres trace] n=%lld G=%lld per=%lld steps=%lld cycles/step mean(max): gemv %.0f(%.0f) "
            "vstage %.0f(%.0f) pass0 %.0f(%.0f) pass1 %.0f(%.0f) norm %.0f(%.0f)\n", (long long)n, (long long)arn_g,
            (long long)arn_per, (long long)total_it, mean[1], mx[1], mean[2], mx[2], mean[3], mx[3], mean[4], mx[4],
            mean[5], mx[5]);
  }
  const int64_t hl = std::min<int64_t>((int64_t)history.size(), hist_cap);
  for (int64_t i = 0; i < hl; ++i) h_hist[i] = history[i];
  const int64_t cl = std::min<int64_t>((int64_t)cycles.size(), cycles_cap);
  for (int64_t i = 0; i < cl; ++i) h_cycles[i] = cycles[i];
  info->converged = converged;
  info->breakdown = breakdown;
  info->iterations = total_it;
  info->final_relative_residual = history.back();
  info->history_len = (int64_t)history.size();
  info->cycles_len = (int64_t)cycles.size();
  info->residual_evals = residual_evals;
  info->kernel_launches = ctx->launches - launches0;
  return DS_OK;
}


// ============================================================================
// BiCGSTAB  (krylov.bicgstab_solve, krylov.py:185-253)
//
// One iteration = two half-iterations, each with its own gate index:
//   half 2k   : p = r + beta (p - omega v) ; v = A p (+ r0hat'v) ; s = r - alpha v
//               (+ ssq s) ; early exit x += alpha p, r = s when ||s||/||b|| <= tol
//   half 2k+1 : t = A s (+ t's, t't) ; x = (x + alpha p) + omega s ;
//               r = s - omega t (+ r0hat'r, ssq r) ; rho, history, stop
// The device stop word counts completed half-iterations: breakdown at the top
// of iteration k or inside it -> 2k, early exit -> 2k+1, normal end -> 2k+2;
// iterations = ceil(stop / 2), exactly the reference's `it`.
// ============================================================================
struct BiDev {
  int64_t stop_h;     // half-iteration index at which the loop stops
  int32_t breakdown;  // DS_BREAKDOWN_NONE / DS_BREAKDOWN_RHO / DS_BREAKDOWN_OMEGA
  int32_t stage;      // where the loop stopped (for the logical counter tally)
  double bnorm, r0n, rnorm;
  double rho, rho_prev, alpha, omega;
};
enum BiStage : int32_t {
  BI_RUN = 0, BI_RHO_TOP = 1, BI_RV_ZERO = 2, BI_OMEGA = 3, BI_EARLY = 4, BI_DONE = 5
};

// setup (krylov.py:196-208): red = EPI_RESID partials of r0 = b - A x0
__global__ void bi_init_kernel(const double* red, int nblk, BiDev* st, double* hist, double tol,
                               int64_t cap) {
  __shared__ double sm[64];
  Ssq q{0.0, 0.0};
  double s2 = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    q = ssq_merge(q, Ssq{red[2 * i], red[2 * i + 1]});
    s2 += red[2 * nblk + i];
  }
  q = block_ssq(q, sm);
  s2 = block_sum(s2, sm);
  if (threadIdx.x == 0) {
    const double res = ssq_norm(q.scale, q.ssq) / st->bnorm;  // nrm2(r)/bnorm (:206)
    hist[0] = res;
    st->r0n = sqrt(s2);           // np.linalg.norm(r0hat) (:199)
    st->rho = s2;                 // dot(r0hat, r) with r0hat = r (:201)
    st->rho_prev = 1.0;
    st->alpha = 1.0;
    st->omega = 1.0;
    st->rnorm = res * st->bnorm;  // (:209)
    st->breakdown = DS_BREAKDOWN_NONE;
    st->stage = BI_RUN;
    st->stop_h = (res > tol && 0 < cap) ? 2 * cap : 0;
  }
}

// top of iteration k: rho-breakdown test, beta, p = axpy(beta, axpy(-omega, v, p), r)
template <typename T>
__global__ void __launch_bounds__(kT)
    bi_p_kernel(int64_t n, T* __restrict__ p, const T* __restrict__ v, const T* __restrict__ r,
                BiDev* st, double u, Gate gate) {
  if (gated(gate)) return;
  const double rho = st->rho;
  if (fabs(rho) < u * st->r0n * st->rnorm) {  // krylov.py:213-215
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->breakdown = DS_BREAKDOWN_RHO;
      st->stage = BI_RHO_TOP;
      st->stop_h = gate.k;
    }
    return;
  }
  const double beta = (rho / st->rho_prev) * (st->alpha / st->omega);  // :216
  const T bt = (T)beta, no = (T)(-st->omega);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T q = add_rn(p[i], mul_rn(no, v[i]));
    p[i] = add_rn(r[i], mul_rn(bt, q));
  }
}

// rv = r0hat'v ; alpha = rho/rv ; s = r - alpha v ; ssq(s) partials  (krylov.py:218-225)
template <typename T>
__global__ void __launch_bounds__(kT)
    bi_s_kernel(int64_t n, T* __restrict__ s, const T* __restrict__ r, const T* __restrict__ v,
                const double* __restrict__ red_rv, int nblk_rv, BiDev* st,
                double* __restrict__ red_out, Gate gate) {
  if (gated(gate)) return;
  __shared__ double sm[64];
  const double rv = reduce_sum_partials(red_rv, nblk_rv, sm);
  if (rv == 0.0) {  // :220-222
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->breakdown = DS_BREAKDOWN_RHO;
      st->stage = BI_RV_ZERO;
      st->stop_h = gate.k;
    }
    return;
  }
  const double alpha = st->rho / rv;
  const T na = (T)(-alpha);
  Ssq q{0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T si = add_rn(r[i], mul_rn(na, v[i]));
    s[i] = si;
    q = ssq_add(q, (double)si);
  }
  q = block_ssq(q, sm);
  if (threadIdx.x == 0) {
    red_out[2 * blockIdx.x] = q.scale;
    red_out[2 * blockIdx.x + 1] = q.ssq;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) st->alpha = alpha;
}

// ||s||/||b|| <= tol: x = axpy(alpha, p, x), r = s, history, stop (krylov.py:224-230)
template <typename T>
__global__ void __launch_bounds__(kT)
    bi_early_kernel(int64_t n, T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p,
                    const T* __restrict__ s, const double* __restrict__ red_s, int nblk,
                    BiDev* st, double* hist, double tol, Gate gate) {
  if (gated(gate)) return;
  __shared__ double sm[64];
  Ssq q{0.0, 0.0};
  for (int i = threadIdx.x; i < nblk; i += blockDim.x)
    q = ssq_merge(q, Ssq{red_s[2 * i], red_s[2 * i + 1]});
  q = block_ssq(q, sm);
  const double snorm = ssq_norm(q.scale, q.ssq);
  if (!(snorm / st->bnorm <= tol)) return;
  const T a = (T)st->alpha;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = add_rn(x[i], mul_rn(a, p[i]));
    r[i] = s[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t k = gate.k / 2;
    hist[k + 1] = snorm / st->bnorm;
    st->stage = BI_EARLY;
    st->stop_h = gate.k + 1;
  }
}

// omega = t's / t't ; x = axpy(omega, s, axpy(alpha, p, x)) ; r = axpy(-omega, t, s);
// partials of r0hat'r and ssq(r)   (krylov.py:230-245)
template <typename T>
__global__ void __launch_bounds__(kT)
    bi_xr_kernel(int64_t n, T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p,
                 const T* __restrict__ s, const T* __restrict__ t, const T* __restrict__ r0hat,
                 const double* __restrict__ red_t, int nblk_t, BiDev* st, double u,
                 double* __restrict__ red_out, Gate gate) {
  if (gated(gate)) return;
  __shared__ double sm[64];
  double ts = 0.0, tt = 0.0;
  for (int i = threadIdx.x; i < nblk_t; i += blockDim.x) {
    ts += red_t[i];
    tt += red_t[nblk_t + i];
  }
  ts = block_sum(ts, sm);
  tt = block_sum(tt, sm);
  const double omega = tt == 0.0 ? 0.0 : ts / tt;
  if (tt == 0.0 || fabs(omega) < u) {  // :232-238
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->breakdown = DS_BREAKDOWN_OMEGA;
      st->stage = BI_OMEGA;
      st->stop_h = gate.k - 1;  // = 2k: the iteration does not count
    }
    return;
  }
  const T a = (T)st->alpha, om = (T)omega, nom = (T)(-omega);
  Ssq q{0.0, 0.0};
  double d = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T x1 = add_rn(x[i], mul_rn(a, p[i]));
    const T si = s[i];
    x[i] = add_rn(x1, mul_rn(om, si));
    const T ri = add_rn(si, mul_rn(nom, t[i]));
    r[i] = ri;
    d = fma((double)r0hat[i], (double)ri, d);
    q = ssq_add(q, (double)ri);
  }
  q = block_ssq(q, sm);
  d = block_sum(d, sm);
  if (threadIdx.x == 0) {
    red_out[blockIdx.x] = d;
    red_out[gridDim.x + 2 * blockIdx.x] = q.scale;
    red_out[gridDim.x + 2 * blockIdx.x + 1] = q.ssq;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) st->omega = omega;
}

// rho_prev, rho = rho, r0hat'r ; rnorm = nrm2(r) ; res ; history ; stop  (:240-245, loop test :212)
__global__ void bi_finish_kernel(const double* red, int nblk, BiDev* st, double* hist, double tol,
                                 int64_t cap, Gate gate) {
  if (gated(gate)) return;
  __shared__ double sm[64];
  double d = 0.0;
  Ssq q{0.0, 0.0};
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    d += red[i];
    q = ssq_merge(q, Ssq{red[nblk + 2 * i], red[nblk + 2 * i + 1]});
  }
  d = block_sum(d, sm);
  q = block_ssq(q, sm);
  if (threadIdx.x == 0) {
    const int64_t k = gate.k / 2;
    st->rho_prev = st->rho;
    st->rho = d;
    const double rnorm = ssq_norm(q.scale, q.ssq);
    st->rnorm = rnorm;
    const double res = rnorm / st->bnorm;
    hist[k + 1] = res;
    if (!(res > tol) || k + 1 >= cap) {
      st->stage = BI_DONE;
      st->stop_h = gate.k + 1;
    }
  }
}

template <typename T>
int bicgstab_impl(ds_ctx* ctx, int64_t n, const T* A, int64_t lda, const T* b, const T* x0, T* x,
                  double tol, int64_t cap, double* h_hist, int64_t hist_cap, ds_solve_info* info) {
  const int64_t launches0 = ctx->launches;
  const double u = (sizeof(T) == 8 ? 1.1102230246251565e-16 : 5.960464477539063e-08);
  const GemvPlan gp = gemv_plan(ctx, n, n, sizeof(T));
  const int rblocks = (int)ceil_div(std::max<int64_t>(n, 1), 256);
  const int vg = vec_grid(ctx, n);
  size_t need = gp.part_bytes + 256 + ((size_t)n * sizeof(T) + 256) * 6 +
                ((size_t)rblocks * 3 + 64) * sizeof(double) * 2 +
                ((size_t)vg * 3 + 64) * sizeof(double) * 2 + (size_t)(cap + 2) * sizeof(double) +
                sizeof(BiDev) + 8 * 256;
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, need, &ws));
  Carver cv{(char*)ws};
  double* part = cv.take<double>(gp.part_bytes);
  T* r = cv.take<T>((size_t)n * sizeof(T));
  T* r0hat = cv.take<T>((size_t)n * sizeof(T));
  T* p = cv.take<T>((size_t)n * sizeof(T));
  T* v = cv.take<T>((size_t)n * sizeof(T));
  T* s = cv.take<T>((size_t)n * sizeof(T));
  T* t = cv.take<T>((size_t)n * sizeof(T));
  double* red_a = cv.take<double>(((size_t)rblocks * 3 + 64) * sizeof(double));
  double* red_b = cv.take<double>(((size_t)vg * 3 + 64) * sizeof(double));
  double* red_c = cv.take<double>(((size_t)vg * 3 + 64) * sizeof(double));
  double* hist = cv.take<double>((size_t)(cap + 2) * sizeof(double));
  BiDev* st = cv.take<BiDev>(sizeof(BiDev));
  double* scal = cv.take<double>(64);

  // ||b|| (krylov.py:195 -> _rhs_norm :29-33)
  int nb = 0;
  DS_TRY(ssq_launch<T>(ctx, n, b, red_b, &nb));
  DS_TRY(finish_ssq(ctx, red_b, nb, scal));
  double bnorm = 0;
  DS_CUDA(cudaMemcpyAsync(&bnorm, scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (bnorm == 0.0) {
    set_error("||b|| = 0");
    return DS_EDEGRHS;
  }
  BiDev init{};
  init.bnorm = bnorm;
  DS_CUDA(cudaMemcpyAsync(st, &init, sizeof(BiDev), cudaMemcpyHostToDevice, ctx->stream));
  // x = x0.copy(); r = axpy(-1, A x, b); r0hat = r; p = v = 0  (krylov.py:196-203)
  if (x != x0) DS_CUDA(cudaMemcpyAsync(x, x0, n * sizeof(T), cudaMemcpyDeviceToDevice, ctx->stream));
  int rb = 0;
  DS_TRY(gemv_launch<T>(ctx, gp, A, lda, x, r, part, EPI_RESID, b, red_a, &rb));
  bi_init_kernel<<<1, 256, 0, ctx->stream>>>(red_a, rb, st, hist, tol, cap);
  count_launch(ctx);
  DS_CUDA(cudaMemcpyAsync(r0hat, r, n * sizeof(T), cudaMemcpyDeviceToDevice, ctx->stream));
  DS_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), ctx->stream));
  DS_CUDA(cudaMemsetAsync(v, 0, n * sizeof(T), ctx->stream));
  DS_CHECK_LAUNCH();

  int64_t* h_stop = nullptr;
  DS_TRY(ctx_hostbuf(ctx, 64, (void**)&h_stop));
  int64_t k = 0, chunk = 2;
  while (true) {
    DS_CUDA(cudaMemcpyAsync(h_stop, &st->stop_h, sizeof(int64_t), cudaMemcpyDeviceToHost,
                            ctx->stream));
    DS_CUDA(cudaStreamSynchronize(ctx->stream));
    const int64_t stop_h = *h_stop;
    if (stop_h <= 2 * k || k >= cap) break;
    const int64_t kend = std::min<int64_t>(cap, k + chunk);
    for (; k < kend; ++k) {
      const Gate g0{&st->stop_h, 2 * k}, g1{&st->stop_h, 2 * k + 1};
      bi_p_kernel<T><<<vg, kT, 0, ctx->stream>>>(n, p, v, r, st, u, g0);
      count_launch(ctx);
      int rb1 = 0, rb2 = 0;
      DS_TRY(gemv_launch<T>(ctx, gp, A, lda, p, v, part, EPI_DOT, r0hat, red_a, &rb1, g0));
      bi_s_kernel<T><<<vg, kT, 0, ctx->stream>>>(n, s, r, v, red_a, rb1, st, red_b, g0);
      bi_early_kernel<T><<<vg, kT, 0, ctx->stream>>>(n, x, r, p, s, red_b, vg, st, hist, tol, g0);
      count_launch(ctx, 2);
      DS_TRY(gemv_launch<T>(ctx, gp, A, lda, s, t, part, EPI_DOT2, s, red_a, &rb2, g1));
      bi_xr_kernel<T><<<vg, kT, 0, ctx->stream>>>(n, x, r, p, s, t, r0hat, red_a, rb2, st, u,
                                                  red_c, g1);
      bi_finish_kernel<<<1, 256, 0, ctx->stream>>>(red_c, vg, st, hist, tol, cap, g1);
      count_launch(ctx, 2);
    }
    DS_CHECK_LAUNCH();
    chunk = std::min<int64_t>(chunk * 2, 64);
  }
  BiDev hst;
  DS_CUDA(cudaMemcpyAsync(&hst, st, sizeof(BiDev), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  const int64_t iters = std::min<int64_t>((hst.stop_h + 1) / 2, cap);
  const int64_t hl = std::min<int64_t>(iters + 1, hist_cap);
  std::vector<double> hh((size_t)iters + 1);
  DS_CUDA(cudaMemcpyAsync(hh.data(), hist, (iters + 1) * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_hist)
    for (int64_t i = 0; i < hl; ++i) h_hist[i] = hh[i];
  const double res = hh[iters];
  info->iterations = iters;
  info->history_len = hl;
  info->final_relative_residual = res;
  info->breakdown = hst.breakdown;
  info->converged = res <= tol && hst.breakdown == DS_BREAKDOWN_NONE;  // krylov.py:246
  info->error_index = hst.stage;  // loop exit stage (BiStage), for the logical counter tally
  info->kernel_launches = ctx->launches - launches0;
  return DS_OK;
}

}  // namespace ds

using namespace ds;

extern "C" {

int ds_cg(ds_ctx* ctx, int dtype, int64_t n, const void* A, int64_t lda, const void* b,
          const void* x0, void* x, double tol, int64_t max_it, int check_sym, double* h_hist,
          int64_t hist_cap, ds_solve_info* info) {
  DS_ENTER(ctx);
  *info = ds_solve_info{};
  info->error_index = -1;
  if (n <= 0) {
    set_error("matrix must be square and non-empty, got n=%lld", (long long)n);
    return DS_EDIM;
  }
  if (!(tol > 0)) {
    set_error("tolerance must be > 0");
    return DS_EINVAL;
  }
  if (max_it < 1) {
    set_error("max_iterations must be >= 1");
    return DS_EINVAL;
  }
  DS_DISPATCH(dtype, T,
              return cg_impl<T>(ctx, n, (const T*)A, lda, (const T*)b, (const T*)x0, (T*)x, tol,
                                max_it, check_sym, h_hist, hist_cap, info));
}

int ds_gmres(ds_ctx* ctx, int dtype, int64_t n, const void* A, int64_t lda, const void* b,
             const void* x0, void* x, double tol, int64_t max_it, int64_t restart_m, int orth,
             double* h_hist, int64_t hist_cap, int64_t* h_cycles, int64_t cycles_cap,
             ds_sink_fn sink, void* sink_user, ds_solve_info* info) {
  DS_ENTER(ctx);
  *info = ds_solve_info{};
  info->error_index = -1;
  if (n <= 0) {
    set_error("matrix must be square and non-empty, got n=%lld", (long long)n);
    return DS_EDIM;
  }
  if (!(tol > 0) || restart_m < 1 || max_it < 1 ||
      (orth != DS_ORTH_MODIFIED && orth != DS_ORTH_CLASSICAL)) {
    set_error("invalid GMRES configuration");
    return DS_EINVAL;
  }
  DS_DISPATCH(dtype, T,
              return gmres_impl<T>(ctx, n, (const T*)A, lda, (const T*)b, (const T*)x0, (T*)x, tol,
                                   max_it, restart_m, orth, h_hist, hist_cap, h_cycles, cycles_cap,
                                   sink, sink_user, info));
}

int ds_bicgstab(ds_ctx* ctx, int dtype, int64_t n, const void* A, int64_t lda, const void* b,
                const void* x0, void* x, double tol, int64_t max_it, double* h_hist,
                int64_t hist_cap, ds_solve_info* info) {
  DS_ENTER(ctx);
  *info = ds_solve_info{};
  info->error_index = -1;
  if (n <= 0) {
    set_error("matrix must be square and non-empty, got n=%lld", (long long)n);
    return DS_EDIM;
  }
  if (!(tol > 0) || max_it < 1) {
    set_error("invalid BiCGSTAB configuration");
    return DS_EINVAL;
  }
  DS_DISPATCH(dtype, T,
              return bicgstab_impl<T>(ctx, n, (const T*)A, lda, (const T*)b, (const T*)x0, (T*)x,
                                      tol, max_it, h_hist, hist_cap, info));
}

}  // extern "C"
