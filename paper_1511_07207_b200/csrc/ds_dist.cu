// ds_dist.cu — building blocks of the multi-GPU (one process per GPU) paths.
//
// Row-sharded CG / GMRES: every rank owns a contiguous block of
// rows of A and of every vector.  The only exchanges are an all-gather of the
// iterate fed to the GEMV and all-gathers of per-rank reduction partials; the
// partials are combined on the device IN RANK ORDER by every rank, so all ranks
// compute bitwise-identical scalars and take identical stopping decisions.
// These entry points are the per-rank compute between those collectives; the
// collectives themselves are issued by the host driver
// (paper_1511_07207_b200/distributed.py) through torch.distributed (NCCL).
//
// 1-D block-cyclic LU: ds_lu_panel factors a tall (m x w) panel in place with
// the reference's b-blocking (the owner's step), ds_laswp applies a pivot range
// to a set of columns (every rank), TRSM/GEMM are the op-contract kernels.
#include <cuda_runtime.h>

#include <algorithm>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

constexpr int kDT = 256;

// (sum x^2, scale, ssq) partials of a local vector, then one record per call
template <typename T>
__global__ void __launch_bounds__(kDT) vec_parts_kernel(int64_t n, const T* __restrict__ x, double* red) {
  __shared__ double sm[64];
  double s2 = 0.0;
  Ssq q{0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)x[i];
    s2 = fma(v, v, s2);
    q = ssq_add(q, v);
  }
  s2 = block_sum(s2, sm);
  q = block_ssq(q, sm);
  if (threadIdx.x == 0) {
    red[3 * blockIdx.x] = s2;
    red[3 * blockIdx.x + 1] = q.scale;
    red[3 * blockIdx.x + 2] = q.ssq;
  }
}

__global__ void parts3_finish_kernel(const double* red, int nblk, double* out) {
  __shared__ double sm[64];
  double s2 = 0.0;
  Ssq q{0.0, 0.0};
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    s2 += red[3 * i];
    q = ssq_merge(q, Ssq{red[3 * i + 1], red[3 * i + 2]});
  }
  s2 = block_sum(s2, sm);
  q = block_ssq(q, sm);
  if (threadIdx.x == 0) {
    out[0] = s2;
    out[1] = q.scale;
    out[2] = q.ssq;
  }
}

// rank-ordered combination of nranks (s2, scale, ssq) records
__device__ __forceinline__ void combine3(const double* parts, int nranks, double& s2, double& nrm) {
  s2 = 0.0;
  Ssq q{0.0, 0.0};
  for (int r = 0; r < nranks; ++r) {
    s2 += parts[3 * r];
    q = ssq_merge(q, Ssq{parts[3 * r + 1], parts[3 * r + 2]});
  }
  nrm = ssq_norm(q.scale, q.ssq);
}

// state layout (doubles), see include/densolve_b200.h DS_SHARD_*
enum { ST_RS = 0, ST_BNORM = 1, ST_STATUS = 2, ST_STOP = 3, ST_BAD = 4, ST_RES = 5, ST_STOP64 = 8 };
// the shard state holds >= 16 doubles; slot ST_STOP64 mirrors ST_STOP as an int64 Gate word

__global__ void cg_shard_init_kernel(const double* bparts, const double* rparts, int nranks, double* st,
                                     double* hist, double tol, int64_t cap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double bs2, bn, rs, rn;
  combine3(bparts, nranks, bs2, bn);
  combine3(rparts, nranks, rs, rn);
  const double res = rn / bn;
  st[ST_RS] = rs;
  st[ST_BNORM] = bn;
  st[ST_STATUS] = 0.0;
  st[ST_STOP] = (res > tol && 0 < cap) ? (double)cap : 0.0;
  st[ST_RES] = res;
  hist[0] = res;
}

// pAp = sum_r pap_parts[r] (rank order); alpha = rs/pAp; x += alpha p; r -= alpha Ap
template <typename T>
__global__ void __launch_bounds__(kDT)
    cg_shard_update_kernel(int64_t n, int nranks, const double* __restrict__ pap_parts, double* st, int64_t k,
                           T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p,
                           const T* __restrict__ Ap, double* red) {
  if (st[ST_STOP] <= (double)k) return;
  __shared__ double sm[64];
  double pAp = 0.0;
  for (int q = 0; q < nranks; ++q) pAp += pap_parts[q];
  if (pAp <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st[ST_STATUS] = (double)DS_ENOTSPD;
      st[ST_BAD] = pAp;
    }
    return;
  }
  const double alpha = st[ST_RS] / pAp;
  const T a = (T)alpha, na = (T)(-alpha);
  double s2 = 0.0;
  Ssq q{0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = add_rn(x[i], mul_rn(a, p[i]));
    const T ri = add_rn(r[i], mul_rn(na, Ap[i]));
    r[i] = ri;
    const double v = (double)ri;
    s2 = fma(v, v, s2);
    q = ssq_add(q, v);
  }
  s2 = block_sum(s2, sm);
  q = block_ssq(q, sm);
  if (threadIdx.x == 0) {
    red[3 * blockIdx.x] = s2;
    red[3 * blockIdx.x + 1] = q.scale;
    red[3 * blockIdx.x + 2] = q.ssq;
  }
}

// rs_new, ||r|| from rank-ordered parts; beta; p = r + beta p; history; stop word
template <typename T>
__global__ void __launch_bounds__(kDT)
    cg_shard_finish_kernel(int64_t n, int nranks, const double* __restrict__ parts, double* st, int64_t k,
                           const T* __restrict__ r, T* __restrict__ p, double* hist, double tol, int64_t cap) {
  if (st[ST_STOP] <= (double)k || st[ST_STATUS] != 0.0) return;
  double rs_new, nrm;
  combine3(parts, nranks, rs_new, nrm);
  const double beta = rs_new / st[ST_RS];
  const T bt = (T)beta;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = add_rn(r[i], mul_rn(bt, p[i]));
  // st[ST_RS] is advanced by cg_shard_commit_kernel, launched after this kernel
}

__global__ void cg_shard_commit_kernel(int nranks, const double* __restrict__ parts, double* st, int64_t k,
                                       double* hist, double tol, int64_t cap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (st[ST_STOP] <= (double)k || st[ST_STATUS] != 0.0) {
    if (st[ST_STATUS] != 0.0 && st[ST_STOP] > (double)k) st[ST_STOP] = (double)k;
    return;
  }
  double rs_new, nrm;
  combine3(parts, nranks, rs_new, nrm);
  const double res = nrm / st[ST_BNORM];
  st[ST_RS] = rs_new;
  st[ST_RES] = res;
  hist[k + 1] = res;
  if (!(res > tol) || k + 1 >= cap) st[ST_STOP] = (double)(k + 1);
}

// ---------------------------------------------------------------------------
// GMRES shard steps
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kDT)
    multidot_dev_kernel(int64_t n, const T* __restrict__ V, int64_t ldv, int kc, const T* __restrict__ w,
                        double* __restrict__ part /* [grid][64] */) {
  __shared__ double sm[kDT / 32][64];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc[1];
  (void)acc;
  for (int j = 0; j < kc; ++j) {
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      s = fma((double)V[i + (int64_t)j * ldv], (double)w[i], s);
    s = warp_sum(s);
    if (lane == 0) sm[wid][j] = s;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < kc; j += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < kDT / 32; ++q) s += sm[q][j];
    part[(int64_t)blockIdx.x * 64 + j] = s;
  }
}

// one warp per dot product: the lanes load the block partials of column j together
// (strided by 32, a fixed order) and combine them with a fixed shuffle tree, instead of
// one thread walking all nblk partials through dependent loads (~23 -> ~4 us at nblk 256)
__global__ void multidot_finish_kernel(const double* part, int nblk, int kc, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = w; j < kc; j += nw) {
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += part[(int64_t)b * 64 + j];
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
}

// w -= sum_j h_j V[:,j] with h_j = sum_r parts[r*kc + j] (rank order); Hcol/hsave as in
// the single-GPU kernel; emits (s2, scale, ssq) partials of the updated w
template <typename T>
__global__ void __launch_bounds__(kDT)
    cgs_update_shard_kernel(int64_t n, const T* __restrict__ V, int64_t ldv, int kc, T* __restrict__ w,
                            int nranks, const double* __restrict__ parts, T* Hcol, double* hsave, int pass,
                            double* red, const double* st, int64_t k) {
  if (st[ST_STOP] <= (double)k) return;
  __shared__ double hs[64];
  __shared__ double sm[64];
  for (int j = threadIdx.x; j < kc; j += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += parts[r * kc + j];
    hs[j] = s;
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < kc; j += blockDim.x) {
      if (pass == 0) {
        hsave[j] = hs[j];
        Hcol[j] = (T)hs[j];
      } else {
        Hcol[j] = (T)(hsave[j] + hs[j]);
      }
    }
  double s2 = 0.0;
  Ssq q{0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T wi = w[i];
    for (int j = 0; j < kc; ++j) wi = add_rn(wi, mul_rn((T)(-hs[j]), V[i + (int64_t)j * ldv]));
    w[i] = wi;
    const double v = (double)wi;
    s2 = fma(v, v, s2);
    q = ssq_add(q, v);
  }
  s2 = block_sum(s2, sm);
  q = block_ssq(q, sm);
  if (threadIdx.x == 0) {
    red[3 * blockIdx.x] = s2;
    red[3 * blockIdx.x + 1] = q.scale;
    red[3 * blockIdx.x + 2] = q.ssq;
  }
}

// scale the local slice of w by 1/h (global norm from rank-ordered parts)
template <typename T>
__global__ void __launch_bounds__(kDT)
    gm_shard_normalize_kernel(int64_t n, T* __restrict__ w, int nranks, const double* __restrict__ parts,
                              const double* st, int64_t k) {
  if (st[ST_STOP] <= (double)k) return;
  double s2, h;
  combine3(parts, nranks, s2, h);
  if (h == 0.0) return;
  const T s = (T)(1.0 / h);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = mul_rn(s, w[i]);
}

// replicated Givens step (krylov.py:139-163); st[ST_STOP] = inner stop index
template <typename T>
__global__ void gm_shard_givens_kernel(int nranks, const double* __restrict__ parts, T* H, T* Hraw, int64_t ldh,
                                       T* g, T* cs, T* sn, int k, double* est_out, double* st, double tol,
                                       int64_t total_before, int64_t cap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (st[ST_STOP] <= (double)k) return;
  double s2, hk1;
  combine3(parts, nranks, s2, hk1);
  const bool happy = hk1 == 0.0;
  T* Hk = H + (int64_t)k * ldh;
  T* Hr = Hraw + (int64_t)k * ldh;
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
  const double est = fabs((double)g[k + 1]) / st[ST_BNORM];
  est_out[k] = est;
  if (happy) st[ST_BAD] = 1.0;  // happy flag
  if (happy || est <= tol || total_before + k + 1 >= cap) {
    st[ST_STOP] = (double)(k + 1);
    reinterpret_cast<int64_t*>(st)[ST_STOP64] = k + 1;  // the Gate word of the GEMVs
  }
}

template <typename T>
__global__ void gm_shard_lsq_kernel(const T* H, int64_t ldh, const T* g, int inner, T* y, double* st) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = 0; i < inner; ++i) y[i] = g[i];
  for (int i = inner - 1; i >= 0; --i) {
    if (i + 1 < inner) {
      double s = 0.0;
      for (int j = i + 1; j < inner; ++j) s = fma((double)H[i + (int64_t)j * ldh], (double)y[j], s);
      y[i] = sub_rn(y[i], (T)s);
    }
    const T d = H[i + (int64_t)i * ldh];
    if (d == T(0)) {
      st[ST_STATUS] = (double)DS_ESINGULAR;
      st[ST_RES] = (double)i;
      return;
    }
    y[i] = div_rn(y[i], d);
  }
}

template <typename T>
__global__ void gm_shard_start_kernel(int64_t n, const T* __restrict__ r, T* __restrict__ v0, int nranks,
                                      const double* __restrict__ parts, T* g, double* st) {
  double s2, beta;
  combine3(parts, nranks, s2, beta);
  const T s = (T)(1.0 / beta);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v0[i] = mul_rn(s, r[i]);
  if (blockIdx.x == 0 && threadIdx.x == 0) g[0] = (T)beta;
}

// max|A[i,j] - B[j,i]| and max|A| over an m x n block A and n x m block B
template <typename T>
__global__ void __launch_bounds__(256)
    absdiff_t_kernel(int64_t m, int64_t n, const T* __restrict__ A, int64_t lda, const T* __restrict__ B,
                     int64_t ldb, double* red) {
  __shared__ T tb[32][33];
  __shared__ double sm[32];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t ti = ceil_div(m, 32), tj = ceil_div(n, 32);
  double dmax = 0.0, amax = 0.0;
  for (int64_t tile = blockIdx.x; tile < ti * tj; tile += gridDim.x) {
    const int64_t r0 = (tile % ti) * 32, c0 = (tile / ti) * 32;
    __syncthreads();
    for (int kk = ty; kk < 32; kk += 8) {  // B[c0+kk, r0+tx] -> tb[kk][tx]
      const int64_t br = c0 + kk, bc = r0 + tx;
      tb[kk][tx] = (br < n && bc < m) ? B[br + bc * ldb] : T(0);
    }
    __syncthreads();
    for (int kk = ty; kk < 32; kk += 8) {  // A[r0+tx, c0+kk] vs B[c0+kk, r0+tx]
      const int64_t r = r0 + tx, c = c0 + kk;
      if (r < m && c < n) {
        const T a = A[r + c * lda];
        dmax = nanmax(dmax, fabs((double)sub_rn(a, tb[kk][tx])));
        amax = nanmax(amax, fabs((double)a));
      }
    }
  }
  dmax = block_nanmax(dmax, sm);
  amax = block_nanmax(amax, sm);
  if (threadIdx.x == 0) {
    red[2 * blockIdx.x] = dmax;
    red[2 * blockIdx.x + 1] = amax;
  }
}

__global__ void max2_finish_kernel(const double* red, int nblk, double* out) {
  __shared__ double sm[32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    a = nanmax(a, red[2 * i]);
    b = nanmax(b, red[2 * i + 1]);
  }
  a = block_nanmax(a, sm);
  b = block_nanmax(b, sm);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
  }
}

static int vgrid(ds_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(std::max<int64_t>(n, 1), kDT), (int64_t)ctx->num_sms * 2));
}

// tall-panel LU and laswp live in ds_lu.cu
template <typename T>
int lu_factor_impl(ds_ctx* ctx, int64_t m, int64_t w, T* W, int64_t ld, int64_t b, int64_t* d_piv, int8_t* d_zero);
template <typename T>
int laswp_range(ds_ctx* ctx, T* W, int64_t ld, int64_t ncols, int64_t k0, int64_t k1, const int64_t* d_piv);

int preload_sharded_kernels_dist() {  // see preload_sharded_kernels_blas
  cudaFuncAttributes a;
  const void* fns[] = {(const void*)absdiff_t_kernel<double>, (const void*)absdiff_t_kernel<float>,
                       (const void*)max2_finish_kernel,
                       // the row-sharded GMRES shard kernels
                       (const void*)vec_parts_kernel<double>, (const void*)vec_parts_kernel<float>,
                       (const void*)parts3_finish_kernel, (const void*)multidot_dev_kernel<double>,
                       (const void*)multidot_dev_kernel<float>, (const void*)multidot_finish_kernel,
                       (const void*)cgs_update_shard_kernel<double>, (const void*)cgs_update_shard_kernel<float>,
                       (const void*)gm_shard_normalize_kernel<double>, (const void*)gm_shard_normalize_kernel<float>,
                       (const void*)gm_shard_givens_kernel<double>, (const void*)gm_shard_givens_kernel<float>,
                       (const void*)gm_shard_lsq_kernel<double>, (const void*)gm_shard_lsq_kernel<float>,
                       (const void*)gm_shard_start_kernel<double>, (const void*)gm_shard_start_kernel<float>};
  for (const void* f : fns) DS_CUDA(cudaFuncGetAttributes(&a, f));
  return DS_OK;
}

}  // namespace ds

using namespace ds;

extern "C" {

int ds_vec_parts(ds_ctx* ctx, int dtype, int64_t n, const void* x, double* d_out3) {
  DS_ENTER(ctx);
  void* ws = nullptr;
  const int g = vgrid(ctx, n);
  DS_TRY(ctx_workspace(ctx, (size_t)g * 3 * sizeof(double) + 256, &ws));
  DS_DISPATCH(dtype, T, vec_parts_kernel<T><<<g, kDT, 0, ctx->stream>>>(n, (const T*)x, (double*)ws));
  parts3_finish_kernel<<<1, 256, 0, ctx->stream>>>((const double*)ws, g, d_out3);
  count_launch(ctx, 2);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

int ds_dot_dev(ds_ctx* ctx, int dtype, int64_t n, const void* x, const void* y, double* d_out) {
  DS_ENTER(ctx);
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, (size_t)ctx->num_sms * 8 * sizeof(double) + 256, &ws));
  int nb = 0;
  DS_DISPATCH(dtype, T, DS_TRY(dot_launch<T>(ctx, n, (const T*)x, (const T*)y, (double*)ws, &nb)));
  DS_TRY(finish_sum(ctx, (const double*)ws, nb, d_out));
  return DS_OK;
}

int ds_gemv_acc(ds_ctx* ctx, int dtype, int64_t m, int64_t n, const void* A, int64_t lda, const void* x, void* y) {
  DS_ENTER(ctx);
  if (m == 0) return DS_OK;
  const GemvPlan p = gemv_plan(ctx, m, n, dtype_size(dtype));
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, p.part_bytes + 4096, &ws));
  DS_DISPATCH(dtype, T,
              DS_TRY(gemv_launch<T>(ctx, p, (const T*)A, lda, (const T*)x, (T*)y, (double*)ws, EPI_AXPY_INTO,
                                    nullptr, nullptr, nullptr)));
  return DS_OK;
}

int ds_resid_parts(ds_ctx* ctx, int dtype, int64_t m, int64_t n, const void* A, int64_t lda, const void* x,
                   const void* b, void* r, double* d_out3) {
  DS_ENTER(ctx);
  if (m == 0) {
    DS_CUDA(cudaMemsetAsync(d_out3, 0, 3 * sizeof(double), ctx->stream));
    return DS_OK;
  }
  const GemvPlan p = gemv_plan(ctx, m, n, dtype_size(dtype));
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, p.part_bytes + 4096, &ws));
  DS_DISPATCH(dtype, T,
              DS_TRY(gemv_launch<T>(ctx, p, (const T*)A, lda, (const T*)x, (T*)r, (double*)ws, EPI_STORE, nullptr,
                                    nullptr, nullptr)));
  // r = b - Ax, then parts of r
  DS_DISPATCH(dtype, T, DS_TRY(axpy_launch<T>(ctx, m, -1.0, (const T*)r, (const T*)b, (T*)r)));
  return ds_vec_parts(ctx, dtype, m, r, d_out3);
}

int ds_cg_shard_init(ds_ctx* ctx, const double* d_bparts, const double* d_rparts, int nranks, double* d_state,
                     double* d_hist, double tol, int64_t cap) {
  DS_ENTER(ctx);
  cg_shard_init_kernel<<<1, 32, 0, ctx->stream>>>(d_bparts, d_rparts, nranks, d_state, d_hist, tol, cap);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

int ds_cg_shard_update(ds_ctx* ctx, int dtype, int64_t n_loc, int nranks, const double* d_pap_parts,
                       double* d_state, int64_t k, void* x, void* r, const void* p, const void* Ap, double* d_out3) {
  DS_ENTER(ctx);
  const int g = vgrid(ctx, n_loc);
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, (size_t)g * 3 * sizeof(double) + 256, &ws));
  DS_CUDA(cudaMemsetAsync(ws, 0, (size_t)g * 3 * sizeof(double), ctx->stream));
  DS_DISPATCH(dtype, T,
              cg_shard_update_kernel<T><<<g, kDT, 0, ctx->stream>>>(n_loc, nranks, d_pap_parts, d_state, k, (T*)x,
                                                                    (T*)r, (const T*)p, (const T*)Ap, (double*)ws));
  parts3_finish_kernel<<<1, 256, 0, ctx->stream>>>((const double*)ws, g, d_out3);
  count_launch(ctx, 2);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

int ds_cg_shard_finish(ds_ctx* ctx, int dtype, int64_t n_loc, int nranks, const double* d_parts3, double* d_state,
                       int64_t k, const void* r, void* p, double* d_hist, double tol, int64_t cap) {
  DS_ENTER(ctx);
  const int g = vgrid(ctx, n_loc);
  DS_DISPATCH(dtype, T,
              cg_shard_finish_kernel<T><<<g, kDT, 0, ctx->stream>>>(n_loc, nranks, d_parts3, d_state, k,
                                                                    (const T*)r, (T*)p, d_hist, tol, cap));
  cg_shard_commit_kernel<<<1, 32, 0, ctx->stream>>>(nranks, d_parts3, d_state, k, d_hist, tol, cap);
  count_launch(ctx, 2);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

int ds_multidot_dev(ds_ctx* ctx, int dtype, int64_t n_loc, const void* V, int64_t ldv, int kc, const void* w,
                    double* d_out) {
  DS_ENTER(ctx);
  if (kc > 64) {
    set_error("multidot: kc > 64");
    return DS_EINVAL;
  }
  const int g = vgrid(ctx, n_loc);
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, (size_t)g * 64 * sizeof(double) + 256, &ws));
  DS_DISPATCH(dtype, T,
              multidot_dev_kernel<T><<<g, kDT, 0, ctx->stream>>>(n_loc, (const T*)V, ldv, kc, (const T*)w,
                                                                 (double*)ws));
  multidot_finish_kernel<<<1, 512, 0, ctx->stream>>>((const double*)ws, g, kc, d_out);
  count_launch(ctx, 2);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

int ds_cgs_update_shard(ds_ctx* ctx, int dtype, int64_t n_loc, const void* V, int64_t ldv, int kc, void* w,
                        int nranks, const double* d_parts, void* Hcol, double* d_hsave, int pass, double* d_out3,
                        const double* d_state, int64_t k) {
  DS_ENTER(ctx);
  const int g = vgrid(ctx, n_loc);
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, (size_t)g * 3 * sizeof(double) + 256, &ws));
  DS_CUDA(cudaMemsetAsync(ws, 0, (size_t)g * 3 * sizeof(double), ctx->stream));
  DS_DISPATCH(dtype, T,
              cgs_update_shard_kernel<T><<<g, kDT, 0, ctx->stream>>>(n_loc, (const T*)V, ldv, kc, (T*)w, nranks,
                                                                     d_parts, (T*)Hcol, d_hsave, pass,
                                                                     (double*)ws, d_state, k));
  parts3_finish_kernel<<<1, 256, 0, ctx->stream>>>((const double*)ws, g, d_out3);
  count_launch(ctx, 2);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

int ds_gmres_shard_step(ds_ctx* ctx, int dtype, int64_t n_loc, void* w, int nranks, const double* d_parts3,
                        void* H, void* Hraw, int64_t ldh, void* g, void* cs, void* sn, int k, double* d_est,
                        double* d_state, double tol, int64_t total_before, int64_t cap) {
  DS_ENTER(ctx);
  const int gr = vgrid(ctx, n_loc);
  DS_DISPATCH(dtype, T,
              gm_shard_normalize_kernel<T><<<gr, kDT, 0, ctx->stream>>>(n_loc, (T*)w, nranks, d_parts3, d_state, k));
  DS_DISPATCH(dtype, T,
              gm_shard_givens_kernel<T><<<1, 32, 0, ctx->stream>>>(nranks, d_parts3, (T*)H, (T*)Hraw, ldh, (T*)g,
                                                                   (T*)cs, (T*)sn, k, d_est, d_state, tol,
                                                                   total_before, cap));
  count_launch(ctx, 2);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

int ds_gmres_shard_start(ds_ctx* ctx, int dtype, int64_t n_loc, const void* r, void* v0, int nranks,
                         const double* d_parts3, void* g, double* d_state) {
  DS_ENTER(ctx);
  const int gr = vgrid(ctx, n_loc);
  DS_DISPATCH(dtype, T,
              gm_shard_start_kernel<T><<<gr, kDT, 0, ctx->stream>>>(n_loc, (const T*)r, (T*)v0, nranks, d_parts3,
                                                                    (T*)g, d_state));
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

int ds_gmres_lsq(ds_ctx* ctx, int dtype, const void* H, int64_t ldh, const void* g, int inner, void* y,
                 double* d_state) {
  DS_ENTER(ctx);
  DS_DISPATCH(dtype, T,
              gm_shard_lsq_kernel<T><<<1, 32, 0, ctx->stream>>>((const T*)H, ldh, (const T*)g, inner, (T*)y, d_state));
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

int ds_absdiff_transposed(ds_ctx* ctx, int dtype, int64_t m, int64_t n, const void* A, int64_t lda, const void* B,
                          int64_t ldb, double* h_out2) {
  DS_ENTER(ctx);
  if (m == 0 || n == 0) {
    h_out2[0] = h_out2[1] = 0.0;
    return DS_OK;
  }
  const int64_t tiles = ceil_div(m, 32) * ceil_div(n, 32);
  const int g = (int)std::min<int64_t>(tiles, (int64_t)ctx->num_sms * 8);
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, ((size_t)g * 2 + 16) * sizeof(double), &ws));
  double* red = (double*)ws;
  double* out = red + 2 * g + 4;
  DS_DISPATCH(dtype, T,
              absdiff_t_kernel<T><<<g, 256, 0, ctx->stream>>>(m, n, (const T*)A, lda, (const T*)B, ldb, red));
  max2_finish_kernel<<<1, 256, 0, ctx->stream>>>(red, g, out);
  count_launch(ctx, 2);
  DS_CHECK_LAUNCH();
  DS_CUDA(cudaMemcpyAsync(h_out2, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

int ds_lu_panel(ds_ctx* ctx, int dtype, int64_t m, int64_t w, void* P, int64_t ldp, int64_t b, int64_t* d_piv,
                int8_t* d_zero) {
  DS_ENTER(ctx);
  if (m < w || ldp < std::max<int64_t>(m, 1) || b < 1) {
    set_error("lu_panel: need m >= w, ldp >= m, b >= 1 (m=%lld w=%lld)", (long long)m, (long long)w);
    return DS_EDIM;
  }
  if (w == 0) return DS_OK;
  DS_DISPATCH(dtype, T, DS_TRY(lu_factor_impl<T>(ctx, m, w, (T*)P, ldp, std::min(b, w), d_piv, d_zero)));
  return DS_OK;
}

int ds_laswp(ds_ctx* ctx, int dtype, int64_t ncols, void* A, int64_t lda, int64_t k0, int64_t k1,
             const int64_t* d_piv) {
  DS_ENTER(ctx);
  if (ncols <= 0 || k1 <= k0) return DS_OK;
  DS_DISPATCH(dtype, T, DS_TRY(laswp_range<T>(ctx, (T*)A, lda, ncols, k0, k1, d_piv)));
  return DS_OK;
}

}  // extern "C"
