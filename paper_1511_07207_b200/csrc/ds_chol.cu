// ds_chol.cu — blocked right-looking Cholesky and cholesky_solve on sm_100a.
//
// Restates direct.cholesky_factor (/root/reference/pkg/src/densolve/direct.py:87-120)
// and direct.cholesky_solve (direct.py:166-171).
//
// The reference factors each b-wide panel column by column to full height
// (sqrt, reciprocal scale, rank-1 update restricted to the panel columns) and
// then applies one GEMM to the whole trailing square.  The column recurrence of
// a panel separates by rows: the b x b diagonal block is factored first (one
// CTA, chol_diag_kernel), after which every row below it runs the same column
// sequence independently (chol_rows_kernel, one thread per row, the row's b
// entries in registers).  Both kernels use the reference's rounding step for
// step (reciprocal in the array dtype, product then subtract), so a panel is
// bitwise the reference's; there is no grid-wide barrier at all.
//
// Trailing update: only the lower triangle of W is ever read again (the panel
// reads W[i:, i]; the result is tril(W)), so the trailing square gets a
// lower-tile SYRK on the FP64 DMMA GEMM (gemm_sub_lower_launch, tiles strictly
// above the diagonal skipped: half the reference's GEMM flops).  As in the LU
// path the b-panels are grouped into NB = 256 outer panels (K = NB trailing
// update); exact-arithmetic identical, rounding grouped differently.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

constexpr int kCholW = 64;  // widest b-panel factored by the exact column kernels

__device__ __forceinline__ double sqrt_rn(double x) { return __dsqrt_rn(x); }
__device__ __forceinline__ float sqrt_rn(float x) { return __fsqrt_rn(x); }

// Factor the nbw x nbw diagonal block W[ib:ib+nbw, ib:ib+nbw] (lower part) with
// the reference's column loop (direct.py:104-115).  err: first failing index.
// One thread per block row, the row rotated in registers (x[k] = column i + k at
// step i, so every step is the same straight-line code): thread i takes the
// square root, every row below scales its column-i entry and publishes it, then
// updates its remaining entries with the published column (W[r, j] -= W[r, i] *
// W[j, i], the reference's order per element).  Two barriers per column.
template <typename T>
__global__ void __launch_bounds__(kCholW)
    chol_diag_kernel(T* __restrict__ W, int64_t ld, int64_t ib, int nbw, long long* err) {
  __shared__ T colv[2][2 * kCholW];  // step parity: column i of the scaled block, colv[.][j] = W[j, i]
  __shared__ T s_rinv[2];
  __shared__ int s_fail;
  if (*((volatile long long*)err) >= 0) return;
  const int r = threadIdx.x;
  const bool mine = r < nbw;
  T x[kCholW];
#pragma unroll
  for (int k = 0; k < kCholW; ++k) x[k] = (mine && k <= r) ? W[(ib + r) + (ib + k) * ld] : T(0);
  if (r == 0) s_fail = 0;
  __syncthreads();
  for (int i = 0; i < nbw; ++i) {
    const int par = i & 1;
    if (r == i) {
      const T aii = x[0];
      if (!(aii > T(0)) || !isfinite((double)aii)) {  // direct.py:106-107
        s_fail = 1;
        *err = (long long)(ib + i);
      } else {
        const T d = sqrt_rn(aii);  // W[i, i] = np.sqrt(aii)
        x[0] = d;
        s_rinv[par] = div_rn(T(1), d);  // 1.0 / W[i, i] in the array dtype
      }
    }
    __syncthreads();
    if (s_fail) return;
    if (mine && r > i) {
      x[0] = mul_rn(s_rinv[par], x[0]);  // scal
      colv[par][r] = x[0];
    }
    if (mine && r >= i) W[(ib + r) + (ib + i) * ld] = x[0];  // column i of row r is final (lower part only)
    __syncthreads();
    // ger restricted to the panel: x[k] (column j = i + k, i < j <= r) -= W[r, i] * W[j, i].
    // Entries of columns j > r are updated too (unpredicated): they are never read for
    // columns <= r (each register slot tracks one column) and never stored.
    if (mine && r > i) {
      const T l = x[0];
      const T* cv = colv[par] + i;
#pragma unroll
      for (int k = 1; k < kCholW; ++k) x[k - 1] = sub_rn(x[k], mul_rn(l, cv[k]));
      x[kCholW - 1] = T(0);
    }
  }
}

// Rows r in [r0, n): the same column sequence on W[r, ib:ib+nbw] given the
// factored diagonal block (direct.py:110-115 restricted to row r).  One thread per
// row, the row rotated in registers (x[k] = column i + k at step i): the update of
// step i and the shift by one are one fused pass, so the loop body is short
// straight-line code (the fully unrolled triangular form was ~13k instructions and
// thrashed the instruction cache).  The last 32 steps only touch x[0..31].
template <typename T>
__global__ void __launch_bounds__(128)
    chol_rows_kernel(T* __restrict__ W, int64_t ld, int64_t n, int64_t ib, int nbw, int64_t r0,
                     const long long* err) {
  __shared__ __align__(16) T Lr[kCholW][kCholW];  // Lr[i][k] = L[ib + i + k, ib + i] (0 past the block)
  __shared__ T rinv[kCholW];
  if (*((volatile const long long*)err) >= 0) return;
  for (int e = threadIdx.x; e < kCholW * kCholW; e += blockDim.x) {
    const int k = e % kCholW, i = e / kCholW;
    Lr[i][k] = (i < nbw && i + k < nbw) ? W[(ib + i + k) + (ib + i) * ld] : T(0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbw; i += blockDim.x) rinv[i] = div_rn(T(1), Lr[i][0]);
  __syncthreads();
  const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  T x[kCholW];
#pragma unroll
  for (int k = 0; k < kCholW; ++k) x[k] = k < nbw ? W[r + (ib + k) * ld] : T(0);
  T* out = W + r + ib * ld;
  const int i_half = nbw < kCholW / 2 ? nbw : kCholW / 2;
  int i = 0;
  for (; i < i_half; ++i) {
    const T l = mul_rn(rinv[i], x[0]);
    out[(int64_t)i * ld] = l;
    const T* li = Lr[i];
#pragma unroll
    for (int k = 1; k < kCholW; ++k) x[k - 1] = sub_rn(x[k], mul_rn(l, li[k]));
    x[kCholW - 1] = T(0);
  }
  for (; i < nbw; ++i) {  // columns >= i + 32 are past the block: only x[0..31] live
    const T l = mul_rn(rinv[i], x[0]);
    out[(int64_t)i * ld] = l;
    const T* li = Lr[i];
#pragma unroll
    for (int k = 1; k < kCholW / 2; ++k) x[k - 1] = sub_rn(x[k], mul_rn(l, li[k]));
    x[kCholW / 2 - 1] = T(0);
  }
}

// out[c + k * ldo] = in[k + c * ldi]  for k < rows, c < cols  (32x32 smem tiles):
// `in` is rows x cols column-major, `out` its cols x rows transpose
template <typename T>
__global__ void transpose_kernel(int64_t rows, int64_t cols, const T* __restrict__ in, int64_t ldi,
                                 T* __restrict__ out, int64_t ldo) {
  __shared__ T t[32][33];
  const int64_t k0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t k = k0 + threadIdx.x, c = c0 + j;
    if (k < rows && c < cols) t[j][threadIdx.x] = in[k + c * ldi];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int64_t c = c0 + threadIdx.x, k = k0 + j;
    if (k < rows && c < cols) out[c + k * ldo] = t[threadIdx.x][j];
  }
}

// np.tril: zero the strict upper triangle
template <typename T>
__global__ void tril_kernel(int64_t n, T* __restrict__ W, int64_t ld) {
  const int64_t c = blockIdx.y;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < c && r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    W[r + c * ld] = T(0);
}

template <typename T>
static int transpose_launch(ds_ctx* ctx, int64_t rows, int64_t cols, const T* in, int64_t ldi, T* out,
                            int64_t ldo) {
  if (rows == 0 || cols == 0) return DS_OK;
  dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(cols, 32));
  transpose_kernel<T><<<grid, dim3(32, 8), 0, ctx->stream>>>(rows, cols, in, ldi, out, ldo);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

template <typename T>
int chol_factor_impl(ds_ctx* ctx, int64_t n, T* W, int64_t ld, int64_t b, long long* d_err) {
  static const int64_t nb_target = [] {
    const char* e = getenv("DENSOLVE_CHOL_NB");  // tuning knob
    return e ? std::max<int64_t>(64, atoll(e)) : (int64_t)512;
  }();
  const int64_t NB = (b >= nb_target || b >= n) ? std::min<int64_t>(b, n)
                                                : std::min<int64_t>(n, b * std::max<int64_t>(1, nb_target / b));
  // scratch for the transposed L blocks (B operands of the SYRKs): NB x n for the main
  // stream, NB x NB... x n for the look-ahead panel on the side stream
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, 2 * (size_t)NB * (size_t)n * sizeof(T) + 8192, &ws));
  T* Bt_main = (T*)ws;
  T* Bt_side = Bt_main + (size_t)NB * (size_t)n + 64;
  const bool lookahead = n > NB && n >= 2048 && !(getenv("DENSOLVE_CHOL_LOOKAHEAD") &&
                                                   getenv("DENSOLVE_CHOL_LOOKAHEAD")[0] == '0');
  if (lookahead && !ctx->side) {
    int lo = 0, hi = 0;
    DS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    DS_CUDA(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, hi));
    DS_CUDA(cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, lo));
    DS_CUDA(cudaEventCreateWithFlags(&ctx->ev_a, cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&ctx->ev_b, cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&ctx->ev_c, cudaEventDisableTiming));
  }
  // factor the outer panel [kb, bf): the reference's b-panels (direct.py:103-115), each
  // followed by the update of the rest of the outer panel
  auto factor_outer = [&](int64_t kb, int64_t bf, T* Bt) -> int {
    for (int64_t ib = kb; ib < bf; ib += b) {
      const int64_t ibf = std::min<int64_t>(ib + b, bf);
      // a b-panel wider than kCholW is factored in kCholW-wide slices with a K-slice
      // GEMM between them (exact-arithmetic identical to the panel's rank-1 sequence)
      for (int64_t sb = ib; sb < ibf; sb += kCholW) {
        const int64_t sbf = std::min<int64_t>(sb + kCholW, ibf);
        const int nbw = (int)(sbf - sb);
        chol_diag_kernel<T><<<1, kCholW, 0, ctx->stream>>>(W, ld, sb, nbw, d_err);
        count_launch(ctx);
        if (sbf < n) {
          const int64_t rows = n - sbf;
          chol_rows_kernel<T><<<(unsigned)ceil_div(rows, 128), 128, 0, ctx->stream>>>(W, ld, n, sb, nbw,
                                                                                    sbf, d_err);
          count_launch(ctx);
        }
        DS_CHECK_LAUNCH();
        // rest of the panel / outer panel: W[sbf:, sbf:bf] -= W[sbf:, sb:sbf] W[sbf:bf, sb:sbf]^T
        if (sbf < bf) {
          const int64_t w = bf - sbf;
          DS_TRY(transpose_launch<T>(ctx, w, nbw, W + sbf + sb * ld, ld, Bt, nbw));
          DS_TRY(gemm_sub_lower_launch<T>(ctx, n - sbf, w, nbw, W + sbf + sb * ld, ld, Bt, nbw,
                                          W + sbf + sbf * ld, ld));
        }
      }
    }
    return DS_OK;
  };
  DS_TRY(factor_outer(0, std::min<int64_t>(NB, n), Bt_main));
  for (int64_t kb = 0; kb < n; kb += NB) {
    const int64_t bf = std::min<int64_t>(kb + NB, n);
    if (bf >= n) break;
    const int64_t bf2 = std::min<int64_t>(bf + NB, n);
    const int64_t K = bf - kb, m = n - bf;
    // trailing SYRK (direct.py:117-119), lower tiles only: the next outer panel's
    // columns [bf, bf2) first, then (overlapping that panel's factorization on the
    // side stream) the rest of the trailing matrix
    DS_TRY(transpose_launch<T>(ctx, m, K, W + bf + kb * ld, ld, Bt_main, K));
    DS_TRY(gemm_sub_lower_launch<T>(ctx, m, bf2 - bf, K, W + bf + kb * ld, ld, Bt_main, K, W + bf + bf * ld, ld));
    if (lookahead) {
      DS_CUDA(cudaEventRecord(ctx->ev_a, ctx->stream));
      DS_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_a, 0));
      cudaStream_t main = ctx->stream;
      ctx->stream = ctx->side;
      const int rc = factor_outer(bf, bf2, Bt_side);
      ctx->stream = main;
      DS_TRY(rc);
      DS_CUDA(cudaEventRecord(ctx->ev_b, ctx->side));
    }
    if (bf2 < n)
      DS_TRY(gemm_sub_lower_launch<T>(ctx, n - bf2, n - bf2, K, W + bf2 + kb * ld, ld, Bt_main + (bf2 - bf) * K,
                                      K, W + bf2 + bf2 * ld, ld));
    if (lookahead)
      DS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_b, 0));
    else
      DS_TRY(factor_outer(bf, bf2, Bt_main));
  }
  dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 64)), (unsigned)n);
  tril_kernel<T><<<g, 256, 0, ctx->stream>>>(n, W, ld);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

template <typename T>
__global__ void diag_zero_first_kernel(int64_t n, const T* M, int64_t ld, long long* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (M[i + i * ld] == T(0)) atomicMin(out, (long long)i);
}

template <typename T>
int chol_solve_impl(ds_ctx* ctx, int64_t n, const T* L, int64_t ld, const T* b, T* x, int64_t* bad) {
  void* ws = nullptr;
  const size_t sc = trsv_scratch_bytes(n);
  DS_TRY(ctx_workspace(ctx, (size_t)n * sizeof(T) + sc + 1024, &ws));
  Carver cv{(char*)ws};
  long long* d_bad = cv.take<long long>(sizeof(long long) * 2);
  T* y = cv.take<T>((size_t)n * sizeof(T));
  char* scratch = cv.take<char>(sc);
  // forward_substitution(L, b) checks L[i, i] == 0 in sweep order (direct.py:130-134); the
  // backward sweep on L^T sees the same diagonal
  const long long init = INT64_MAX;
  DS_CUDA(cudaMemcpyAsync(d_bad, &init, sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
  diag_zero_first_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, ctx->stream>>>(
      n, L, ld, d_bad);
  count_launch(ctx);
  long long hb = 0;
  DS_CUDA(cudaMemcpyAsync(&hb, d_bad, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hb != INT64_MAX) {
    *bad = hb;
    set_error("zero diagonal at row %lld", hb);
    return DS_ESINGULAR;
  }
  DS_TRY(trsv_launch<T>(ctx, n, L, ld, b, y, true, false, scratch));       // L y = b
  DS_TRY(trsv_upper_trans_launch<T>(ctx, n, L, ld, y, x, scratch));        // L^T x = y
  return DS_OK;
}

}  // namespace ds

using namespace ds;

extern "C" {

int ds_cholesky_factor(ds_ctx* ctx, int dtype, int64_t n, void* A, int64_t lda, int64_t nb,
                       int64_t* h_bad_index) {
  DS_ENTER(ctx);
  if (h_bad_index) *h_bad_index = -1;
  if (n < 0 || lda < std::max<int64_t>(n, 1)) {
    set_error("cholesky: bad shape n=%lld lda=%lld", (long long)n, (long long)lda);
    return DS_EDIM;
  }
  if (nb < 1) {
    set_error("block size must be >= 1");
    return DS_EINVAL;
  }
  if (n == 0) return DS_OK;
  if (nb > n) nb = n;
  // symmetric gate (direct.py:99-101)
  double md = 0, am = 0;
  DS_TRY(ds_symmetry_check(ctx, dtype, n, A, lda, &md, &am));
  const double u = dtype == DS_F64 ? 1.1102230246251565e-16 : 5.960464477539063e-08;
  if (md > 10.0 * u * am) {
    set_error("matrix is not symmetric");
    return DS_ENOTSPD;
  }
  long long* d_err = nullptr;
  DS_CUDA(cudaMallocAsync((void**)&d_err, sizeof(long long), ctx->stream));
  DS_CUDA(cudaMemsetAsync(d_err, 0xFF, sizeof(long long), ctx->stream));  // -1
  int rc = DS_OK;
  DS_DISPATCH(dtype, T, rc = chol_factor_impl<T>(ctx, n, (T*)A, lda, nb, d_err));
  long long herr = -1;
  DS_CUDA(cudaMemcpyAsync(&herr, d_err, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaFreeAsync(d_err, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (rc != DS_OK) return rc;
  if (herr >= 0) {
    if (h_bad_index) *h_bad_index = herr;
    set_error("nonpositive pivot at index %lld", herr);
    return DS_ENOTSPD;
  }
  return DS_OK;
}

int ds_cholesky_solve(ds_ctx* ctx, int dtype, int64_t n, const void* L, int64_t ldl, const void* b,
                      void* x, int64_t* h_bad_row) {
  DS_ENTER(ctx);
  if (h_bad_row) *h_bad_row = -1;
  if (n == 0) return DS_OK;
  int64_t bad = -1;
  int rc = DS_OK;
  DS_DISPATCH(dtype, T, rc = chol_solve_impl<T>(ctx, n, (const T*)L, ldl, (const T*)b, (T*)x, &bad));
  if (rc == DS_ESINGULAR && h_bad_row) *h_bad_row = bad;
  if (rc != DS_OK) return rc;
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

}  // extern "C"
