// ds_lu.cu — blocked right-looking LU with partial pivoting + triangular solves.
//
// Restates direct.lu_factor_blocked (/root/reference/pkg/src/densolve/direct.py:50-84),
// direct.lu_factor_unblocked (direct.py:25-47, == blocked with b = n),
// direct.lu_solve (direct.py:155-163) with core.apply_pivots (core.py:94-100),
// and forward/backward_substitution (direct.py:123-152).
//
// Panel (K10): one cooperative kernel per panel; rows [kb, n) are split into
//   contiguous per-CTA ranges.  Per column: CTA-local iamax -> grid barrier ->
//   global first-max pivot (np.argmax(np.abs(.)) semantics) + copy of the pivot
//   and diagonal rows -> grid barrier -> swap, reciprocal scale, rank-1 update
//   of the panel columns (NumPy rounding, so the panel is bitwise the
//   reference's), fused with the next column's local iamax.
// laswp (K11): the panel's swaps applied to the columns outside the panel
//   (deferring them is exact: swaps are pure data movement).
// TRSM (K12) + DMMA GEMM (K13) for the trailing update.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

constexpr int kPanelThreads = 256;

__device__ __forceinline__ bool piv_better(double av, int64_t ai, double bv, int64_t bi) {
  const bool an = av != av, bn = bv != bv;
  if (an || bn) {
    if (an && bn) return ai < bi;
    return an;
  }
  if (av != bv) return av > bv;
  return ai < bi;
}

struct PanelArgs {
  int64_t n, ld, kb, bf;
  int64_t* piv;        // device, global row indices
  int8_t* zero_cols;   // device
  unsigned* bar;       // grid barrier words (2)
  double* cand_v;      // [grid]
  int64_t* cand_i;     // [grid]
  void* rowP;          // scratch: pivot row (panel columns)
  void* rowI;          // scratch: row i before the swap
};

template <typename T>
__device__ void panel_local_iamax(const T* W, const PanelArgs& a, int64_t col, int64_t r_lo,
                                  int64_t r_hi, double* sv, int64_t* si) {
  double bv = -1.0;
  int64_t bi = INT64_MAX;
  for (int64_t r = r_lo + threadIdx.x; r < r_hi; r += blockDim.x) {
    const double v = fabs((double)W[r + col * a.ld]);
    if (piv_better(v, r, bv, bi)) {
      bv = v;
      bi = r;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (piv_better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    sv[wid] = bv;
    si[wid] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (piv_better(sv[w], si[w], bv, bi)) {
        bv = sv[w];
        bi = si[w];
      }
    a.cand_v[blockIdx.x] = bv;
    a.cand_i[blockIdx.x] = bi;
  }
}

template <typename T>
__global__ void __launch_bounds__(kPanelThreads) lu_panel_kernel(T* __restrict__ W, PanelArgs a) {
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  __shared__ int64_t s_piv;
  const unsigned G = gridDim.x;
  const int64_t rows = a.n - a.kb;
  const int64_t per = ceil_div(rows, (int64_t)G);
  const int64_t my_lo = a.kb + (int64_t)blockIdx.x * per;
  const int64_t my_hi = min(a.n, my_lo + per);
  const int64_t ncol = a.bf - a.kb;
  T* rowP = reinterpret_cast<T*>(a.rowP);
  T* rowI = reinterpret_cast<T*>(a.rowI);

  // local iamax of the first panel column
  panel_local_iamax<T>(W, a, a.kb, max(my_lo, a.kb), my_hi, sv, si);
  for (int64_t i = a.kb; i < a.bf; ++i) {
    grid_barrier(a.bar, G);
    // --- global pivot: same fixed order in every CTA ---
    if (threadIdx.x == 0) {
      double bv = -1.0;
      int64_t bi = INT64_MAX;
      for (unsigned b = 0; b < G; ++b) {
        const double v = ((volatile double*)a.cand_v)[b];
        const int64_t ix = ((volatile int64_t*)a.cand_i)[b];
        if (piv_better(v, ix, bv, bi)) {
          bv = v;
          bi = ix;
        }
      }
      if (bi == INT64_MAX) bi = i;  // empty (cannot happen for i < n)
      s_piv = bi;
    }
    __syncthreads();
    const int64_t p = s_piv;
    if (blockIdx.x == 0) {
      if (threadIdx.x == 0) a.piv[i] = p;  // piv[i] = v (direct.py:67)
      for (int64_t j = threadIdx.x; j < ncol; j += blockDim.x) {
        // L1-bypassing loads: these rows were last written by other CTAs
        rowP[j] = __ldcg(W + p + (a.kb + j) * a.ld);
        rowI[j] = __ldcg(W + i + (a.kb + j) * a.ld);
      }
    }
    grid_barrier(a.bar, G);
    // --- swap rows i <-> p within the panel (direct.py:68-70) ---
    if (p != i) {
      if (i >= my_lo && i < my_hi)
        for (int64_t j = threadIdx.x; j < ncol; j += blockDim.x)
          W[i + (a.kb + j) * a.ld] = ((volatile T*)rowP)[j];
      if (p >= my_lo && p < my_hi)
        for (int64_t j = threadIdx.x; j < ncol; j += blockDim.x)
          W[p + (a.kb + j) * a.ld] = ((volatile T*)rowI)[j];
    }
    __syncthreads();
    const T aii = ((volatile T*)rowP)[i - a.kb];
    if (aii == T(0)) {
      // singular column: elimination skipped (direct.py:71-74)
      if (blockIdx.x == 0 && threadIdx.x == 0) a.zero_cols[i] = 1;
    } else {
      const T recip = div_rn(T(1), aii);  // 1.0 / aii in the array dtype (direct.py:76)
      const int64_t r_lo = max(my_lo, i + 1);
      // scale + rank-1 update restricted to the panel (direct.py:75-79, backends.py:152-155)
      for (int64_t r = r_lo + threadIdx.x; r < my_hi; r += blockDim.x) {
        const T l = mul_rn(recip, W[r + i * a.ld]);
        W[r + i * a.ld] = l;
        for (int64_t j = i + 1; j < a.bf; ++j) {
          const T uj = ((volatile T*)rowP)[j - a.kb];
          W[r + j * a.ld] = sub_rn(W[r + j * a.ld], mul_rn(l, uj));
        }
      }
    }
    __syncthreads();
    if (i + 1 < a.bf) panel_local_iamax<T>(W, a, i + 1, max(my_lo, i + 1), my_hi, sv, si);
  }
}

// laswp: apply piv[kb..bf) to columns [c_lo, c_hi) (one thread per column)
template <typename T>
__global__ void laswp_kernel(T* W, int64_t ld, int64_t c_lo, int64_t c_hi, int64_t kb, int64_t bf,
                             const int64_t* __restrict__ piv) {
  __shared__ int64_t sp[1024];
  const int64_t cnt = bf - kb;
  for (int64_t i = threadIdx.x; i < cnt && i < 1024; i += blockDim.x) sp[i] = piv[kb + i];
  __syncthreads();
  const int64_t c = c_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c_hi) return;
  T* col = W + c * ld;
  for (int64_t i = 0; i < cnt; ++i) {
    const int64_t p = i < 1024 ? sp[i] : piv[kb + i];
    const int64_t r = kb + i;
    if (p != r) {
      const T t = col[r];
      col[r] = col[p];
      col[p] = t;
    }
  }
}

template <typename T>
int laswp_launch(ds_ctx* ctx, T* W, int64_t ld, int64_t c_lo, int64_t c_hi, int64_t kb, int64_t bf,
                 const int64_t* piv) {
  if (c_hi <= c_lo) return DS_OK;
  laswp_kernel<T><<<(unsigned)ceil_div(c_hi - c_lo, 128), 128, 0, ctx->stream>>>(W, ld, c_lo, c_hi,
                                                                                 kb, bf, piv);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

template <typename T>
int panel_launch(ds_ctx* ctx, T* W, int64_t n, int64_t ld, int64_t kb, int64_t bf, int64_t* piv,
                 int8_t* zero_cols, char* scratch) {
  static int max_blocks_per_sm[2] = {0, 0};
  int& mb = max_blocks_per_sm[sizeof(T) == 8 ? 1 : 0];
  if (mb == 0) {
    DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&mb, lu_panel_kernel<T>, kPanelThreads, 0));
    if (mb < 1) mb = 1;
  }
  const int64_t rows = n - kb;
  // ~128 rows per CTA minimum; at most one wave of co-resident CTAs (<= 1 per SM
  // keeps the barrier cheap)
  int64_t g = std::min<int64_t>(ceil_div(rows, 128), (int64_t)ctx->num_sms);
  g = std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)ctx->num_sms * mb));
  PanelArgs a;
  a.n = n;
  a.ld = ld;
  a.kb = kb;
  a.bf = bf;
  a.piv = piv;
  a.zero_cols = zero_cols;
  Carver cv{scratch};
  a.bar = cv.take<unsigned>(64);
  a.cand_v = cv.take<double>(sizeof(double) * 1024);
  a.cand_i = cv.take<int64_t>(sizeof(int64_t) * 1024);
  a.rowP = cv.take<T>(sizeof(T) * (bf - kb));
  a.rowI = cv.take<T>(sizeof(T) * (bf - kb));
  void* args[] = {(void*)&W, (void*)&a};
  DS_CUDA(cudaLaunchCooperativeKernel((void*)lu_panel_kernel<T>, dim3((unsigned)g),
                                      dim3(kPanelThreads), args, 0, ctx->stream));
  count_launch(ctx);
  return DS_OK;
}

template <typename T>
int lu_factor_impl(ds_ctx* ctx, int64_t n, T* W, int64_t ld, int64_t nb, int64_t* d_piv,
                   int8_t* d_zero) {
  void* ws = nullptr;
  const size_t scratch_bytes = 64 * 4 + 1024 * 16 + 2 * sizeof(T) * (size_t)std::max<int64_t>(nb, 1) + 8 * 256;
  DS_TRY(ctx_workspace(ctx, scratch_bytes + 256, &ws));
  char* scratch = (char*)ws;
  DS_CUDA(cudaMemsetAsync(scratch, 0, 256, ctx->stream));  // barrier words
  for (int64_t kb = 0; kb < n; kb += nb) {
    const int64_t bf = std::min<int64_t>(kb + nb, n);
    DS_TRY(panel_launch<T>(ctx, W, n, ld, kb, bf, d_piv, d_zero, scratch));
    DS_TRY(laswp_launch<T>(ctx, W, ld, 0, kb, kb, bf, d_piv));
    DS_TRY(laswp_launch<T>(ctx, W, ld, bf, n, kb, bf, d_piv));
    if (bf < n) {
      T* A01 = W + kb + bf * ld;
      const T* L00 = W + kb + kb * ld;
      DS_TRY(trsm_lower_unit_launch<T>(ctx, bf - kb, n - bf, L00, ld, A01, ld, A01, ld));
      const T* L10 = W + bf + kb * ld;
      T* A11 = W + bf + bf * ld;
      DS_TRY(gemm_launch<T>(ctx, n - bf, n - bf, bf - kb, -1.0, L10, ld, A01, ld, 1.0, A11, ld,
                            A11, ld));
    }
  }
  return DS_OK;
}

// ----------------------------------------------------------------------------
// pivots -> gather permutation: idx = apply_pivots(piv, arange(n))  (core.py:94-100)
// ----------------------------------------------------------------------------
__global__ void perm_build_kernel(int64_t n, const int64_t* __restrict__ piv, int* idx_g,
                                  int use_smem) {
  extern __shared__ int idx_s[];
  int* idx = use_smem ? idx_s : idx_g;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) idx[i] = (int)i;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t k = 0; k < n; ++k) {
      const int64_t p = piv[k];
      if (p != k) {
        const int t = idx[k];
        idx[k] = idx[p];
        idx[p] = t;
      }
    }
  }
  __syncthreads();
  if (use_smem)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) idx_g[i] = idx_s[i];
}

template <typename T>
__global__ void gather_kernel(int64_t n, const int* __restrict__ idx, const T* __restrict__ b,
                              T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = b[idx[i]];
}

// ----------------------------------------------------------------------------
// TRSV: sync-free blocked triangular solve, one CTA per 64-row block.  CTAs take
// row blocks in dependency order from an atomic ticket and wait on per-block
// ready flags of the blocks they depend on (column-major tiles streamed
// coalesced).  lower: y = L^-1 b (unit or not); upper: x = U^-1 y.
// ----------------------------------------------------------------------------
constexpr int kTrsvNB = 64;
constexpr int kTrsvThreads = 256;

template <typename T, bool LOWER, bool UNIT>
__global__ void __launch_bounds__(kTrsvThreads)
    trsv_kernel(int64_t n, const T* __restrict__ M, int64_t ld, const T* __restrict__ rhs,
                T* out, int* flags, int* ticket) {
  __shared__ int s_blk;
  __shared__ double part[kTrsvThreads / kTrsvNB][kTrsvNB];
  __shared__ T xs[kTrsvNB];
  __shared__ T ysol[kTrsvNB];
  const int64_t nblk = ceil_div(n, kTrsvNB);
  if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t t = s_blk;
  const int64_t bi = LOWER ? t : nblk - 1 - t;
  const int64_t r0 = bi * kTrsvNB;
  const int nr = (int)min((int64_t)kTrsvNB, n - r0);
  const int rr = threadIdx.x % kTrsvNB, cg = threadIdx.x / kTrsvNB;
  double acc = 0.0;
  // contributions of the already-solved blocks
  for (int64_t s = 0; s < t; ++s) {
    const int64_t bj = LOWER ? s : nblk - 1 - s;
    const int64_t c0 = bj * kTrsvNB;
    const int nc = (int)min((int64_t)kTrsvNB, n - c0);
    if (threadIdx.x == 0) {
      while (((volatile int*)flags)[bj] == 0) __nanosleep(64);
      __threadfence();
    }
    __syncthreads();
    if (threadIdx.x < nc) xs[threadIdx.x] = ((volatile T*)out)[c0 + threadIdx.x];
    __syncthreads();
    if (rr < nr)
      for (int c = cg; c < nc; c += kTrsvThreads / kTrsvNB)
        acc = fma((double)M[(r0 + rr) + (c0 + c) * ld], (double)xs[c], acc);
    __syncthreads();
  }
  part[cg][rr] = acc;
  __syncthreads();
  // diagonal block: one warp, sequential rows
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (LOWER) {
      for (int r = 0; r < nr; ++r) {
        double s = 0.0;
        for (int c = lane; c < r; c += 32) s = fma((double)M[(r0 + r) + (r0 + c) * ld], (double)ysol[c], s);
        s = warp_sum(s);
        if (lane == 0) {
          double off = s;
          for (int q = 0; q < kTrsvThreads / kTrsvNB; ++q) off += part[q][r];
          T v = sub_rn(rhs[r0 + r], (T)off);  // y[i] -= L[i,:i] @ y[:i]
          if (!UNIT) v = div_rn(v, M[(r0 + r) + (r0 + r) * ld]);
          ysol[r] = v;
        }
        __syncwarp();
      }
    } else {
      for (int r = nr - 1; r >= 0; --r) {
        double s = 0.0;
        for (int c = r + 1 + lane; c < nr; c += 32)
          s = fma((double)M[(r0 + r) + (r0 + c) * ld], (double)ysol[c], s);
        s = warp_sum(s);
        if (lane == 0) {
          double off = s;
          for (int q = 0; q < kTrsvThreads / kTrsvNB; ++q) off += part[q][r];
          T v = sub_rn(rhs[r0 + r], (T)off);  // x[i] -= U[i,i+1:] @ x[i+1:]
          v = div_rn(v, M[(r0 + r) + (r0 + r) * ld]);  // x[i] /= U[i,i]
          ysol[r] = v;
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < nr) out[r0 + threadIdx.x] = ysol[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicExch(flags + bi, 1);
}

// zero-diagonal scan: first offending row in the reference's sweep order
template <typename T>
__global__ void diag_zero_kernel(int64_t n, const T* M, int64_t ld, int lower, long long* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (M[i + i * ld] == T(0)) {
      if (lower)
        atomicMin(out, (long long)i);
      else
        atomicMax(out, (long long)i);
    }
  }
}

template <typename T>
int trsv_launch(ds_ctx* ctx, int64_t n, const T* M, int64_t ld, const T* rhs, T* out, bool lower,
                bool unit, char* scratch) {
  if (n == 0) return DS_OK;
  const int64_t nblk = ceil_div(n, kTrsvNB);
  int* ticket = (int*)scratch;
  int* flags = ticket + 64;
  DS_CUDA(cudaMemsetAsync(scratch, 0, (64 + nblk) * sizeof(int), ctx->stream));
  if (lower && unit)
    trsv_kernel<T, true, true><<<(unsigned)nblk, kTrsvThreads, 0, ctx->stream>>>(n, M, ld, rhs, out,
                                                                                 flags, ticket);
  else if (lower)
    trsv_kernel<T, true, false><<<(unsigned)nblk, kTrsvThreads, 0, ctx->stream>>>(n, M, ld, rhs,
                                                                                  out, flags, ticket);
  else
    trsv_kernel<T, false, false><<<(unsigned)nblk, kTrsvThreads, 0, ctx->stream>>>(n, M, ld, rhs,
                                                                                   out, flags, ticket);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

template <typename T>
int diag_check(ds_ctx* ctx, int64_t n, const T* M, int64_t ld, bool lower, int64_t* bad,
               char* scratch) {
  long long* d = (long long*)scratch;
  long long init = lower ? (long long)INT64_MAX : -1LL;
  DS_CUDA(cudaMemcpyAsync(d, &init, sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
  diag_zero_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, ctx->stream>>>(
      n, M, ld, lower ? 1 : 0, d);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  long long h = 0;
  DS_CUDA(cudaMemcpyAsync(&h, d, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  *bad = (lower ? (h == (long long)INT64_MAX) : (h < 0)) ? -1 : (int64_t)h;
  return DS_OK;
}

template <typename T>
int lu_solve_impl(ds_ctx* ctx, int64_t n, const T* LU, int64_t ld, const int64_t* d_piv,
                  const T* b, T* x) {
  void* ws = nullptr;
  const size_t need = (size_t)n * (sizeof(int) + sizeof(T) * 2) + (size_t)(ceil_div(n, 64) + 64) * 4 + 8 * 256;
  DS_TRY(ctx_workspace(ctx, need, &ws));
  Carver cv{(char*)ws};
  int* idx = cv.take<int>((size_t)n * sizeof(int));
  T* pb = cv.take<T>((size_t)n * sizeof(T));
  T* y = cv.take<T>((size_t)n * sizeof(T));
  char* scratch = cv.take<char>((size_t)(ceil_div(n, 64) + 64) * 4);
  const size_t smem = (size_t)n * sizeof(int);
  const int use_smem = smem <= ctx->smem_optin ? 1 : 0;
  if (use_smem) {
    DS_CUDA(cudaFuncSetAttribute(perm_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  }
  perm_build_kernel<<<1, 1024, use_smem ? smem : 0, ctx->stream>>>(n, d_piv, idx, use_smem);
  gather_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, ctx->stream>>>(
      n, idx, b, pb);
  count_launch(ctx, 2);
  DS_CHECK_LAUNCH();
  DS_TRY(trsv_launch<T>(ctx, n, LU, ld, pb, y, true, true, scratch));
  DS_TRY(trsv_launch<T>(ctx, n, LU, ld, y, x, false, false, scratch));
  return DS_OK;
}

}  // namespace ds

using namespace ds;

extern "C" {

int ds_lu_factor_dev(ds_ctx* ctx, int dtype, int64_t n, void* A, int64_t lda, int64_t nb,
                     int64_t* d_piv, int32_t* h_singular) {
  DS_TRY(ctx_begin(ctx));
  if (n < 0 || lda < std::max<int64_t>(n, 1)) {
    set_error("lu: bad shape n=%lld lda=%lld", (long long)n, (long long)lda);
    return DS_EDIM;
  }
  if (nb < 1) {
    set_error("block size must be >= 1");
    return DS_EINVAL;
  }
  if (nb > n) nb = n;
  if (n == 0) {
    if (h_singular) *h_singular = 0;
    return DS_OK;
  }
  int8_t* d_zero = nullptr;
  DS_CUDA(cudaMallocAsync((void**)&d_zero, (size_t)n, ctx->stream));
  DS_CUDA(cudaMemsetAsync(d_zero, 0, (size_t)n, ctx->stream));
  int rc = DS_OK;
  DS_DISPATCH(dtype, T, rc = lu_factor_impl<T>(ctx, n, (T*)A, lda, nb, d_piv, d_zero));
  if (rc != DS_OK) return rc;
  std::vector<int8_t> hz((size_t)n);
  DS_CUDA(cudaMemcpyAsync(hz.data(), d_zero, (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaFreeAsync(d_zero, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_singular) {
    int32_t s = 0;
    for (int64_t i = 0; i < n; ++i) s |= hz[i] ? 1 : 0;
    *h_singular = s;
  }
  return DS_OK;
}

int ds_lu_factor(ds_ctx* ctx, int dtype, int64_t n, void* A, int64_t lda, int64_t nb,
                 int64_t* h_piv, int8_t* h_zero_cols, int32_t* h_singular) {
  DS_TRY(ctx_begin(ctx));
  if (n < 0 || lda < std::max<int64_t>(n, 1)) {
    set_error("lu: bad shape n=%lld lda=%lld", (long long)n, (long long)lda);
    return DS_EDIM;
  }
  if (nb < 1) {
    set_error("block size must be >= 1");
    return DS_EINVAL;
  }
  if (nb > n) nb = n;
  if (n == 0) {
    if (h_singular) *h_singular = 0;
    return DS_OK;
  }
  int64_t* d_piv = nullptr;
  int8_t* d_zero = nullptr;
  DS_CUDA(cudaMallocAsync((void**)&d_piv, (size_t)n * sizeof(int64_t), ctx->stream));
  DS_CUDA(cudaMallocAsync((void**)&d_zero, (size_t)n, ctx->stream));
  DS_CUDA(cudaMemsetAsync(d_zero, 0, (size_t)n, ctx->stream));
  int rc = DS_OK;
  DS_DISPATCH(dtype, T, rc = lu_factor_impl<T>(ctx, n, (T*)A, lda, nb, d_piv, d_zero));
  if (rc != DS_OK) return rc;
  std::vector<int8_t> hz((size_t)n);
  DS_CUDA(cudaMemcpyAsync(h_piv, d_piv, (size_t)n * sizeof(int64_t), cudaMemcpyDeviceToHost,
                          ctx->stream));
  DS_CUDA(cudaMemcpyAsync(hz.data(), d_zero, (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaFreeAsync(d_piv, ctx->stream));
  DS_CUDA(cudaFreeAsync(d_zero, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  int32_t s = 0;
  for (int64_t i = 0; i < n; ++i) s |= hz[i] ? 1 : 0;
  if (h_zero_cols) memcpy(h_zero_cols, hz.data(), (size_t)n);
  if (h_singular) *h_singular = s;
  return DS_OK;
}

int ds_lu_solve(ds_ctx* ctx, int dtype, int64_t n, const void* LU, int64_t lda,
                const int64_t* h_piv, const void* b, void* x) {
  DS_TRY(ctx_begin(ctx));
  if (n == 0) return DS_OK;
  int64_t* d_piv = nullptr;
  DS_CUDA(cudaMallocAsync((void**)&d_piv, (size_t)n * sizeof(int64_t), ctx->stream));
  DS_CUDA(cudaMemcpyAsync(d_piv, h_piv, (size_t)n * sizeof(int64_t), cudaMemcpyHostToDevice,
                          ctx->stream));
  int rc = DS_OK;
  DS_DISPATCH(dtype, T,
              rc = lu_solve_impl<T>(ctx, n, (const T*)LU, lda, d_piv, (const T*)b, (T*)x));
  DS_CUDA(cudaFreeAsync(d_piv, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return rc;
}

int ds_forward_substitution(ds_ctx* ctx, int dtype, int64_t n, const void* L, int64_t ldl,
                            const void* b, void* y, int unit_diagonal, int64_t* h_bad_row) {
  DS_TRY(ctx_begin(ctx));
  if (h_bad_row) *h_bad_row = -1;
  if (n == 0) return DS_OK;
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, (size_t)(ceil_div(n, 64) + 128) * 4 + 512, &ws));
  if (!unit_diagonal) {
    int64_t bad = -1;
    DS_DISPATCH(dtype, T, DS_TRY(diag_check<T>(ctx, n, (const T*)L, ldl, true, &bad, (char*)ws)));
    if (bad >= 0) {
      if (h_bad_row) *h_bad_row = bad;
      set_error("zero diagonal at row %lld", (long long)bad);
      return DS_ESINGULAR;
    }
  }
  DS_DISPATCH(dtype, T,
              DS_TRY(trsv_launch<T>(ctx, n, (const T*)L, ldl, (const T*)b, (T*)y, true,
                                    unit_diagonal != 0, (char*)ws)));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

int ds_backward_substitution(ds_ctx* ctx, int dtype, int64_t n, const void* U, int64_t ldu,
                             const void* y, void* x, int64_t* h_bad_row) {
  DS_TRY(ctx_begin(ctx));
  if (h_bad_row) *h_bad_row = -1;
  if (n == 0) return DS_OK;
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, (size_t)(ceil_div(n, 64) + 128) * 4 + 512, &ws));
  int64_t bad = -1;
  DS_DISPATCH(dtype, T, DS_TRY(diag_check<T>(ctx, n, (const T*)U, ldu, false, &bad, (char*)ws)));
  if (bad >= 0) {
    if (h_bad_row) *h_bad_row = bad;
    set_error("zero diagonal at row %lld", (long long)bad);
    return DS_ESINGULAR;
  }
  DS_DISPATCH(dtype, T,
              DS_TRY(trsv_launch<T>(ctx, n, (const T*)U, ldu, (const T*)y, (T*)x, false, false,
                                    (char*)ws)));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

}  // extern "C"
