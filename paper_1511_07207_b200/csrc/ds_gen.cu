// ds_gen.cu — the reference's seeded problem generators (harness.py:73-104) at
// config scale, on the device and bit-identical to NumPy.
//
// harness.generate_problem draws every matrix from ONE stream,
// np.random.default_rng([seed, n, kind]) (harness.py:70-74), i.e. a PCG64
// (XSL-RR 128/64) generator.  Generator.uniform(lo, hi) returns
// lo + (hi - lo) * ((next_uint64 >> 11) * 2^-53), and an (n, n) draw fills a
// C-order array row by row, so element (i, j) of the k-th n x n draw is stream
// position k n^2 + i n + j.  A PCG64 state can be advanced by any distance in
// O(log distance) 128-bit multiply-adds (LCG jump-ahead), so every thread starts
// at its own position and the stream is produced in parallel, bit-for-bit.
//
// The host side (SeedSequence hashing of [seed, n, kind] into the initial
// state / increment) stays in NumPy: the caller passes the generator's state.
//
// Kinds (PROBLEM_KINDS order, harness.py:20):
//   1 diag_dominant        A = U; fill_diagonal(A, 0); diag = 4 * rowsum|A|   (:84-87)
//   2 spd                  M = U; A = M^T M + n I; A = tril(A) + tril(A,-1)^T   (:88-91)
//   3 general_nonsymmetric E = U, diag 0; R = U; A = E + 0.5 (R - R^T);
//                          diag 0; diag = 4 * rowsum|A|                        (:92-98)
//   100 uniform            A = U (the C3 pivoting family: diag_dominant's stream
//                          without the diagonal)
// then x_true = U(n) cast to the dtype, b = A x_true (:101-104).
//
// Exactness: uniform draws, the elementwise combinations (one rounding per NumPy
// binary op), the row abs-sums (NumPy's pairwise summation restated exactly,
// see pairwise_abs_rowsum_kernel) and the casts are bitwise NumPy's.  Two
// products are not: M^T M (the FP64 DMMA GEMM, lower triangle; NumPy's BLAS
// syrk/gemm sums in another order, and at n=32768 the reference's own syrk call
// crashes) and b = A x_true (the library GEMV).  Callers that
// need "the same bytes" on both sides download A and b.
#include <vector>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

typedef unsigned __int128 u128;

static __host__ __device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) {
  return ((u128)hi << 64) | (u128)lo;
}
// PCG_DEFAULT_MULTIPLIER_128 of NumPy's pcg64.h
static __host__ __device__ __forceinline__ u128 pcg_mult() {
  return mk128(0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL);
}

// Affine map of `delta` LCG steps: s -> mul * s + add  (pcg_advance_lcg_128).
struct Jump {
  u128 mul, add;
};
static __host__ __device__ __forceinline__ Jump pcg_jump(u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return Jump{acc_mult, acc_plus};
}

// XSL-RR output of a (post-step) state.
static __device__ __forceinline__ uint64_t pcg_output(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const uint64_t x = hi ^ lo;
  const unsigned r = (unsigned)(hi >> 58);
  return (x >> r) | (x << ((64u - r) & 63u));
}

// random_uniform: low + range * next_double  (two roundings, no contraction)
static __device__ __forceinline__ double pcg_uniform(uint64_t raw, double low, double range) {
  const double d = (double)(raw >> 11) * 0x1.0p-53;
  return __dadd_rn(low, __dmul_rn(range, d));
}

struct PcgArgs {
  uint64_t s_hi, s_lo, i_hi, i_lo;  // state and increment after seeding
};

constexpr int GT = 64;  // generator tile edge

// Logical (rows x cols) C-order draw starting at stream position `off`
// (element (i, j) = position off + i cols + j), cast to T and stored
//   COLMAJOR = false: out[i * ld + j]   (the raw C-order array)
//   COLMAJOR = true : out[i + j * ld]   (np.asfortranarray of it)
// 256 threads; thread (ty, tx) draws rows ty, ty + 4, ... of column tx of a
// 64 x 64 tile, stepping the state by 4 cols positions with a precomputed jump.
template <typename T, bool COLMAJOR>
__global__ void __launch_bounds__(256)
    pcg_fill_kernel(PcgArgs a, uint64_t off, int64_t rows, int64_t cols, double low, double range,
                    uint64_t jm_hi, uint64_t jm_lo, uint64_t ja_hi, uint64_t ja_lo, T* __restrict__ out,
                    int64_t ld) {
  __shared__ double tile[COLMAJOR ? GT : 1][GT + 1];
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int64_t i0 = (int64_t)blockIdx.y * GT, j0 = (int64_t)blockIdx.x * GT;
  const int64_t j = j0 + tx;
  const u128 inc = mk128(a.i_hi, a.i_lo);
  const u128 jm = mk128(jm_hi, jm_lo), ja = mk128(ja_hi, ja_lo);
  if (j < cols && i0 + ty < rows) {
    const uint64_t p = off + (uint64_t)(i0 + ty) * (uint64_t)cols + (uint64_t)j;
    const Jump J = pcg_jump(inc, p + 1);  // draw p is the output of the (p+1)-th step
    u128 s = J.mul * mk128(a.s_hi, a.s_lo) + J.add;
#pragma unroll 4
    for (int r = ty; r < GT; r += 4) {
      const int64_t i = i0 + r;
      if (i >= rows) break;
      const double v = pcg_uniform(pcg_output(s), low, range);
      if (COLMAJOR)
        tile[r][tx] = v;
      else
        out[i * ld + j] = (T)v;
      s = jm * s + ja;
    }
  }
  if (COLMAJOR) {
    __syncthreads();
    const int rr = threadIdx.x & 63;
    for (int c = threadIdx.x >> 6; c < GT; c += 4) {
      const int64_t i = i0 + rr, jj = j0 + c;
      if (i < rows && jj < cols) out[i + jj * ld] = (T)tile[rr][c];
    }
  }
}

// general_nonsymmetric, in place on E (C-order, ld n):  A[i,j] = E[i,j] + 0.5 * (R[i,j] - R[j,i]),
// diagonal 0 (harness.py:93-97: E's diagonal is zeroed first, A's again after).
__global__ void __launch_bounds__(256)
    nonsym_combine_kernel(int64_t n, double* __restrict__ E, const double* __restrict__ R) {
  __shared__ double rt[GT][GT + 1];  // rt[c][r] = R[j0 + c, i0 + r]
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int64_t i0 = (int64_t)blockIdx.y * GT, j0 = (int64_t)blockIdx.x * GT;
  for (int c = ty; c < GT; c += 4) {
    const int64_t jr = j0 + c, ir = i0 + tx;
    if (jr < n && ir < n) rt[c][tx] = R[jr * n + ir];
  }
  __syncthreads();
  for (int r = ty; r < GT; r += 4) {
    const int64_t i = i0 + r, j = j0 + tx;
    if (i >= n || j >= n) continue;
    double v = 0.0;
    if (i != j) v = __dadd_rn(E[i * n + j], __dmul_rn(0.5, __dsub_rn(R[i * n + j], rt[tx][r])));
    E[i * n + j] = v;
  }
}

// One CTA per row of the C-order fp64 matrix A (ld n): diag[row] = 4 * sum_j |A[row, j]|
// with A[row, row] read as 0 (fill_diagonal(A, 0.0) precedes the sum), summed in
// exactly NumPy's order.  np.sum(.., axis=1) over a contiguous row is
// pairwise_sum(row, n) (numpy/_core/src/umath/loops_utils.h.src):
//   n < 8:      res = 0.; res += a[i] in order
//   n <= 128:   8 accumulators r[k] = a[k], r[k] += a[i + k] for whole groups of 8,
//               res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)), then the
//               n % 8 tail added in order
//   else:       n2 = n / 2 - (n / 2) % 8; pairwise(a, n2) + pairwise(a + n2, n - n2)
// The split tree depends only on n: the host flattens it into leaves (start, len)
// and a post-order program (>= 0: push leaf k, -1: add the top two).  Each group of
// 8 lanes computes one leaf (lane k owns accumulator k); thread 0 runs the program.
__global__ void __launch_bounds__(256)
    pairwise_abs_rowsum_kernel(int64_t n, const double* __restrict__ A, const int* __restrict__ leaf_start,
                               const int* __restrict__ leaf_len, int nleaves, const int* __restrict__ prog,
                               int nprog, double* __restrict__ diag) {
  extern __shared__ double leaf_sum[];
  const int64_t row = blockIdx.x;
  const double* a = A + row * n;
  const int lane8 = threadIdx.x & 7, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // warp-uniform loop: 4 leaves per warp per pass, every lane takes part in the shuffles
  for (int base = warp * 4; base < nleaves; base += nw * 4) {
    const int lf = base + ((threadIdx.x & 31) >> 3);
    const bool act = lf < nleaves;
    const int64_t st = act ? leaf_start[lf] : 0;
    const int len = act ? leaf_len[lf] : 0;
    const int whole = len >= 8 ? len - len % 8 : 0;
    double r = 0.0;
    if (whole > 0) {
      r = (st + lane8 == row) ? 0.0 : fabs(a[st + lane8]);
      for (int q = 8; q < whole; q += 8) {
        const int64_t c = st + q + lane8;
        r = __dadd_rn(r, c == row ? 0.0 : fabs(a[c]));
      }
    }
    // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) inside each group of 8 lanes
    const unsigned m = 0xffffffffu;
    double t = __dadd_rn(r, __shfl_down_sync(m, r, 1, 8));
    t = __dadd_rn(t, __shfl_down_sync(m, t, 2, 8));
    t = __dadd_rn(t, __shfl_down_sync(m, t, 4, 8));
    if (act && lane8 == 0) {
      double res = whole > 0 ? t : 0.0;  // len < 8: res = 0. then the elements in order
      for (int q = whole; q < len; ++q) res = __dadd_rn(res, st + q == row ? 0.0 : fabs(a[st + q]));
      leaf_sum[lf] = res;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double stack[64];
    int sp = 0;
    for (int k = 0; k < nprog; ++k) {
      const int op = prog[k];
      if (op >= 0) {
        stack[sp++] = leaf_sum[op];
      } else {
        const double rhs = stack[--sp];
        stack[sp - 1] = __dadd_rn(stack[sp - 1], rhs);
      }
    }
    diag[row] = __dmul_rn(4.0, stack[0]);
  }
}

// C-order fp64 A (ld n) -> F-order T output, diagonal replaced by diag[] (fill_diagonal),
// then the dtype cast of np.asfortranarray(A, dtype=dt).
template <typename T>
__global__ void __launch_bounds__(256)
    rowmajor_to_f_kernel(int64_t n, const double* __restrict__ A, const double* __restrict__ diag,
                         T* __restrict__ out, int64_t ld) {
  __shared__ double tile[GT][GT + 1];
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int64_t i0 = (int64_t)blockIdx.y * GT, j0 = (int64_t)blockIdx.x * GT;
  for (int r = ty; r < GT; r += 4) {
    const int64_t i = i0 + r, j = j0 + tx;
    if (i < n && j < n) tile[r][tx] = (i == j) ? diag[i] : A[i * n + j];
  }
  __syncthreads();
  for (int c = ty; c < GT; c += 4) {
    const int64_t i = i0 + tx, j = j0 + c;
    if (i < n && j < n) out[i + j * ld] = (T)tile[tx][c];
  }
}

// spd assembly from the lower triangle of C = -(M^T M) (F-order, ld ldc, the SYRK
// result with C initialised to 0):  S = G + n I with G = -C (harness.py:89), then
// A = tril(S) + tril(S, -1)^T (:91).  Every "+ 0.0" of NumPy's elementwise sums is
// kept (it only turns -0.0 into +0.0).  One CTA per tile pair (I >= J): it reads the
// lower tile, writes it back and its mirror, so `out` may alias C (fp64).
template <typename T>
__global__ void __launch_bounds__(256)
    spd_assemble_kernel(int64_t n, const double* C, int64_t ldc, T* out, int64_t ldo) {
  if (blockIdx.x > blockIdx.y) return;
  __shared__ double tile[GT][GT + 1];  // tile[r][c] = S[i0 + r, j0 + c]
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int64_t i0 = (int64_t)blockIdx.y * GT, j0 = (int64_t)blockIdx.x * GT;
  const double dn = (double)n;
  for (int c = ty; c < GT; c += 4) {
    const int64_t i = i0 + tx, j = j0 + c;
    if (i < n && j < n && i >= j) {
      const double g = -C[i + j * ldc];
      tile[tx][c] = __dadd_rn(g, i == j ? dn : 0.0);
    }
  }
  __syncthreads();
  for (int c = ty; c < GT; c += 4) {  // lower part: column j, rows along tx
    const int64_t i = i0 + tx, j = j0 + c;
    if (i < n && j < n && i >= j) out[i + j * ldo] = (T)__dadd_rn(tile[tx][c], 0.0);
  }
  for (int r = ty; r < GT; r += 4) {  // mirror: out[j, i] = 0.0 + S[i, j] for i > j
    const int64_t i = i0 + r, j = j0 + tx;
    if (i < n && j < n && i > j) out[j + i * ldo] = (T)__dadd_rn(0.0, tile[r][tx]);
  }
}

template <typename T>
__global__ void cast_kernel(int64_t n, const double* __restrict__ x, T* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (T)x[i];
}

// ---- host side ----------------------------------------------------------------------
static int fill(ds_ctx* ctx, int dtype, const PcgArgs& a, uint64_t off, int64_t rows, int64_t cols, double low,
                double high, bool colmajor, void* out, int64_t ld) {
  if (rows <= 0 || cols <= 0) return DS_OK;
  const Jump J = pcg_jump(mk128(a.i_hi, a.i_lo), 4ull * (uint64_t)cols);
  const uint64_t jm_hi = (uint64_t)(J.mul >> 64), jm_lo = (uint64_t)J.mul;
  const uint64_t ja_hi = (uint64_t)(J.add >> 64), ja_lo = (uint64_t)J.add;
  const double range = high - low;
  dim3 grid((unsigned)ceil_div(cols, GT), (unsigned)ceil_div(rows, GT));
  if (grid.y > 65535u) {
    set_error("generator: %lld rows exceed the launch grid", (long long)rows);
    return DS_EINVAL;
  }
#define DS_FILL(T, CM)                                                                                    \
  pcg_fill_kernel<T, CM><<<grid, 256, 0, ctx->stream>>>(a, off, rows, cols, low, range, jm_hi, jm_lo, ja_hi, \
                                                         ja_lo, (T*)out, ld)
  if (dtype == DS_F64) {
    if (colmajor) DS_FILL(double, true); else DS_FILL(double, false);
  } else {
    if (colmajor) DS_FILL(float, true); else DS_FILL(float, false);
  }
#undef DS_FILL
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

// NumPy's pairwise split tree for length n, flattened (see the kernel comment).
static void pairwise_plan(int64_t start, int64_t n, std::vector<int>& ls, std::vector<int>& ll,
                          std::vector<int>& prog) {
  if (n <= 128) {
    prog.push_back((int)ls.size());
    ls.push_back((int)start);
    ll.push_back((int)n);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  pairwise_plan(start, n2, ls, ll, prog);
  pairwise_plan(start + n2, n - n2, ls, ll, prog);
  prog.push_back(-1);
}

static int dominant_diagonal(ds_ctx* ctx, int64_t n, const double* A, double* diag) {
  std::vector<int> ls, ll, prog;
  pairwise_plan(0, n, ls, ll, prog);
  const size_t bytes = (ls.size() * 2 + prog.size()) * sizeof(int);
  std::vector<int> host(ls);
  host.insert(host.end(), ll.begin(), ll.end());
  host.insert(host.end(), prog.begin(), prog.end());
  int* d = nullptr;
  DS_CUDA(cudaMallocAsync((void**)&d, bytes, ctx->stream));
  DS_CUDA(cudaMemcpyAsync(d, host.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
  const int nl = (int)ls.size();
  const size_t smem = (size_t)nl * sizeof(double);
  if (smem > 200 * 1024) {
    set_error("generator: n=%lld too large for the row-sum kernel", (long long)n);
    return DS_EINVAL;
  }
  if (smem > 48 * 1024)
    DS_CUDA(cudaFuncSetAttribute(pairwise_abs_rowsum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  pairwise_abs_rowsum_kernel<<<(unsigned)n, 256, smem, ctx->stream>>>(n, A, d, d + nl, nl, d + 2 * nl,
                                                                      (int)prog.size(), diag);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  // the stack program must not be freed before the kernel ran: stream-ordered free
  DS_CUDA(cudaFreeAsync(d, ctx->stream));
  return DS_OK;
}

template <typename T>
static int generate(ds_ctx* ctx, int kind, int64_t n, const PcgArgs& a, T* A, int64_t lda, T* b, T* xt) {
  const int dt = sizeof(T) == 8 ? DS_F64 : DS_F32;
  const uint64_t nn = (uint64_t)n * (uint64_t)n;
  uint64_t x_off = nn;  // stream position of x_true
  cudaStream_t st = ctx->stream;
  dim3 tiles((unsigned)ceil_div(n, GT), (unsigned)ceil_div(n, GT));
  if (kind == DS_GEN_UNIFORM) {
    DS_TRY(fill(ctx, dt, a, 0, n, n, -1.0, 1.0, true, A, lda));
  } else if (kind == DS_GEN_DIAG_DOMINANT || kind == DS_GEN_GENERAL_NONSYMMETRIC) {
    double *E = nullptr, *R = nullptr, *diag = nullptr;
    DS_CUDA(cudaMallocAsync((void**)&E, nn * 8, st));
    DS_CUDA(cudaMallocAsync((void**)&diag, (size_t)n * 8, st));
    DS_TRY(fill(ctx, DS_F64, a, 0, n, n, -1.0, 1.0, false, E, n));
    if (kind == DS_GEN_GENERAL_NONSYMMETRIC) {
      DS_CUDA(cudaMallocAsync((void**)&R, nn * 8, st));
      DS_TRY(fill(ctx, DS_F64, a, nn, n, n, -1.0, 1.0, false, R, n));
      nonsym_combine_kernel<<<tiles, 256, 0, st>>>(n, E, R);
      count_launch(ctx);
      DS_CHECK_LAUNCH();
      DS_CUDA(cudaFreeAsync(R, st));
      x_off = 2 * nn;
    }
    DS_TRY(dominant_diagonal(ctx, n, E, diag));
    rowmajor_to_f_kernel<T><<<tiles, 256, 0, st>>>(n, E, diag, A, lda);
    count_launch(ctx);
    DS_CHECK_LAUNCH();
    DS_CUDA(cudaFreeAsync(E, st));
    DS_CUDA(cudaFreeAsync(diag, st));
  } else if (kind == DS_GEN_SPD) {
    // M^T M = (M^T)(M): the raw C-order draw read column-major IS M^T; M itself is
    // the same draw stored column-major.  Lower-tile SYRK C -= M^T M from C = 0.
    double *Mt = nullptr, *Mf = nullptr, *C = nullptr;
    DS_CUDA(cudaMallocAsync((void**)&Mt, nn * 8, st));
    DS_CUDA(cudaMallocAsync((void**)&Mf, nn * 8, st));
    DS_TRY(fill(ctx, DS_F64, a, 0, n, n, -1.0, 1.0, false, Mt, n));
    DS_TRY(fill(ctx, DS_F64, a, 0, n, n, -1.0, 1.0, true, Mf, n));
    int64_t ldc = n;
    if (sizeof(T) == 8) {
      C = (double*)A;
      ldc = lda;
    } else {
      DS_CUDA(cudaMallocAsync((void**)&C, nn * 8, st));
    }
    DS_CUDA(cudaMemset2DAsync(C, (size_t)ldc * 8, 0, (size_t)n * 8, (size_t)n, st));
    DS_TRY(gemm_sub_lower_launch<double>(ctx, n, n, n, Mt, n, Mf, n, C, ldc));
    spd_assemble_kernel<T><<<tiles, 256, 0, st>>>(n, C, ldc, A, lda);
    count_launch(ctx);
    DS_CHECK_LAUNCH();
    DS_CUDA(cudaFreeAsync(Mt, st));
    DS_CUDA(cudaFreeAsync(Mf, st));
    if ((void*)C != (void*)A) DS_CUDA(cudaFreeAsync(C, st));
  } else {
    set_error("cannot generate kind code %d", kind);
    return DS_EINVAL;
  }
  if (xt == nullptr && b == nullptr) return DS_OK;
  // x_true = U(n) drawn in fp64 after the matrix, cast to the dtype (harness.py:101-103)
  T* x = xt;
  if (x == nullptr) DS_CUDA(cudaMallocAsync((void**)&x, (size_t)n * sizeof(T), st));
  DS_TRY(fill(ctx, dt, a, x_off, 1, n, -1.0, 1.0, false, x, n));
  if (b != nullptr) {  // b = A @ x_true (harness.py:104), library GEMV
    const GemvPlan p = gemv_plan(ctx, n, n, sizeof(T));
    void* ws = nullptr;
    DS_TRY(ctx_workspace(ctx, p.part_bytes + 4096, &ws));
    DS_TRY(gemv_launch<T>(ctx, p, A, lda, x, b, (double*)ws, EPI_STORE, nullptr, nullptr, nullptr));
  }
  if (x != xt) DS_CUDA(cudaFreeAsync(x, st));
  return DS_OK;
}

}  // namespace ds

using namespace ds;

extern "C" {

int ds_rng_uniform(ds_ctx* ctx, int dtype, const uint64_t* h_pcg, uint64_t offset, int64_t rows, int64_t cols,
                   double low, double high, int colmajor, void* d_out, int64_t ld) {
  DS_ENTER(ctx);
  if (dtype != DS_F64 && dtype != DS_F32) {
    set_error("unsupported dtype code %d", dtype);
    return DS_EPREC;
  }
  if (rows < 0 || cols < 0 || ld < (colmajor ? rows : cols)) {
    set_error("rng_uniform: bad shape %lld x %lld (ld %lld)", (long long)rows, (long long)cols, (long long)ld);
    return DS_EDIM;
  }
  const PcgArgs a{h_pcg[0], h_pcg[1], h_pcg[2], h_pcg[3]};
  return fill(ctx, dtype, a, offset, rows, cols, low, high, colmajor != 0, d_out, ld);
}

int ds_generate(ds_ctx* ctx, int kind, int dtype, int64_t n, const uint64_t* h_pcg, void* d_A, int64_t lda,
                void* d_b, void* d_x_true) {
  DS_ENTER(ctx);
  if (n < 1 || lda < n) {
    set_error("generate: bad size n=%lld lda=%lld", (long long)n, (long long)lda);
    return DS_EDIM;
  }
  const PcgArgs a{h_pcg[0], h_pcg[1], h_pcg[2], h_pcg[3]};
  DS_DISPATCH(dtype, T, DS_TRY(generate<T>(ctx, kind, n, a, (T*)d_A, lda, (T*)d_b, (T*)d_x_true)));
  return DS_OK;
}

}  // extern "C"
