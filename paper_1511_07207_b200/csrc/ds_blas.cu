// ds_blas.cu — the Backend op contract on sm_100a (backends.py:104-200).
//
// Level-1 ops are single-pass grid-stride kernels with deterministic
// two-stage reductions; GEMV is the HBM-streaming kernel every Krylov
// iteration is built on (K1 in SURVEY.md §2b); GEMM is the FP64 DMMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4) trailing-update kernel of the
// blocked LU (K13); TRSM/GER are the panel-side helpers (K12, K10).
#include <cuda.h>  // CUtensorMap (types only; the encoder is resolved at run time)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

// ============================================================================
// vector load helpers
// ============================================================================
template <typename T, int VEC>
struct VecT;
template <>
struct VecT<double, 2> {
  using type = double2;
};
template <>
struct VecT<float, 4> {
  using type = float4;
};
template <>
struct VecT<double, 1> {
  using type = double;
};
template <>
struct VecT<float, 1> {
  using type = float;
};

template <typename V>
__device__ __forceinline__ V ldg_stream(const V* p) {
  return __ldg(p);
}

template <typename T, int VEC>
__device__ __forceinline__ void vec_to_array(const typename VecT<T, VEC>::type& v, T* out);
template <>
__device__ __forceinline__ void vec_to_array<double, 2>(const double2& v, double* o) {
  o[0] = v.x;
  o[1] = v.y;
}
template <>
__device__ __forceinline__ void vec_to_array<float, 4>(const float4& v, float* o) {
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.z;
  o[3] = v.w;
}
template <>
__device__ __forceinline__ void vec_to_array<double, 1>(const double& v, double* o) {
  o[0] = v;
}
template <>
__device__ __forceinline__ void vec_to_array<float, 1>(const float& v, float* o) {
  o[0] = v;
}

// ============================================================================
// GEMV  (Backend.gemv, backends.py:136-142; call sites krylov.py:47,55,104,128,167)
// ============================================================================
constexpr int kGemvThreads = 256;

GemvPlan gemv_plan(ds_ctx* ctx, int64_t m, int64_t n, size_t elem) {
  GemvPlan p;
  p.m = m;
  p.n = n;
  const int vec = elem == 8 ? 2 : 4;
  p.rows_per_cta = kGemvThreads * vec;
  p.rowtiles = ceil_div(std::max<int64_t>(m, 1), p.rows_per_cta);
  // aim for ~8 CTAs per SM in flight across several waves; chunk >= 64 columns
  const int64_t target = (int64_t)ctx->num_sms * 16;
  int64_t nch = std::max<int64_t>(1, target / p.rowtiles);
  int64_t chunk = ceil_div(std::max<int64_t>(n, 1), nch);
  chunk = std::max<int64_t>(chunk, 64);
  chunk = std::min<int64_t>(chunk, 2048);
  chunk = ceil_div(chunk, 8) * 8;
  static const int64_t forced = [] {
    const char* e = getenv("DENSOLVE_GEMV_CHUNK");  // tuning experiments only
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();
  if (forced >= 8) chunk = ceil_div(forced, 8) * 8;
  p.chunk = chunk;
  p.nchunks = ceil_div(std::max<int64_t>(n, 1), chunk);
  p.part_bytes = (size_t)p.nchunks * (size_t)std::max<int64_t>(m, 1) * sizeof(double);
  return p;
}

template <typename T, int VEC, int UNR>
__global__ void __launch_bounds__(kGemvThreads)
    ds_colstream_mv_kernel(const T* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                        const T* __restrict__ x, int64_t chunk, double* __restrict__ part,
                        Gate gate) {
  pdl_wait();  // x and the stop word come from the previous kernel
  if (gated(gate)) return;
  pdl_launch_dependents();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* xs = reinterpret_cast<T*>(smem_raw);
  const int64_t c0 = (int64_t)blockIdx.y * chunk;
  const int64_t cn = min(chunk, n - c0);
  // the x chunk is staged by the bulk-copy engine (cp.async.bulk, the 1-D TMA path) into
  // shared memory, completing on an mbarrier; unaligned / ragged chunks use plain loads
  const unsigned xbytes = (unsigned)(cn * (int64_t)sizeof(T));
  if (((reinterpret_cast<uintptr_t>(x + c0) | xbytes) & 15u) == 0 && xbytes > 0) {
    __shared__ __align__(8) uint64_t xbar;
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&xbar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(xbytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              (unsigned)__cvta_generic_to_shared(xs)),
          "l"(x + c0), "r"(xbytes), "r"(bar)
          : "memory");
    }
    __syncthreads();  // the barrier is initialised before anyone polls it
    asm volatile(
        "{\n .reg .pred P1;\n XW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra XW_%=;\n}\n" ::"r"(
            bar)
        : "memory");
  } else {
    for (int64_t j = threadIdx.x; j < cn; j += blockDim.x) xs[j] = x[c0 + j];
    __syncthreads();
  }
  using V = typename VecT<T, VEC>::type;
  const int64_t r0 = (int64_t)blockIdx.x * (kGemvThreads * VEC) + (int64_t)threadIdx.x * VEC;
  if (r0 >= m) return;
  double acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = 0.0;
  const T* a = A + c0 * lda + r0;
  if (r0 + VEC <= m) {
    int64_t j = 0;
    for (; j + UNR <= cn; j += UNR) {
      V v[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) v[u] = ldg_stream(reinterpret_cast<const V*>(a + (j + u) * lda));
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        T t[VEC];
        vec_to_array<T, VEC>(v[u], t);
        const double xv = (double)xs[j + u];
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = fma((double)t[e], xv, acc[e]);
      }
    }
    for (; j < cn; ++j) {
      V v = ldg_stream(reinterpret_cast<const V*>(a + j * lda));
      T t[VEC];
      vec_to_array<T, VEC>(v, t);
      const double xv = (double)xs[j];
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[e] = fma((double)t[e], xv, acc[e]);
    }
  } else {
    // ragged row tail (m not a multiple of VEC)
    for (int64_t j = 0; j < cn; ++j) {
      const double xv = (double)xs[j];
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (r0 + e < m) acc[e] = fma((double)__ldg(a + j * lda + e), xv, acc[e]);
    }
  }
  double* out = part + (int64_t)blockIdx.y * m + r0;
#pragma unroll
  for (int e = 0; e < VEC; ++e)
    if (r0 + e < m) out[e] = acc[e];
}

// Wide-CTA stage 1 for small matrices (the GMRES C2 step, n <= 8192): about one CTA per SM,
// CS column groups of 256 threads per CTA (CS x 32 KB of loads in flight per SM instead of
// short-lived CTAs of one group), the group partials summed in a fixed order through shared
// memory: one partial per row per CTA, so the orthogonalisation cluster that sums the
// partials reads ~4x fewer of them.
int wide_groups() {  // column groups per CTA of the wide GEMV (DENSOLVE_GEMV_WIDE=2|4, default 4)
  static const int g = [] {
    const char* e = getenv("DENSOLVE_GEMV_WIDE");
    return e && atoi(e) == 2 ? 2 : 4;
  }();
  return g;
}
GemvPlan gemv_wide_plan(ds_ctx* ctx, int64_t m, int64_t n, size_t elem) {
  const int kWideGroups = wide_groups();
  GemvPlan p;
  p.m = m;
  p.n = n;
  const int vec = elem == 8 ? 2 : 4;
  p.rows_per_cta = kGemvThreads * vec;
  p.rowtiles = ceil_div(std::max<int64_t>(m, 1), p.rows_per_cta);
  const int64_t nch = std::max<int64_t>(1, (int64_t)ctx->num_sms / p.rowtiles);
  p.chunk = ceil_div(ceil_div(std::max<int64_t>(n, 1), nch), 8 * kWideGroups) * 8 * kWideGroups;
  p.nchunks = ceil_div(std::max<int64_t>(n, 1), p.chunk);
  p.part_bytes = (size_t)p.nchunks * (size_t)std::max<int64_t>(m, 1) * sizeof(double);
  return p;
}

// Prefetch (pf > 0, full row tiles): before griddepcontrol.wait — i.e. while the previous
// kernel (the orthogonalisation cluster) still runs and HBM is otherwise idle — one thread
// moves the first pf columns of every column group's A tile into shared memory with
// cp.async.bulk (each column segment of the tile is contiguous); A is not written by the
// solver, so reading it early is safe.  The group loops then take those columns from shared
// memory: same values, same order of accumulation (bitwise the non-prefetching kernel).
template <typename T, int VEC, int UNR, int CS>
__global__ void __launch_bounds__(kGemvThreads * CS)
    ds_colstream_mv_wide_kernel(const T* __restrict__ A, int64_t lda, int64_t m, int64_t n, const T* __restrict__ x,
                                int64_t chunk, double* __restrict__ part, Gate gate, int pf) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* xs = reinterpret_cast<T*>(smem_raw);
  unsigned char* region = smem_raw + ((size_t)chunk * sizeof(T) + 15) / 16 * 16;
  T* pre = reinterpret_cast<T*>(region);       // [CS][pf][kGemvThreads * VEC]
  double* red = reinterpret_cast<double*>(region);  // reuses the prefetch region at the end
  constexpr int kRows = kGemvThreads * VEC;
  const int tl = threadIdx.x % kGemvThreads, grp = threadIdx.x / kGemvThreads;
  const int64_t c0 = (int64_t)blockIdx.y * chunk;
  const int64_t cn = min(chunk, n - c0);
  const int64_t gsz = ceil_div(cn, (int64_t)CS);
  const int64_t rbase = (int64_t)blockIdx.x * kRows;
  // columns prefetched per group: only for full row tiles and whole groups
  const int npf = (rbase + kRows <= m && gsz * CS == cn) ? (int)min((int64_t)pf, gsz) : 0;
  __shared__ __align__(8) uint64_t pbar;
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&pbar);
  if (npf > 0 && threadIdx.x == 0) {
    constexpr unsigned colbytes = kRows * sizeof(T);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                 "r"((unsigned)(CS * npf) * colbytes)
                 : "memory");
    for (int g = 0; g < CS; ++g)
      for (int jj = 0; jj < npf; ++jj) {
        const T* src = A + (c0 + g * gsz + jj) * lda + rbase;
        T* dst = pre + ((size_t)g * npf + jj) * kRows;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                (unsigned)__cvta_generic_to_shared(dst)),
            "l"(src), "r"(colbytes), "r"(bar)
            : "memory");
      }
  }
  pdl_wait();  // x and the stop word come from the previous kernel
  if (gated(gate)) {
    if (npf > 0) {  // no bulk copy may still target the shared memory of an exited CTA
      __syncthreads();
      asm volatile(
          "{\n .reg .pred P1;\n PG_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra PG_%=;\n}\n" ::"r"(
              bar)
          : "memory");
    }
    return;
  }
  pdl_launch_dependents();
  for (int64_t j = threadIdx.x; j < cn; j += blockDim.x) xs[j] = x[c0 + j];
  __syncthreads();
  if (npf > 0)
    asm volatile(
        "{\n .reg .pred P1;\n PW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra PW_%=;\n}\n" ::"r"(
            bar)
        : "memory");
  const int64_t g0 = min(cn, grp * gsz), g1 = min(cn, g0 + gsz);
  using V = typename VecT<T, VEC>::type;
  const int64_t r0 = rbase + (int64_t)tl * VEC;
  double acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = 0.0;
  if (r0 < m) {
    const T* a = A + c0 * lda + r0;
    if (r0 + VEC <= m) {
      int64_t j = g0;
      // the prefetched columns (npf > 0 only for full tiles), then the rest from HBM
      for (int jj = 0; jj < npf; ++jj, ++j) {
        const V v = *reinterpret_cast<const V*>(pre + ((size_t)grp * npf + jj) * kRows + tl * VEC);
        T t[VEC];
        vec_to_array<T, VEC>(v, t);
        const double xv = (double)xs[j];
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = fma((double)t[e], xv, acc[e]);
      }
      for (; j + UNR <= g1; j += UNR) {
        V v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) v[u] = ldg_stream(reinterpret_cast<const V*>(a + (j + u) * lda));
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          T t[VEC];
          vec_to_array<T, VEC>(v[u], t);
          const double xv = (double)xs[j + u];
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[e] = fma((double)t[e], xv, acc[e]);
        }
      }
      for (; j < g1; ++j) {
        V v = ldg_stream(reinterpret_cast<const V*>(a + j * lda));
        T t[VEC];
        vec_to_array<T, VEC>(v, t);
        const double xv = (double)xs[j];
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = fma((double)t[e], xv, acc[e]);
      }
    } else {
      for (int64_t j = g0; j < g1; ++j) {
        const double xv = (double)xs[j];
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          if (r0 + e < m) acc[e] = fma((double)__ldg(a + j * lda + e), xv, acc[e]);
      }
    }
  }
  if (npf > 0) __syncthreads();  // every group is done with the prefetched columns: red reuses them
  if (grp > 0) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) red[(size_t)(grp - 1) * kGemvThreads * VEC + tl * VEC + e] = acc[e];
  }
  __syncthreads();
  if (grp == 0 && r0 < m) {
    double* out = part + (int64_t)blockIdx.y * m + r0;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      double sum = acc[e];
      for (int g = 1; g < CS; ++g) sum += red[(size_t)(g - 1) * kGemvThreads * VEC + tl * VEC + e];  // group order
      if (r0 + e < m) out[e] = sum;
    }
  }
}

template <typename T>
int gemv_partial_wide_pdl_launch(ds_ctx* ctx, const GemvPlan& p, const T* A, int64_t lda, const T* x, double* part,
                                 Gate stop) {
  constexpr int VEC = sizeof(T) == 8 ? 2 : 4;
  const bool aligned = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (lda % VEC == 0);
  if (p.m == 0 || p.n == 0 || !aligned) {
    set_error("wide GEMV needs a non-empty, 16-byte aligned matrix");
    return DS_EINVAL;
  }
  const int kWideGroups = wide_groups();
  // A-tile prefetch depth (columns per group, DENSOLVE_GEMV_PREFETCH; 0 disables): as many as
  // fit beside the x chunk in ~200 KB of shared memory
  static const int pf_env = [] {
    const char* e = getenv("DENSOLVE_GEMV_PREFETCH");
    return e ? std::max(0, atoi(e)) : 12;
  }();
  const size_t xbytes = ((size_t)p.chunk * sizeof(T) + 15) / 16 * 16;
  const size_t colbytes = (size_t)kGemvThreads * VEC * sizeof(T);
  const size_t red_bytes = (size_t)(kWideGroups - 1) * kGemvThreads * VEC * sizeof(double);
  const size_t budget = 200 * 1024;
  int pf = pf_env;
  while (pf > 0 && xbytes + (size_t)kWideGroups * pf * colbytes > budget) --pf;
  const size_t region = std::max(red_bytes, (size_t)kWideGroups * pf * colbytes);
  static size_t attr_done[2] = {0, 0};
  size_t& done = attr_done[sizeof(T) == 8 ? 1 : 0];
  if (xbytes + region > 48 * 1024 && done == 0) {
    DS_CUDA(cudaFuncSetAttribute(ds_colstream_mv_wide_kernel<T, VEC, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(budget + 16 * 1024)));
    DS_CUDA(cudaFuncSetAttribute(ds_colstream_mv_wide_kernel<T, VEC, 8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(budget + 16 * 1024)));
    done = 1;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)p.rowtiles, (unsigned)p.nchunks);
  lc.blockDim = dim3(kGemvThreads * kWideGroups);
  lc.dynamicSmemBytes = xbytes + region;
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const int64_t m = p.m, n = p.n, chunk = p.chunk;
  if (kWideGroups == 2)
    DS_CUDA(cudaLaunchKernelEx(&lc, ds_colstream_mv_wide_kernel<T, VEC, 8, 2>, A, lda, m, n, x, chunk, part, stop, pf));
  else
    DS_CUDA(cudaLaunchKernelEx(&lc, ds_colstream_mv_wide_kernel<T, VEC, 8, 4>, A, lda, m, n, x, chunk, part, stop, pf));
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
template int gemv_partial_wide_pdl_launch<double>(ds_ctx*, const GemvPlan&, const double*, int64_t, const double*,
                                                  double*, Gate);
template int gemv_partial_wide_pdl_launch<float>(ds_ctx*, const GemvPlan&, const float*, int64_t, const float*,
                                                 double*, Gate);

constexpr int kRedThreads = 256;

template <typename T, int EPI>
__global__ void __launch_bounds__(kRedThreads)
    ds_colstream_reduce_kernel(const double* __restrict__ part, int64_t m, int64_t nchunks, T* y,
                       const T* __restrict__ v, double* __restrict__ red, Gate gate) {
  if (gated(gate)) return;
  __shared__ double sm[64];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (i < m) {
    // the chunk partials are summed in chunk order; loads are batched 8 at a time so the
    // L2 round trips overlap instead of serialising behind the dependent adds
    int64_t c = 0;
    for (; c + 8 <= nchunks; c += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = part[(c + u) * m + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; c < nchunks; ++c) s += part[c * m + i];
  }
  const T yi = (T)s;
  if (EPI == EPI_STORE) {
    if (i < m) y[i] = yi;
  } else if (EPI == EPI_DOT) {
    double d = 0.0;
    if (i < m) {
      y[i] = yi;
      d = (double)v[i] * (double)yi;
    }
    d = block_sum(d, sm);
    if (threadIdx.x == 0) red[blockIdx.x] = d;
  } else if (EPI == EPI_DOT2) {
    double d = 0.0, e = 0.0;
    if (i < m) {
      y[i] = yi;
      d = (double)v[i] * (double)yi;
      e = (double)yi * (double)yi;
    }
    d = block_sum(d, sm);
    e = block_sum(e, sm);
    if (threadIdx.x == 0) {
      red[blockIdx.x] = d;
      red[gridDim.x + blockIdx.x] = e;
    }
  } else if (EPI == EPI_RESID) {
    // r = axpy(-1, A x, b) = b - A x  (krylov.py:47,104: one rounding, the -1 is exact)
    Ssq q{0.0, 0.0};
    double p2 = 0.0;
    if (i < m) {
      const T r = sub_rn(v[i], yi);
      y[i] = r;
      q = ssq_add(q, (double)r);
      p2 = (double)r * (double)r;
    }
    Ssq b = block_ssq(q, sm);
    p2 = block_sum(p2, sm);
    if (threadIdx.x == 0) {
      red[2 * blockIdx.x] = b.scale;
      red[2 * blockIdx.x + 1] = b.ssq;
      red[2 * gridDim.x + blockIdx.x] = p2;
    }
  } else if (EPI == EPI_AXPY_INTO) {
    // x = axpy(1.0, V y, x) = x + 1.0*(V y)   (krylov.py:167)
    if (i < m) y[i] = add_rn(y[i], yi);
  }
}

template <typename T>
int gemv_launch(ds_ctx* ctx, const GemvPlan& p, const T* A, int64_t lda, const T* x, T* y,
                double* part, GemvEpi epi, const T* v, double* red, int* red_blocks,
                Gate stop) {
  const int64_t m = p.m, n = p.n;
  const int rblocks = (int)ceil_div(std::max<int64_t>(m, 1), kRedThreads);
  if (red_blocks) *red_blocks = rblocks;
  if (m == 0) return DS_OK;
  if (n == 0) {
    // A x = 0: run the reduce kernel over a zeroed partial row
    DS_CUDA(cudaMemsetAsync(part, 0, (size_t)m * sizeof(double), ctx->stream));
  } else {
    dim3 grid((unsigned)p.rowtiles, (unsigned)p.nchunks);
    const size_t smem = (size_t)p.chunk * sizeof(T);
    constexpr int VEC = sizeof(T) == 8 ? 2 : 4;
    const bool aligned = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (lda % VEC == 0);
    if (aligned) {
      ds_colstream_mv_kernel<T, VEC, 8>
          <<<grid, kGemvThreads, smem, ctx->stream>>>(A, lda, m, n, x, p.chunk, part, stop);
    } else {
      dim3 g1((unsigned)ceil_div(m, kGemvThreads), (unsigned)p.nchunks);
      ds_colstream_mv_kernel<T, 1, 8>
          <<<g1, kGemvThreads, smem, ctx->stream>>>(A, lda, m, n, x, p.chunk, part, stop);
    }
    count_launch(ctx);
    DS_CHECK_LAUNCH();
  }
  if (epi == EPI_PARTIAL) return DS_OK;
  const int64_t nch = n == 0 ? 1 : p.nchunks;
  switch (epi) {
    case EPI_STORE:
      ds_colstream_reduce_kernel<T, EPI_STORE>
          <<<rblocks, kRedThreads, 0, ctx->stream>>>(part, m, nch, y, v, red, stop);
      break;
    case EPI_DOT:
      ds_colstream_reduce_kernel<T, EPI_DOT>
          <<<rblocks, kRedThreads, 0, ctx->stream>>>(part, m, nch, y, v, red, stop);
      break;
    case EPI_RESID:
      ds_colstream_reduce_kernel<T, EPI_RESID>
          <<<rblocks, kRedThreads, 0, ctx->stream>>>(part, m, nch, y, v, red, stop);
      break;
    case EPI_AXPY_INTO:
      ds_colstream_reduce_kernel<T, EPI_AXPY_INTO>
          <<<rblocks, kRedThreads, 0, ctx->stream>>>(part, m, nch, y, v, red, stop);
      break;
    case EPI_DOT2:
      ds_colstream_reduce_kernel<T, EPI_DOT2>
          <<<rblocks, kRedThreads, 0, ctx->stream>>>(part, m, nch, y, v, red, stop);
      break;
    default:
      break;
  }
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

template <typename T>
int gemv_partial_pdl_launch(ds_ctx* ctx, const GemvPlan& p, const T* A, int64_t lda, const T* x, double* part,
                            Gate stop) {
  constexpr int VEC = sizeof(T) == 8 ? 2 : 4;
  const bool aligned = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (lda % VEC == 0);
  if (p.m == 0 || p.n == 0 || !aligned)
    return gemv_launch<T>(ctx, p, A, lda, x, nullptr, part, EPI_PARTIAL, nullptr, nullptr, nullptr, stop);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)p.rowtiles, (unsigned)p.nchunks);
  lc.blockDim = dim3(kGemvThreads);
  lc.dynamicSmemBytes = (size_t)p.chunk * sizeof(T);
  lc.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const int64_t m = p.m, n = p.n, chunk = p.chunk;
  DS_CUDA(cudaLaunchKernelEx(&lc, ds_colstream_mv_kernel<T, VEC, 8>, A, lda, m, n, x, chunk, part, stop));
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
template int gemv_partial_pdl_launch<double>(ds_ctx*, const GemvPlan&, const double*, int64_t, const double*, double*,
                                             Gate);
template int gemv_partial_pdl_launch<float>(ds_ctx*, const GemvPlan&, const float*, int64_t, const float*, double*,
                                            Gate);
template int gemv_launch<double>(ds_ctx*, const GemvPlan&, const double*, int64_t, const double*,
                                 double*, double*, GemvEpi, const double*, double*, int*,
                                 Gate);
template int gemv_launch<float>(ds_ctx*, const GemvPlan&, const float*, int64_t, const float*,
                                float*, double*, GemvEpi, const float*, double*, int*, Gate);

// ============================================================================
// level-1 reductions
// ============================================================================
int reduce_grid(ds_ctx* ctx, int64_t n) {
  int64_t want = ceil_div(std::max<int64_t>(n, 1), (int64_t)kRedThreads * 4);
  return (int)std::min<int64_t>(want, (int64_t)ctx->num_sms * 4);
}

template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    dot_kernel(int64_t n, const T* __restrict__ x, const T* __restrict__ y, double* red) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = fma((double)x[i], (double)y[i], s);
  s = block_sum(s, sm);
  if (threadIdx.x == 0) red[blockIdx.x] = s;
}

template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    ssq_kernel(int64_t n, const T* __restrict__ x, double* red) {
  __shared__ double sm[64];
  Ssq q{0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    q = ssq_add(q, (double)x[i]);
  q = block_ssq(q, sm);
  if (threadIdx.x == 0) {
    red[2 * blockIdx.x] = q.scale;
    red[2 * blockIdx.x + 1] = q.ssq;
  }
}

__global__ void finish_sum_kernel(const double* red, int nblk, double* out) {
  __shared__ double sm[32];
  double s = reduce_sum_partials(red, nblk, sm);
  if (threadIdx.x == 0) out[0] = s;
}

__global__ void finish_ssq_kernel(const double* red, int nblk, double* out) {
  __shared__ double sm[64];
  Ssq q{0.0, 0.0};
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) q = ssq_merge(q, Ssq{red[2 * i], red[2 * i + 1]});
  q = block_ssq(q, sm);
  if (threadIdx.x == 0) out[0] = ssq_norm(q.scale, q.ssq);
}

template <typename T>
int dot_launch(ds_ctx* ctx, int64_t n, const T* x, const T* y, double* red, int* nblk) {
  int g = reduce_grid(ctx, n);
  *nblk = g;
  dot_kernel<T><<<g, kRedThreads, 0, ctx->stream>>>(n, x, y, red);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
template <typename T>
int ssq_launch(ds_ctx* ctx, int64_t n, const T* x, double* red, int* nblk) {
  int g = reduce_grid(ctx, n);
  *nblk = g;
  ssq_kernel<T><<<g, kRedThreads, 0, ctx->stream>>>(n, x, red);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
int finish_sum(ds_ctx* ctx, const double* red, int nblk, double* out) {
  finish_sum_kernel<<<1, kRedThreads, 0, ctx->stream>>>(red, nblk, out);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
int finish_ssq(ds_ctx* ctx, const double* red, int nblk, double* out) {
  finish_ssq_kernel<<<1, kRedThreads, 0, ctx->stream>>>(red, nblk, out);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
template int dot_launch<double>(ds_ctx*, int64_t, const double*, const double*, double*, int*);
template int dot_launch<float>(ds_ctx*, int64_t, const float*, const float*, double*, int*);
template int ssq_launch<double>(ds_ctx*, int64_t, const double*, double*, int*);
template int ssq_launch<float>(ds_ctx*, int64_t, const float*, double*, int*);

// iamax: first index of the maximum |x|; NaN wins (first NaN), ties -> lowest
// index (np.argmax(np.abs(x)), backends.py:128-132).
__device__ __forceinline__ bool iamax_better(double av, int64_t ai, double bv, int64_t bi) {
  const bool an = av != av, bn = bv != bv;
  if (an || bn) {
    if (an && bn) return ai < bi;
    return an;
  }
  if (av != bv) return av > bv;
  return ai < bi;
}

template <typename T>
__global__ void __launch_bounds__(kRedThreads)
    iamax_kernel(int64_t n, const T* __restrict__ x, double* red_v, int64_t* red_i) {
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  double bv = -1.0;
  int64_t bi = INT64_MAX;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = fabs((double)x[i]);
    if (iamax_better(v, i, bv, bi)) {
      bv = v;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (iamax_better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sv[wid] = bv;
    si[wid] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (iamax_better(sv[w], si[w], bv, bi)) {
        bv = sv[w];
        bi = si[w];
      }
    red_v[blockIdx.x] = bv;
    red_i[blockIdx.x] = bi;
  }
}

__global__ void iamax_finish_kernel(const double* red_v, const int64_t* red_i, int nblk,
                                    int64_t* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int b = 0; b < nblk; ++b)
      if (iamax_better(red_v[b], red_i[b], bv, bi)) {
        bv = red_v[b];
        bi = red_i[b];
      }
    out[0] = bi;
  }
}

// ============================================================================
// elementwise ops (NumPy rounding: alpha cast to the array dtype, NEP 50)
// ============================================================================
template <typename T>
__global__ void axpy_kernel(int64_t n, T alpha, const T* __restrict__ x, const T* y, T* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = add_rn(y[i], mul_rn(alpha, x[i]));
}
template <typename T>
__global__ void scal_kernel(int64_t n, T alpha, const T* x, T* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mul_rn(alpha, x[i]);
}

static int ew_grid(ds_ctx* ctx, int64_t n) {
  int64_t want = ceil_div(std::max<int64_t>(n, 1), 256);
  return (int)std::min<int64_t>(want, (int64_t)ctx->num_sms * 8);
}

template <typename T>
int axpy_launch(ds_ctx* ctx, int64_t n, double alpha, const T* x, const T* y, T* out) {
  if (n == 0) return DS_OK;
  axpy_kernel<T><<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, (T)alpha, x, y, out);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
template <typename T>
int scal_launch(ds_ctx* ctx, int64_t n, double alpha, const T* x, T* out) {
  if (n == 0) return DS_OK;
  scal_kernel<T><<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, (T)alpha, x, out);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
template int axpy_launch<double>(ds_ctx*, int64_t, double, const double*, const double*, double*);
template int axpy_launch<float>(ds_ctx*, int64_t, double, const float*, const float*, float*);
template int scal_launch<double>(ds_ctx*, int64_t, double, const double*, double*);
template int scal_launch<float>(ds_ctx*, int64_t, double, const float*, float*);

// ============================================================================
// GER: out = A + alpha * outer(x, y)   (backends.py:144-156)
//   outer element rounded, times alpha rounded, then added: three roundings,
//   exactly NumPy's `A + alpha * np.outer(x, y)`.
// ============================================================================
template <typename T>
__global__ void ger_kernel(int64_t m, int64_t n, const T* A, int64_t lda, T alpha,
                           const T* __restrict__ x, const T* __restrict__ y, T* out, int64_t ldo) {
  const int64_t total = m * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % m, j = t / m;
    out[i + j * ldo] = add_rn(A[i + j * lda], mul_rn(alpha, mul_rn(x[i], y[j])));
  }
}
template <typename T>
int ger_launch(ds_ctx* ctx, int64_t m, int64_t n, const T* A, int64_t lda, double alpha,
               const T* x, const T* y, T* out, int64_t ldo) {
  if (m == 0 || n == 0) return DS_OK;
  ger_kernel<T><<<ew_grid(ctx, m * n), 256, 0, ctx->stream>>>(m, n, A, lda, (T)alpha, x, y, out,
                                                              ldo);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
template int ger_launch<double>(ds_ctx*, int64_t, int64_t, const double*, int64_t, double,
                                const double*, const double*, double*, int64_t);
template int ger_launch<float>(ds_ctx*, int64_t, int64_t, const float*, int64_t, double,
                               const float*, const float*, float*, int64_t);

// ============================================================================
// symmetry gate (krylov.py:41-44): max|A - A^T| (difference rounded in T, as
// NumPy's A - A.T) and max|A|, over upper-triangular 32x32 tile pairs.
// ============================================================================
// max|A - A^T| and max|A| (krylov.py:42-44) over 64 x 64 tile pairs (bi <= bj): every
// thread issues its 32 loads of both tiles at once (512-byte column runs), then the
// transposed tile goes through shared memory.  Each element is read once.
constexpr int kSymT = 64;
template <typename T>
__global__ void __launch_bounds__(256)
    symcheck_kernel(int64_t n, const T* __restrict__ A, int64_t lda, double* red) {
  __shared__ T tu[kSymT][kSymT + 1];  // the transposed tile; the (bi,bj) tile stays in registers
  __shared__ double sm[32];
  const int64_t nt = ceil_div(n, (int64_t)kSymT);
  const int64_t npairs = nt * (nt + 1) / 2;
  double dmax = 0.0, amax = 0.0;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  for (int64_t p = blockIdx.x; p < npairs; p += gridDim.x) {
    // p -> (bi, bj) with bi <= bj, row-major over the upper triangle
    int64_t bi = (int64_t)((2.0 * nt + 1.0 - sqrt((2.0 * nt + 1.0) * (2.0 * nt + 1.0) - 8.0 * p)) / 2.0);
    if (bi < 0) bi = 0;
    while (bi > 0 && bi * nt - bi * (bi - 1) / 2 > p) --bi;
    while ((bi + 1) * nt - (bi + 1) * bi / 2 <= p) ++bi;
    const int64_t bj = bi + (p - (bi * nt - bi * (bi - 1) / 2));
    const int64_t r0 = bi * kSymT, c0 = bj * kSymT;
    T vl[kSymT / 4], vu[kSymT / 4];
#pragma unroll
    for (int q = 0; q < kSymT / 4; ++q) {
      const int k = ty + 4 * q;
      const int64_t r = r0 + tx, c = c0 + k;    // tile (bi,bj): element (r, c)
      vl[q] = (r < n && c < n) ? A[r + c * lda] : T(0);
      const int64_t r2 = c0 + tx, c2 = r0 + k;  // tile (bj,bi): element (r2, c2)
      vu[q] = (r2 < n && c2 < n) ? A[r2 + c2 * lda] : T(0);
    }
    __syncthreads();  // the previous pair's compare is done with the tiles
#pragma unroll
    for (int q = 0; q < kSymT / 4; ++q) {
      tu[ty + 4 * q][tx] = vu[q];
      amax = nanmax(amax, fabs((double)vl[q]));
      amax = nanmax(amax, fabs((double)vu[q]));
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kSymT / 4; ++q) {
      const int k = ty + 4 * q;
      // element (r0+tx, c0+k) vs its transpose (c0+k, r0+tx) = tu[tx][k]
      dmax = nanmax(dmax, fabs((double)sub_rn(vl[q], tu[tx][k])));
    }
  }
  dmax = block_nanmax(dmax, sm);
  amax = block_nanmax(amax, sm);
  if (threadIdx.x == 0) {
    red[2 * blockIdx.x] = dmax;
    red[2 * blockIdx.x + 1] = amax;
  }
}

template <typename T>
int symcheck_launch(ds_ctx* ctx, int64_t n, const T* A, int64_t lda, double* red, int* nblk) {
  const int64_t nt = ceil_div(n, (int64_t)kSymT);
  const int64_t npairs = nt * (nt + 1) / 2;
  int g = (int)std::min<int64_t>(npairs, (int64_t)ctx->num_sms * 6);  // 6 x 33 KB smem per SM
  *nblk = g;
  symcheck_kernel<T><<<g, 256, 0, ctx->stream>>>(n, A, lda, red);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
template int symcheck_launch<double>(ds_ctx*, int64_t, const double*, int64_t, double*, int*);
template int symcheck_launch<float>(ds_ctx*, int64_t, const float*, int64_t, double*, int*);

__global__ void finish_max2_kernel(const double* red, int nblk, double* out) {
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

// ============================================================================
// GEMM — FP64 on the DMMA tensor pipe.  out = beta*C + alpha*(A B).
//   CTA tile 128x64, 8 warps (4x2) of 32x32, BK=16 k-slab, 4-stage cp.async pipeline with
//   per-stage full/empty mbarriers (no CTA barrier per slab: 32.2 -> 32.8 TFLOP/s at K=512)
//   (96 KB, 2 CTAs/SM; 4 stages measured 32.3 vs 31.4 TFLOP/s for 3 at K = 512),
//   mma.sync.m8n8k4.row.col.f64 (native DMMA.8x8x4; the only FP64 tensor-core
//   instruction on sm_100a — tcgen05 has no kind::f64).
// ============================================================================
namespace gemm64 {
constexpr int BM = 128, BN = 64, BK = 16, STAGES = 4;
// warp tile WR x 32: 8 warps of 32 x 32 (4 warps per SM sub-partition at 2 CTAs/SM)
constexpr int WR = 32, MI = WR / 8, WARPS_M = BM / WR, THREADS = WARPS_M * (BN / 32) * 32;
constexpr int LDA_S = BM + 4;  // smem row (one k) of the A slab, +4 doubles: conflict-free frags
constexpr int LDB_S = BK + 4;  // smem row (one n) of the B slab
constexpr int A_STAGE = BK * LDA_S;
constexpr int B_STAGE = BN * LDB_S;
constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
}  // namespace gemm64

__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void mbar_init_cta(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cta(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra WAIT_%=;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}
// the mbarrier receives one arrival once all of this thread's prior cp.async copies land
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool VEC16>
__device__ __forceinline__ void gemm64_load_stage(double* As, double* Bs, const double* A,
                                                  int64_t lda, const double* B, int64_t ldb,
                                                  int64_t m, int64_t n, int64_t k, int64_t m0,
                                                  int64_t n0, int64_t k0) {
  using namespace gemm64;
  const int tid = threadIdx.x;
  if (VEC16) {
    // A slab: BK columns x BM rows, 2 doubles per 16 B chunk -> BK*BM/2 chunks
#pragma unroll
    for (int it = 0; it < (BK * BM / 2) / THREADS; ++it) {
      const int c = tid + it * THREADS;
      const int kk = c / (BM / 2), mm = (c % (BM / 2)) * 2;
      const int64_t gr = m0 + mm, gk = k0 + kk;
      int bytes = 0;
      if (gk < k) bytes = gr + 1 < m ? 16 : (gr < m ? 8 : 0);
      const double* src = bytes ? A + gk * lda + gr : A;
      cp_async_16(As + kk * LDA_S + mm, src, bytes);
    }
    // B slab: BN columns x BK rows
#pragma unroll
    for (int it = 0; it < (BK * BN / 2) / THREADS; ++it) {
      const int c = tid + it * THREADS;
      const int nn = c / (BK / 2), kk = (c % (BK / 2)) * 2;
      const int64_t gk = k0 + kk, gc = n0 + nn;
      int bytes = 0;
      if (gc < n) bytes = gk + 1 < k ? 16 : (gk < k ? 8 : 0);
      const double* src = bytes ? B + gc * ldb + gk : B;
      cp_async_16(Bs + nn * LDB_S + kk, src, bytes);
    }
  } else {
#pragma unroll 4
    for (int it = 0; it < (BK * BM) / THREADS; ++it) {
      const int c = tid + it * THREADS;
      const int kk = c / BM, mm = c % BM;
      const int64_t gr = m0 + mm, gk = k0 + kk;
      const bool ok = gk < k && gr < m;
      cp_async_8(As + kk * LDA_S + mm, ok ? A + gk * lda + gr : A, ok ? 8 : 0);
    }
#pragma unroll 4
    for (int it = 0; it < (BK * BN) / THREADS; ++it) {
      const int c = tid + it * THREADS;
      const int nn = c / BK, kk = c % BK;
      const int64_t gk = k0 + kk, gc = n0 + nn;
      const bool ok = gc < n && gk < k;
      cp_async_8(Bs + nn * LDB_S + kk, ok ? B + gc * ldb + gk : B, ok ? 8 : 0);
    }
  }
}

template <bool VEC16, int MODE /*0: general, 1: out = C - AB*/>
__global__ void __launch_bounds__(gemm64::THREADS, 2)
    gemm64_kernel(int64_t m, int64_t n, int64_t k, double alpha, const double* __restrict__ A,
                  int64_t lda, const double* __restrict__ B, int64_t ldb, double beta,
                  const double* C, int64_t ldc, double* out, int64_t ldo, int tri) {
  using namespace gemm64;
  // tri: only tiles holding some row >= column (the lower-triangle SYRK update of
  // the Cholesky trailing matrix, direct.py:117-119); tiles strictly above exit
  if (tri && (int64_t)(blockIdx.x + 1) * BM <= (int64_t)blockIdx.y * BN) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);
  double* Bs = As + STAGES * A_STAGE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int g = lane >> 2, t = lane & 3;

  // MODE 1 (out = C - A B, the LU update): the accumulators start from C (loaded
  // before the main loop, so its latency hides under the cp.async prologue) and
  // the A fragments are negated, making the epilogue store-only.
  double acc[MI][4][2];
  if (MODE == 1) {
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int64_t r = m0 + wm * WR + i * 8 + g;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + wn * 32 + j * 8 + 2 * t + e;
          acc[i][j][e] = (r < m && c < n) ? C[r + c * ldc] : 0.0;
        }
    }
  } else {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }
  const int64_t ktiles = ceil_div(k, BK);
  // per-stage mbarriers instead of one CTA barrier per k-slab: full[s] completes when every
  // thread's cp.async copies of the slab have landed (cp.async.mbarrier.arrive.noinc), empty[s]
  // when all 8 warps have read it, so warps drift up to STAGES - 1 slabs apart
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init_cta(&full_bar[s], THREADS);
      mbar_init_cta(&empty_bar[s], THREADS / 32);
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) {
      gemm64_load_stage<VEC16>(As + s * A_STAGE, Bs + s * B_STAGE, A, lda, B, ldb, m, n, k, m0, n0,
                               (int64_t)s * BK);
      cp_async_mbar_arrive(&full_bar[s]);
    }
  }
  // interior tiles (the bulk of every LU / SYRK update): the cp.async sources are two
  // running pointers plus constant strides, no per-chunk index math or bounds checks
  const bool interior = VEC16 && m0 + BM <= m && n0 + BN <= n;
  const int tid = threadIdx.x;
  const double* a_src = A + (int64_t)(tid / (BM / 2)) * lda + m0 + (tid % (BM / 2)) * 2;  // chunk it: + it * 4 lda
  const double* b_src = B + (n0 + tid / (BK / 2)) * ldb + (tid % (BK / 2)) * 2;             // chunk it: + it * 32 ldb
  const int a_dst = (tid / (BM / 2)) * LDA_S + (tid % (BM / 2)) * 2;
  const int b_dst = (tid / (BK / 2)) * LDB_S + (tid % (BK / 2)) * 2;
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    mbar_wait_cta(&full_bar[kt % STAGES], (unsigned)((kt / STAGES) & 1));
    // prefetch slab kt + STAGES - 1 into the stage every warp released at iteration kt - 1
    const int64_t pf = kt + STAGES - 1;
    if (pf < ktiles) {
      const int s = (int)(pf % STAGES);
      if (kt >= 1) mbar_wait_cta(&empty_bar[s], (unsigned)(((kt - 1) / STAGES) & 1));
      if (interior && (pf + 1) * BK <= k) {
        const int64_t k0 = pf * BK;
        const double* ap = a_src + k0 * lda;
        const double* bp = b_src + k0;
        double* as_ = As + s * A_STAGE + a_dst;
        double* bs_ = Bs + s * B_STAGE + b_dst;
#pragma unroll
        for (int it = 0; it < (BK * BM / 2) / THREADS; ++it)
          cp_async_16(as_ + it * (THREADS / (BM / 2)) * LDA_S, ap + (int64_t)it * (THREADS / (BM / 2)) * lda, 16);
#pragma unroll
        for (int it = 0; it < (BK * BN / 2) / THREADS; ++it)
          cp_async_16(bs_ + it * (THREADS / (BK / 2)) * LDB_S, bp + (int64_t)it * (THREADS / (BK / 2)) * ldb, 16);
      } else {
        gemm64_load_stage<VEC16>(As + s * A_STAGE, Bs + s * B_STAGE, A, lda, B, ldb, m, n, k, m0, n0,
                                 pf * BK);
      }
      cp_async_mbar_arrive(&full_bar[s]);
    }
    const int s = (int)(kt % STAGES);
    const double* as = As + s * A_STAGE + wm * WR + g;
    const double* bs = Bs + s * B_STAGE + (wn * 32 + g) * LDB_S + t;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[MI], b[4];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = MODE == 1 ? -as[(kk + t) * LDA_S + i * 8] : as[(kk + t) * LDA_S + i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[j * 8 * LDB_S + kk];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&empty_bar[s]);
  }
  cp_async_wait<0>();
  // epilogue.  MODE 1: acc already holds C - A B.  MODE 0: out = beta*C + alpha*acc
  // with NumPy's rounding (backends.py:244); C is read in one batch per row group
  // before any store so the loads overlap.
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t r = m0 + wm * WR + i * 8 + g;
    if (r >= m) continue;
    double cv[4][2];
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + wn * 32 + j * 8 + 2 * t + e;
          cv[j][e] = (c < n && beta != 0.0) ? C[r + c * ldc] : 0.0;
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn * 32 + j * 8 + 2 * t + e;
        if (c >= n) continue;
        double o;
        if (MODE == 1) {
          o = acc[i][j][e];
        } else {
          const double cb = beta == 0.0 ? 0.0 : __dmul_rn(beta, cv[j][e]);
          o = __dadd_rn(cb, __dmul_rn(alpha, acc[i][j][e]));
        }
        out[r + c * ldo] = o;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// TMA-fed variant (the default for 16-byte aligned operands with even leading
// dimensions): the A and B slabs are moved by the tensor-memory accelerator
// (cp.async.bulk.tensor, 128-byte swizzle) into a 4-stage ring; one elected thread
// issues the copies and arms the stage's full mbarrier with the byte count, the 8
// compute warps release a stage through its empty mbarrier.  No per-thread address
// math or LDGSTS in the main loop, and out-of-range rows/columns/k are zero-filled
// by the TMA unit (no ragged-tile code).  Same CTA/warp tiling and the same DMMA
// sequence per output element as gemm64_kernel, so results are bitwise equal.
//   A stage: 8 boxes of 16 (m) x 16 (k), box b at b*2 KB, row k = 128 B, 16-byte chunk
//            index (m/2) ^ (k & 7)          (SWIZZLE_128B, stage base 1024-B aligned)
//   B stage: 64 rows (n) of 16 (k) doubles, chunk index (k/2) ^ (n & 7)
// ---------------------------------------------------------------------------
namespace gemm64 {
constexpr int A_TMA_BYTES = BM * BK * 8;  // 16 KB
constexpr int B_TMA_BYTES = BN * BK * 8;  // 8 KB
constexpr int STAGE_TMA_BYTES = A_TMA_BYTES + B_TMA_BYTES;
constexpr size_t SMEM_TMA = (size_t)STAGES * STAGE_TMA_BYTES + 1024;  // + alignment slack
}  // namespace gemm64

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}

template <int MODE /*0: general, 1: out = C - AB*/>
__global__ void __launch_bounds__(gemm64::THREADS, 2)
    gemm64_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t m,
                      int64_t n, int64_t k, double alpha, double beta, const double* C, int64_t ldc, double* out,
                      int64_t ldo, int tri) {
  using namespace gemm64;
  if (tri && (int64_t)(blockIdx.x + 1) * BM <= (int64_t)blockIdx.y * BN) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int g = lane >> 2, t = lane & 3;
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  const int64_t ktiles = ceil_div(k, BK);
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init_cta(&full_bar[s], 1);
      mbar_init_cta(&empty_bar[s], THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t kt) {  // one thread: arm full[s] and copy slab kt
    const int s = (int)(kt % STAGES);
    unsigned char* st = sm + (size_t)s * STAGE_TMA_BYTES;
    mbar_arrive_expect_tx(&full_bar[s], STAGE_TMA_BYTES);
    const int kc = (int)(kt * BK);
#pragma unroll
    for (int b = 0; b < BM / 16; ++b) tma_load_2d(st + b * 2048, &tmA, (int)(m0 + 16 * b), kc, &full_bar[s]);
    tma_load_2d(st + A_TMA_BYTES, &tmB, kc, (int)n0, &full_bar[s]);
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES - 1; ++s)
      if (s < ktiles) issue(s);

  double acc[MI][4][2];
  if (MODE == 1) {  // accumulators start from C (the LU update out = C - A B, A negated)
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int64_t r = m0 + wm * WR + i * 8 + g;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + wn * 32 + j * 8 + 2 * t + e;
          acc[i][j][e] = (r < m && c < n) ? C[r + c * ldc] : 0.0;
        }
    }
  } else {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }
  // per-lane swizzled fragment offsets (bytes within a stage), see the layout above
  const unsigned a_lane = (unsigned)(wm * 2) * 2048u + (unsigned)t * 128u + ((unsigned)((g >> 1) ^ t) << 4) +
                          ((unsigned)(g & 1) << 3);
  unsigned b_lane[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    b_lane[q] = (unsigned)A_TMA_BYTES + (unsigned)(wn * 32 + g) * 128u +
                ((unsigned)(((t >> 1) ^ g) ^ (2 * q)) << 4) + ((unsigned)(t & 1) << 3);

  for (int64_t kt = 0; kt < ktiles; ++kt) {
    if (warp == 0) {
      if (lane == 0) {
        const int64_t pf = kt + STAGES - 1;  // refill the stage every warp released at kt - 1
        if (pf < ktiles) {
          if (kt >= 1) mbar_wait_cta(&empty_bar[pf % STAGES], (unsigned)(((kt - 1) / STAGES) & 1));
          issue(pf);
        }
      }
      __syncwarp();
    }
    const int s = (int)(kt % STAGES);
    mbar_wait_cta(&full_bar[s], (unsigned)((kt / STAGES) & 1));
    const unsigned char* st = sm + (size_t)s * STAGE_TMA_BYTES;
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) {
      double a[MI], b[4];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const unsigned off = a_lane + (unsigned)(i >> 1) * 2048u + (unsigned)q * 512u +
                             ((unsigned)(((i & 1) << 2) ^ ((q & 1) << 2)) << 4);
        const double v = *reinterpret_cast<const double*>(st + off);
        a[i] = MODE == 1 ? -v : v;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = *reinterpret_cast<const double*>(st + b_lane[q] + (unsigned)j * 1024u);
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    // Release the stage to the TMA unit: this thread's generic-proxy reads of it are ordered
    // before the async-proxy writes that refill it (without the proxy fence the refill raced
    // with fragment loads still in flight under concurrent kernels: rare, wrong products)
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&empty_bar[s]);
  }
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t r = m0 + wm * WR + i * 8 + g;
    if (r >= m) continue;
    double cv[4][2];
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + wn * 32 + j * 8 + 2 * t + e;
          cv[j][e] = (c < n && beta != 0.0) ? C[r + c * ldc] : 0.0;
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn * 32 + j * 8 + 2 * t + e;
        if (c >= n) continue;
        double o;
        if (MODE == 1) {
          o = acc[i][j][e];
        } else {
          const double cb = beta == 0.0 ? 0.0 : __dmul_rn(beta, cv[j][e]);
          o = __dadd_rn(cb, __dmul_rn(alpha, acc[i][j][e]));
        }
        out[r + c * ldo] = o;
      }
    }
  }
}

// Persistent form of gemm64_tma_kernel<1> (out = C - A B) for the LU trailing update that
// runs beside the look-ahead panel on the side stream.  A CTA that lands on one of the
// first `reserve` SMs leaves at once (unless no worker has registered yet), so the side
// stream's panel and inner kernels find those SMs free instead of waiting for trailing-GEMM
// CTAs (~67 us each at K = 512) to retire.  The workers take 128 x 64 tiles from a device
// counter in the non-persistent kernel's order (m fastest); the elected producer thread
// claims the tiles, passes their indices to the compute warps through a shared-memory queue
// published by the stage's full mbarrier, and keeps the TMA ring full across tile
// boundaries (slab counters run over the CTA's whole tile sequence); a sentinel index ends
// the loop.  Per tile the same accumulator start (C), DMMA sequence and store: bitwise equal
// to the non-persistent kernel.
//   ctr[0]: next tile, ctr[1]: registered workers (both zeroed before the launch)
__global__ void __launch_bounds__(gemm64::THREADS, 2)
    gemm64_tma_persist_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                              int64_t m, int64_t n, int64_t k, const double* C, int64_t ldc, double* out,
                              int64_t ldo, int reserve, unsigned* ctr) {
  using namespace gemm64;
  constexpr int Q = 8;  // tile-index queue (the producer runs <= STAGES - 1 slabs ahead)
  __shared__ int tile_q[Q];
  __shared__ int s_work;
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;\n" : "=r"(smid));
    int work = (int)smid >= reserve;
    if (!work) work = atomicAdd(&ctr[1], 0u) == 0u;  // never leave the tiles without a worker
    if (work) atomicAdd(&ctr[1], 1u);
    s_work = work;
  }
  __syncthreads();
  if (!s_work) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int g = lane >> 2, t = lane & 3;
  const int64_t ktiles = ceil_div(k, BK);
  const int64_t mtiles = ceil_div(m, BM);
  const int64_t ntiles = mtiles * ceil_div(n, BN);
  // producer state (thread 0 only; in shared memory to keep the compute warps' registers):
  // slabs issued, slab within the current tile, current tile, tile ordinal, done
  __shared__ int p_cnt, p_kt, p_tile, p_j, p_done;
  auto produce = [&]() {  // issue the next slab (or the sentinel) into ring slot p_cnt
    if (p_done) return;
    const int s = p_cnt % STAGES;
    if (p_cnt >= STAGES) mbar_wait_cta(&empty_bar[s], (unsigned)(((p_cnt - STAGES) / STAGES) & 1));
    if (p_kt == (int)ktiles) {  // claim the next tile
      const unsigned tl = atomicAdd(&ctr[0], 1u);
      if ((int64_t)tl >= ntiles) {
        tile_q[p_j % Q] = -1;
        mbar_arrive_cta(&full_bar[s]);  // releases the sentinel (count 1, no bytes)
        p_done = 1;
        ++p_cnt;
        return;
      }
      p_tile = (int)tl;
      tile_q[p_j % Q] = p_tile;
      ++p_j;
      p_kt = 0;
    }
    unsigned char* st = sm + (size_t)s * STAGE_TMA_BYTES;
    mbar_arrive_expect_tx(&full_bar[s], STAGE_TMA_BYTES);
    const int kc = p_kt * BK;
    const int pm0 = (int)((p_tile % mtiles) * BM), pn0 = (int)((p_tile / mtiles) * BN);
#pragma unroll
    for (int b = 0; b < BM / 16; ++b) tma_load_2d(st + b * 2048, &tmA, pm0 + 16 * b, kc, &full_bar[s]);
    tma_load_2d(st + A_TMA_BYTES, &tmB, kc, pn0, &full_bar[s]);
    ++p_kt;
    ++p_cnt;
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init_cta(&full_bar[s], 1);
      mbar_init_cta(&empty_bar[s], THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    p_cnt = 0;
    p_kt = (int)ktiles;
    p_tile = 0;
    p_j = 0;
    p_done = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES - 1; ++s) produce();

  const unsigned a_lane = (unsigned)(wm * 2) * 2048u + (unsigned)t * 128u + ((unsigned)((g >> 1) ^ t) << 4) +
                          ((unsigned)(g & 1) << 3);
  unsigned b_lane[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    b_lane[q] = (unsigned)A_TMA_BYTES + (unsigned)(wn * 32 + g) * 128u +
                ((unsigned)(((t >> 1) ^ g) ^ (2 * q)) << 4) + ((unsigned)(t & 1) << 3);
  int c_cnt = 0;  // slabs consumed
  for (int jc = 0;; ++jc) {
    mbar_wait_cta(&full_bar[c_cnt % STAGES], (unsigned)((c_cnt / STAGES) & 1));  // first slab of tile jc
    const int tile = tile_q[jc % Q];
    if (tile < 0) break;
    const int64_t m0 = (tile % mtiles) * BM, n0 = (tile / mtiles) * BN;
    double acc[MI][4][2];
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int64_t r = m0 + wm * WR + i * 8 + g;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + wn * 32 + j * 8 + 2 * t + e;
          acc[i][j][e] = (r < m && c < n) ? C[r + c * ldc] : 0.0;
        }
    }
    for (int kt = 0; kt < (int)ktiles; ++kt, ++c_cnt) {
      if (warp == 0) {
        if (lane == 0) produce();  // slab c_cnt + STAGES - 1 (its slot was released at c_cnt - 1)
        __syncwarp();
      }
      const int s = (int)(c_cnt % STAGES);
      if (kt > 0) mbar_wait_cta(&full_bar[s], (unsigned)((c_cnt / STAGES) & 1));
      const unsigned char* st = sm + (size_t)s * STAGE_TMA_BYTES;
#pragma unroll
      for (int q = 0; q < BK / 4; ++q) {
        double a[MI], b[4];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const unsigned off = a_lane + (unsigned)(i >> 1) * 2048u + (unsigned)q * 512u +
                               ((unsigned)(((i & 1) << 2) ^ ((q & 1) << 2)) << 4);
          a[i] = -*reinterpret_cast<const double*>(st + off);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = *reinterpret_cast<const double*>(st + b_lane[q] + (unsigned)j * 1024u);
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty_bar[s]);
    }
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int64_t r = m0 + wm * WR + i * 8 + g;
      if (r >= m) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + wn * 32 + j * 8 + 2 * t + e;
          if (c < n) out[r + c * ldo] = acc[i][j][e];
        }
    }
  }
}

// Host side: the driver's tensor-map encoder, resolved once through the runtime (no
// libcuda link).  A 2-D map of a column-major matrix: dim 0 = rows (contiguous), dim 1 =
// columns, box {16, box_cols}, 128-byte swizzle, out-of-range elements zero-filled.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn tensor_map_encoder() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
static bool encode_colmajor_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                                unsigned box_rows, unsigned box_cols) {
  EncodeTiledFn enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  const cuuint32_t box[2] = {box_rows, box_cols};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool gemm_tma_enabled() {
  static const bool on = [] {
    const char* e = getenv("DENSOLVE_GEMM_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

// FP32 GEMM, large tiles (the fp32 LU / Cholesky trailing update): CTA tile 128 x 128,
// k-slab 8, 256 threads of 8 x 8 outputs (two 4 x 4 quadrants per dimension, so the
// fragment reads are two float4 per operand per k), the next slab prefetched into
// registers while the current one is consumed from a double-buffered shared-memory
// stage (one CTA barrier per slab).  B's slab is transposed on its way into shared
// memory ([k][n]).  Every output accumulates fmaf(a_k, b_k, acc) for k = 0, 1, ...
// from 0 exactly like gemm32_kernel, so the two are bitwise equal.
namespace gemm32 {
constexpr int BM = 128, BN = 128, BK = 8, THREADS = 256, PAD = 4;
}
template <int MODE, bool VEC>
__global__ void __launch_bounds__(gemm32::THREADS, 2)
    gemm32_big_kernel(int64_t m, int64_t n, int64_t k, float alpha, const float* __restrict__ A, int64_t lda,
                      const float* __restrict__ B, int64_t ldb, float beta, const float* C, int64_t ldc, float* out,
                      int64_t ldo, int tri) {
  using namespace gemm32;
  if (tri && (int64_t)(blockIdx.x + 1) * BM <= (int64_t)blockIdx.y * BN) return;
  __shared__ __align__(16) float As[2][BK][BM + PAD];
  __shared__ __align__(16) float Bs[2][BK][BN + PAD];
  const int t = threadIdx.x;
  const int tx = t & 15, ty = t >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  // loader roles: A: k row t/32, m = 4 (t%32) .. +3;  B: column n = t/2, k = 4 (t%2) .. +3
  const int la_k = t >> 5, la_m = (t & 31) * 4;
  const int lb_n = t >> 1, lb_k = (t & 1) * 4;
  float ra[4], rb[4];
  auto load = [&](int64_t k0) {
    const int64_t gk = k0 + la_k, gm = m0 + la_m;
    if (VEC && gk < k && gm + 3 < m) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(A + gk * lda + gm));
      ra[0] = v.x; ra[1] = v.y; ra[2] = v.z; ra[3] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) ra[e] = (gk < k && gm + e < m) ? A[gk * lda + gm + e] : 0.f;
    }
    const int64_t gn = n0 + lb_n, gk2 = k0 + lb_k;
    if (VEC && gn < n && gk2 + 3 < k) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(B + gn * ldb + gk2));
      rb[0] = v.x; rb[1] = v.y; rb[2] = v.z; rb[3] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) rb[e] = (gn < n && gk2 + e < k) ? B[gn * ldb + gk2 + e] : 0.f;
    }
  };
  auto store = [&](int buf) {
    *reinterpret_cast<float4*>(&As[buf][la_k][la_m]) = make_float4(ra[0], ra[1], ra[2], ra[3]);
#pragma unroll
    for (int e = 0; e < 4; ++e) Bs[buf][lb_k + e][lb_n] = rb[e];
  };
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  const int64_t ktiles = ceil_div(k, BK);
  if (ktiles > 0) {
    load(0);
    store(0);
  }
  __syncthreads();
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    const int buf = (int)(kt & 1);
    if (kt + 1 < ktiles) load((kt + 1) * BK);  // in flight during the FMAs below
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (kt + 1 < ktiles) store(buf ^ 1);  // the other buffer: its readers passed the last barrier
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (r >= m) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (c >= n) continue;
      float o;
      if (MODE == 1) {
        o = __fsub_rn(C[r + c * ldc], acc[i][j]);
      } else {
        const float cb = beta == 0.f ? 0.f : __fmul_rn(beta, C[r + c * ldc]);
        o = __fadd_rn(cb, __fmul_rn(alpha, acc[i][j]));
      }
      out[r + c * ldo] = o;
    }
  }
}

// FP32 GEMM (FFMA, fp32 accumulation like sgemm): 64x64 tile, 256 threads, 4x4 per thread.
template <int MODE>
__global__ void __launch_bounds__(256)
    gemm32_kernel(int64_t m, int64_t n, int64_t k, float alpha, const float* __restrict__ A,
                  int64_t lda, const float* __restrict__ B, int64_t ldb, float beta, const float* C,
                  int64_t ldc, float* out, int64_t ldo, int tri) {
  if (tri && (int64_t)(blockIdx.x + 1) * 64 <= (int64_t)blockIdx.y * 64) return;
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * 64, n0 = (int64_t)blockIdx.y * 64;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < k; k0 += 16) {
    for (int c = threadIdx.x; c < 16 * 64; c += 256) {
      const int kk = c / 64, mm = c % 64;
      const int64_t gr = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gr < m && gk < k) ? A[gr + gk * lda] : 0.f;
      const int nn = c / 16, kb = c % 16;
      const int64_t gc = n0 + nn, gk2 = k0 + kb;
      Bs[kb][nn] = (gc < n && gk2 < k) ? B[gk2 + gc * ldb] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tx + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][ty + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = m0 + tx + 16 * i, c = n0 + ty + 16 * j;
      if (r < m && c < n) {
        float o;
        if (MODE == 1)
          o = __fsub_rn(C[r + c * ldc], acc[i][j]);
        else {
          const float cb = beta == 0.f ? 0.f : __fmul_rn(beta, C[r + c * ldc]);
          o = __fadd_rn(cb, __fmul_rn(alpha, acc[i][j]));
        }
        out[r + c * ldo] = o;
      }
    }
}

static int gemm_impl(ds_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha,
                     const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                     const double* C, int64_t ldc, double* out, int64_t ldo, int tri) {
  using namespace gemm64;
  if (m == 0 || n == 0) return DS_OK;
  static bool attr_done = false;
  if (!attr_done) {
    DS_CUDA(cudaFuncSetAttribute(gemm64_kernel<true, 0>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    DS_CUDA(cudaFuncSetAttribute(gemm64_kernel<true, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    DS_CUDA(cudaFuncSetAttribute(gemm64_kernel<false, 0>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    DS_CUDA(cudaFuncSetAttribute(gemm64_kernel<false, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    attr_done = true;
  }
  dim3 grid((unsigned)ceil_div(m, BM), (unsigned)ceil_div(n, BN));
  const bool vec = (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(B) % 16 == 0) && (lda % 2 == 0) && (ldb % 2 == 0);
  const bool sub = (alpha == -1.0 && beta == 1.0);
  if (vec && k > 0 && gemm_tma_enabled() && m < (1ll << 31) && n < (1ll << 31) && k < (1ll << 31)) {
    CUtensorMap ta, tb;
    if (encode_colmajor_map(&ta, A, m, k, lda, 16, BK) && encode_colmajor_map(&tb, B, k, n, ldb, BK, BN)) {
      static bool tma_attr = false;
      if (!tma_attr) {
        DS_CUDA(cudaFuncSetAttribute(gemm64_tma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)SMEM_TMA));
        DS_CUDA(cudaFuncSetAttribute(gemm64_tma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)SMEM_TMA));
        tma_attr = true;
      }
      if (sub && !tri && ctx->gemm_reserve > 0 && ctx->gemm_ctr) {  // LU trailing update beside the look-ahead panel
        static bool pattr = false;
        if (!pattr) {
          DS_CUDA(cudaFuncSetAttribute(gemm64_tma_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMEM_TMA));
          pattr = true;
        }
        DS_CUDA(cudaMemsetAsync(ctx->gemm_ctr, 0, 2 * sizeof(unsigned), ctx->stream));
        gemm64_tma_persist_kernel<<<2 * ctx->num_sms, THREADS, SMEM_TMA, ctx->stream>>>(
            ta, tb, m, n, k, C, ldc, out, ldo, ctx->gemm_reserve, ctx->gemm_ctr);
      } else if (sub)
        gemm64_tma_kernel<1><<<grid, THREADS, SMEM_TMA, ctx->stream>>>(ta, tb, m, n, k, alpha, beta, C, ldc, out,
                                                                       ldo, tri);
      else
        gemm64_tma_kernel<0><<<grid, THREADS, SMEM_TMA, ctx->stream>>>(ta, tb, m, n, k, alpha, beta, C, ldc, out,
                                                                       ldo, tri);
      count_launch(ctx);
      DS_CHECK_LAUNCH();
      return DS_OK;
    }
  }
  if (k == 0) {
    // out = beta*C (alpha*0 added)
    if (vec && sub)
      gemm64_kernel<true, 1><<<grid, THREADS, SMEM, ctx->stream>>>(m, n, k, alpha, A, lda, B, ldb,
                                                                    beta, C, ldc, out, ldo, tri);
    else
      gemm64_kernel<false, 0><<<grid, THREADS, SMEM, ctx->stream>>>(m, n, k, alpha, A, lda, B,
                                                                     ldb, beta, C, ldc, out, ldo, tri);
  } else if (vec) {
    if (sub)
      gemm64_kernel<true, 1><<<grid, THREADS, SMEM, ctx->stream>>>(m, n, k, alpha, A, lda, B, ldb,
                                                                    beta, C, ldc, out, ldo, tri);
    else
      gemm64_kernel<true, 0><<<grid, THREADS, SMEM, ctx->stream>>>(m, n, k, alpha, A, lda, B, ldb,
                                                                    beta, C, ldc, out, ldo, tri);
  } else {
    if (sub)
      gemm64_kernel<false, 1><<<grid, THREADS, SMEM, ctx->stream>>>(m, n, k, alpha, A, lda, B,
                                                                     ldb, beta, C, ldc, out, ldo, tri);
    else
      gemm64_kernel<false, 0><<<grid, THREADS, SMEM, ctx->stream>>>(m, n, k, alpha, A, lda, B,
                                                                     ldb, beta, C, ldc, out, ldo, tri);
  }
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

static int gemm_impl(ds_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A,
                     int64_t lda, const float* B, int64_t ldb, double beta, const float* C,
                     int64_t ldc, float* out, int64_t ldo, int tri) {
  if (m == 0 || n == 0) return DS_OK;
  const bool sub = alpha == -1.0 && beta == 1.0;
  static const bool small_only = [] {
    const char* e = getenv("DENSOLVE_GEMM32_SMALL");  // A/B switch: the 64 x 64 kernel everywhere
    return e && e[0] == '1';
  }();
  if (!small_only && m >= 128 && n >= 128 && k >= 128) {  // K = 64 panels: more CTAs win (21.7 vs 12.4 TF)
    using namespace gemm32;
    dim3 grid((unsigned)ceil_div(m, BM), (unsigned)ceil_div(n, BN));
    const bool vec = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0) &&
                     (lda % 4 == 0) && (ldb % 4 == 0);
    const float fa = (float)alpha, fb = (float)beta;
    if (sub && vec)
      gemm32_big_kernel<1, true><<<grid, THREADS, 0, ctx->stream>>>(m, n, k, fa, A, lda, B, ldb, fb, C, ldc, out, ldo, tri);
    else if (sub)
      gemm32_big_kernel<1, false><<<grid, THREADS, 0, ctx->stream>>>(m, n, k, fa, A, lda, B, ldb, fb, C, ldc, out, ldo, tri);
    else if (vec)
      gemm32_big_kernel<0, true><<<grid, THREADS, 0, ctx->stream>>>(m, n, k, fa, A, lda, B, ldb, fb, C, ldc, out, ldo, tri);
    else
      gemm32_big_kernel<0, false><<<grid, THREADS, 0, ctx->stream>>>(m, n, k, fa, A, lda, B, ldb, fb, C, ldc, out, ldo, tri);
    count_launch(ctx);
    DS_CHECK_LAUNCH();
    return DS_OK;
  }
  dim3 grid((unsigned)ceil_div(m, 64), (unsigned)ceil_div(n, 64));
  if (sub)
    gemm32_kernel<1><<<grid, 256, 0, ctx->stream>>>(m, n, k, (float)alpha, A, lda, B, ldb,
                                                    (float)beta, C, ldc, out, ldo, tri);
  else
    gemm32_kernel<0><<<grid, 256, 0, ctx->stream>>>(m, n, k, (float)alpha, A, lda, B, ldb,
                                                    (float)beta, C, ldc, out, ldo, tri);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

template <>
int gemm_launch<double>(ds_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha,
                        const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                        const double* C, int64_t ldc, double* out, int64_t ldo) {
  return gemm_impl(ctx, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, out, ldo, 0);
}
template <>
int gemm_launch<float>(ds_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const float* A,
                       int64_t lda, const float* B, int64_t ldb, double beta, const float* C,
                       int64_t ldc, float* out, int64_t ldo) {
  return gemm_impl(ctx, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, out, ldo, 0);
}
template <typename T>
int gemm_sub_lower_launch(ds_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, int64_t lda,
                          const T* B, int64_t ldb, T* C, int64_t ldc) {
  return gemm_impl(ctx, m, n, k, -1.0, A, lda, B, ldb, 1.0, C, ldc, C, ldc, 1);
}
template int gemm_sub_lower_launch<double>(ds_ctx*, int64_t, int64_t, int64_t, const double*, int64_t,
                                           const double*, int64_t, double*, int64_t);
template int gemm_sub_lower_launch<float>(ds_ctx*, int64_t, int64_t, int64_t, const float*, int64_t,
                                          const float*, int64_t, float*, int64_t);

// ============================================================================
// TRSM (backends.py:176-200).
//   lower-unit: z_i = b_i - (L[i,:i] . z[:i])           (stored diagonal ignored)
//   upper:      z_i = (b_i - U[i,i+1:] . z[i+1:]) / U_ii
// b <= 64: shared-memory tile kernel; b > 64: generic path, one thread per column.
// ============================================================================
// Tile form for b <= 64 (the LU U-block-row solve): one CTA per 64 x 32 tile of
// the right-hand side, L and the tile staged in shared memory, right-looking
// column sweep (z_i -= L_ij z_j for all i > j and all 32 columns per step, one
// fused multiply-add each), so the dependent chain is spread over 256 threads.
template <typename T>
__global__ void __launch_bounds__(256)
    trsm_lower_unit_tile(int b, int64_t m, const T* __restrict__ L, int64_t ldl,
                         const T* __restrict__ B, int64_t ldb, T* Z, int64_t ldz) {
  __shared__ T Ls[63][64];  // Ls[j][i] = L[i, j] (column j contiguous; column b-1 unused)
  __shared__ T Zs[32][65];  // Zs[c][i]
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * 32;
  const int nc = (int)min((int64_t)32, m - c0);
  for (int idx = tid; idx < b * (b - 1); idx += blockDim.x) {
    const int i = idx % b, j = idx / b;
    Ls[j][i] = L[i + (int64_t)j * ldl];
  }
  for (int idx = tid; idx < b * nc; idx += blockDim.x) {
    const int i = idx % b, c = idx / b;
    Zs[c][i] = B[i + (c0 + c) * ldb];
  }
  __syncthreads();
  const int c = tid & 31, rg = tid >> 5;
  for (int j = 0; j + 1 < b; ++j) {
    const T zj = Zs[c][j];
    for (int i = j + 1 + rg; i < b; i += 8) Zs[c][i] = fma(-Ls[j][i], zj, Zs[c][i]);
    __syncthreads();
  }
  for (int idx = tid; idx < b * nc; idx += blockDim.x) {
    const int i = idx % b, cc = idx / b;
    Z[i + (c0 + cc) * ldz] = Zs[cc][i];
  }
}

// b == 64 (every full LU panel): 8 threads per right-hand-side column, thread
// `sub` owning rows sub, sub + 8, ..., sub + 56 in registers.  Step j broadcasts
// z_j from its owner with one shuffle inside the 8-lane group and every thread
// updates its rows i > j with L[i, j] from shared memory (the 8 lanes of a group
// read 8 consecutive elements; the 4 groups of a warp read the same ones).  The
// dependent chain is 63 x (shuffle + FMA) and each thread issues 504 FMAs, so a
// launch of any width costs ~1-2 us (was one thread per column: 2016 dependent
// FMAs, ~20 us per launch).
template <typename T>
__global__ void __launch_bounds__(256)
    trsm_lower_unit_cols64(int64_t m, const T* __restrict__ L, int64_t ldl, const T* B, int64_t ldb,
                           T* Z, int64_t ldz) {
  __shared__ __align__(16) T Ls[64][64];  // Ls[j][i] = L[i, j] (i > j), column j contiguous
  const int tid = threadIdx.x, lane = tid & 31, sub = lane & 7;
  const int gbase = lane & ~7;
  {
    T v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = tid + u * 256, i = e & 63, j = e >> 6;
      v[u] = i > j ? L[i + (int64_t)j * ldl] : T(0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = tid + u * 256;
      Ls[e >> 6][e & 63] = v[u];
    }
  }
  __syncthreads();
  const int64_t col = (int64_t)blockIdx.x * 32 + (tid >> 3);
  const bool act = col < m;
  T z[8];
  const T* bb = B + (act ? col : 0) * ldb;
#pragma unroll
  for (int k = 0; k < 8; ++k) z[k] = act ? bb[sub + 8 * k] : T(0);
#pragma unroll
  for (int j = 0; j < 63; ++j) {
    const T zj = __shfl_sync(0xffffffffu, z[j >> 3], gbase + (j & 7));
#pragma unroll
    for (int k = j >> 3; k < 8; ++k) {
      const int i = sub + 8 * k;
      if (i > j) z[k] = fma(-Ls[j][i], zj, z[k]);
    }
  }
  if (act) {
    T* zz = Z + col * ldz;
#pragma unroll
    for (int k = 0; k < 8; ++k) zz[sub + 8 * k] = z[k];
  }
}

template <typename T>
__global__ void trsm_lower_unit_big(int64_t b, int64_t m, const T* __restrict__ L, int64_t ldl,
                                    const T* B, int64_t ldb, T* Z, int64_t ldz) {
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= m) return;
  T* z = Z + col * ldz;
  const T* bb = B + col * ldb;
  if (z != bb)
    for (int64_t i = 0; i < b; ++i) z[i] = bb[i];
  for (int64_t i = 1; i < b; ++i) {
    T acc = T(0);
    for (int64_t j = 0; j < i; ++j) acc = fma(L[i + j * ldl], z[j], acc);
    z[i] = sub_rn(z[i], acc);
  }
}

template <typename T>
__global__ void trsm_upper_kernel(int64_t b, int64_t m, const T* __restrict__ U, int64_t ldu,
                                  const T* B, int64_t ldb, T* Z, int64_t ldz) {
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= m) return;
  T* z = Z + col * ldz;
  const T* bb = B + col * ldb;
  if (z != bb)
    for (int64_t i = 0; i < b; ++i) z[i] = bb[i];
  for (int64_t i = b - 1; i >= 0; --i) {
    T acc = T(0);
    for (int64_t j = i + 1; j < b; ++j) acc = fma(U[i + j * ldu], z[j], acc);
    T v = i + 1 < b ? sub_rn(z[i], acc) : z[i];
    z[i] = div_rn(v, U[i + i * ldu]);
  }
}

template <typename T>
int trsm_lower_unit_launch(ds_ctx* ctx, int64_t b, int64_t m, const T* L, int64_t ldl, const T* B,
                           int64_t ldb, T* Z, int64_t ldz) {
  if (b == 0 || m == 0) return DS_OK;
  if (b == 64) {
    trsm_lower_unit_cols64<T><<<(unsigned)ceil_div(m, 32), 256, 0, ctx->stream>>>(m, L, ldl, B, ldb, Z, ldz);
  } else if (b < 64) {
    trsm_lower_unit_tile<T><<<(unsigned)ceil_div(m, 32), 256, 0, ctx->stream>>>(
        (int)b, m, L, ldl, B, ldb, Z, ldz);
  } else {
    trsm_lower_unit_big<T><<<(unsigned)ceil_div(m, 128), 128, 0, ctx->stream>>>(b, m, L, ldl, B,
                                                                               ldb, Z, ldz);
  }
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
// U01 of an outer panel, one CTA per 32 columns (the thread <-> column mapping of
// trsm_lower_unit_cols64: 8 threads per column, 8 rows each).  Per 64-row block ib:
//   (a) z = L_ib^-1 (rows of the block): the same shuffle substitution, same order;
//   (b) rows below the block inside the outer panel -= L[below, ib] z: per element the
//       accumulator starts from the stored value and takes the 16 k-steps of 4 of
//       mma.m8n8k4 with the negated L operand, in k order: the K = 64 chain of
//       gemm64(_tma)_kernel<1>, hence bitwise its result.
// Shared memory: the block's strict lower triangle (column-major) and the solved z strip.
__global__ void __launch_bounds__(256, 1)
    u01_fused_kernel(double* __restrict__ W, int64_t ld, int64_t kb, int nblk, int64_t c0, int64_t c1) {
  extern __shared__ __align__(16) double u01_smem[];
  double (*Ls)[64] = reinterpret_cast<double (*)[64]>(u01_smem);           // Ls[j][i] = L[i, j], i > j
  double (*Zs)[33] = reinterpret_cast<double (*)[33]>(u01_smem + 64 * 64);  // Zs[k][col]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, sub = lane & 7, gbase = lane & ~7;
  const int g = lane >> 2, t = lane & 3;
  const int64_t cs = c0 + (int64_t)blockIdx.x * 32;  // first column of the strip
  const int cl = tid >> 3;                            // trsm: my column in the strip
  const bool act = cs + cl < c1;
  const int64_t rend = kb + (int64_t)nblk * 64;
  for (int ib = 0; ib < nblk; ++ib) {
    const int64_t r0 = kb + (int64_t)ib * 64;
    __syncthreads();  // the previous block's update is done with Zs / Ls
    {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = tid + u * 256, i = e & 63, j = e >> 6;
        v[u] = i > j ? W[(r0 + i) + (r0 + j) * ld] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = tid + u * 256;
        Ls[e >> 6][e & 63] = v[u];
      }
    }
    __syncthreads();
    double z[8];
    double* bb = W + (act ? cs + cl : c0) * ld + r0;
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = act ? bb[sub + 8 * k] : 0.0;
#pragma unroll
    for (int j = 0; j < 63; ++j) {
      const double zj = __shfl_sync(0xffffffffu, z[j >> 3], gbase + (j & 7));
#pragma unroll
      for (int k = j >> 3; k < 8; ++k) {
        const int i = sub + 8 * k;
        if (i > j) z[k] = fma(-Ls[j][i], zj, z[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      Zs[sub + 8 * k][cl] = act ? z[k] : 0.0;
      if (act) bb[sub + 8 * k] = z[k];
    }
    __syncthreads();
    // (b) rows [r0 + 64, rend) x the strip, 32-row tiles over the 8 warps
    const int64_t rb = r0 + 64;
    const int ntile = (int)((rend - rb) / 32);
    for (int tl = warp; tl < ntile; tl += 8) {
      const int64_t m0 = rb + (int64_t)tl * 32;
      double acc[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t c = cs + j * 8 + 2 * t + e;
            acc[i][j][e] = c < c1 ? W[(m0 + i * 8 + g) + c * ld] : 0.0;
          }
#pragma unroll 4
      for (int q = 0; q < 16; ++q) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = -W[(m0 + i * 8 + g) + (r0 + 4 * q + t) * ld];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Zs[4 * q + t][j * 8 + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t c = cs + j * 8 + 2 * t + e;
            if (c < c1) W[(m0 + i * 8 + g) + c * ld] = acc[i][j][e];
          }
    }
  }
}

int u01_fused_launch(ds_ctx* ctx, double* W, int64_t ld, int64_t kb, int nblk, int64_t c0, int64_t c1) {
  if (c1 <= c0 || nblk <= 0) return DS_OK;
  constexpr int smem = (64 * 64 + 64 * 33) * (int)sizeof(double);
  static bool attr = false;
  if (!attr) {
    DS_CUDA(cudaFuncSetAttribute(u01_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  u01_fused_kernel<<<(unsigned)ceil_div(c1 - c0, (int64_t)32), 256, smem, ctx->stream>>>(W, ld, kb, nblk, c0, c1);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

template <typename T>
int trsm_upper_launch(ds_ctx* ctx, int64_t b, int64_t m, const T* U, int64_t ldu, const T* B,
                      int64_t ldb, T* Z, int64_t ldz) {
  if (b == 0 || m == 0) return DS_OK;
  trsm_upper_kernel<T><<<(unsigned)ceil_div(m, 128), 128, 0, ctx->stream>>>(b, m, U, ldu, B, ldb,
                                                                           Z, ldz);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
template int trsm_lower_unit_launch<double>(ds_ctx*, int64_t, int64_t, const double*, int64_t,
                                            const double*, int64_t, double*, int64_t);
template int trsm_lower_unit_launch<float>(ds_ctx*, int64_t, int64_t, const float*, int64_t,
                                           const float*, int64_t, float*, int64_t);
template int trsm_upper_launch<double>(ds_ctx*, int64_t, int64_t, const double*, int64_t,
                                       const double*, int64_t, double*, int64_t);
template int trsm_upper_launch<float>(ds_ctx*, int64_t, int64_t, const float*, int64_t,
                                      const float*, int64_t, float*, int64_t);

// Load (lazy module loading) every kernel the row-sharded solver launches from this
// file, before any shard starts spinning on an exchange: a first launch that loads its
// module waits for the device, i.e. for the peers' exchange kernels on a shared GPU.
int preload_dense_kernels_blas() {  // TRSM and GEMM of the block-cyclic LU shards
  cudaFuncAttributes a;
  const void* fns[] = {(const void*)trsm_lower_unit_cols64<double>, (const void*)trsm_lower_unit_cols64<float>,
                       (const void*)trsm_lower_unit_tile<double>,   (const void*)trsm_lower_unit_tile<float>,
                       (const void*)trsm_lower_unit_big<double>,    (const void*)trsm_lower_unit_big<float>,
                       (const void*)gemm64_tma_kernel<0>,           (const void*)gemm64_tma_kernel<1>,
                       (const void*)gemm64_kernel<true, 0>,         (const void*)gemm64_kernel<true, 1>,
                       (const void*)gemm64_kernel<false, 0>,        (const void*)gemm64_kernel<false, 1>,
                       (const void*)gemm32_kernel<0>,               (const void*)gemm32_kernel<1>,
                       (const void*)gemm32_big_kernel<0, true>,     (const void*)gemm32_big_kernel<1, true>,
                       (const void*)gemm32_big_kernel<0, false>,    (const void*)gemm32_big_kernel<1, false>};
  for (const void* f : fns) DS_CUDA(cudaFuncGetAttributes(&a, f));
  return DS_OK;
}
int preload_sharded_kernels_blas() {
  cudaFuncAttributes a;
  const void* fns[] = {
      (const void*)ds_colstream_mv_kernel<double, 2, 8>, (const void*)ds_colstream_mv_kernel<double, 1, 8>,
      (const void*)ds_colstream_mv_kernel<float, 4, 8>,  (const void*)ds_colstream_mv_kernel<float, 1, 8>,
      (const void*)ds_colstream_reduce_kernel<double, EPI_DOT>, (const void*)ds_colstream_reduce_kernel<float, EPI_DOT>,
      (const void*)ds_colstream_reduce_kernel<double, EPI_RESID>,
      (const void*)ds_colstream_reduce_kernel<float, EPI_RESID>,
      (const void*)symcheck_kernel<double>, (const void*)symcheck_kernel<float>, (const void*)finish_max2_kernel,
      // the row-sharded GMRES: r = b - A x, x += V y
      (const void*)ds_colstream_reduce_kernel<double, EPI_STORE>, (const void*)ds_colstream_reduce_kernel<float, EPI_STORE>,
      (const void*)ds_colstream_reduce_kernel<double, EPI_AXPY_INTO>,
      (const void*)ds_colstream_reduce_kernel<float, EPI_AXPY_INTO>, (const void*)axpy_kernel<double>,
      (const void*)axpy_kernel<float>};
  for (const void* f : fns) DS_CUDA(cudaFuncGetAttributes(&a, f));
  return DS_OK;
}

}  // namespace ds

// ============================================================================
// extern "C" op contract
// ============================================================================
using namespace ds;

namespace {
struct Scratch {
  double* red = nullptr;  // reduction partials
  double* out = nullptr;  // 8 doubles of results
  int64_t* iout = nullptr;
};
int get_scratch(ds_ctx* ctx, size_t red_doubles, Scratch* s) {
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, (red_doubles + 16) * sizeof(double) * 2, &ws));
  s->out = reinterpret_cast<double*>(ws);
  s->iout = reinterpret_cast<int64_t*>(s->out + 8);
  s->red = s->out + 16;
  return DS_OK;
}
int fetch(ds_ctx* ctx, void* host, const void* dev, size_t bytes) {
  DS_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}
}  // namespace

extern "C" {

int ds_axpy(ds_ctx* ctx, int dtype, int64_t n, double alpha, const void* x, const void* y,
            void* out) {
  DS_ENTER(ctx);
  DS_DISPATCH(dtype, T, DS_TRY(axpy_launch<T>(ctx, n, alpha, (const T*)x, (const T*)y, (T*)out)));
  return DS_OK;
}

int ds_scal(ds_ctx* ctx, int dtype, int64_t n, double alpha, const void* x, void* out) {
  DS_ENTER(ctx);
  DS_DISPATCH(dtype, T, DS_TRY(scal_launch<T>(ctx, n, alpha, (const T*)x, (T*)out)));
  return DS_OK;
}

int ds_dot(ds_ctx* ctx, int dtype, int64_t n, const void* x, const void* y, double* result) {
  DS_ENTER(ctx);
  Scratch s;
  DS_TRY(get_scratch(ctx, (size_t)ctx->num_sms * 4, &s));
  int nblk = 0;
  DS_DISPATCH(dtype, T, DS_TRY(dot_launch<T>(ctx, n, (const T*)x, (const T*)y, s.red, &nblk)));
  DS_TRY(finish_sum(ctx, s.red, nblk, s.out));
  return fetch(ctx, result, s.out, sizeof(double));
}

int ds_nrm2(ds_ctx* ctx, int dtype, int64_t n, const void* x, double* result) {
  DS_ENTER(ctx);
  if (n == 0) {
    *result = 0.0;
    return DS_OK;
  }
  Scratch s;
  DS_TRY(get_scratch(ctx, (size_t)ctx->num_sms * 8, &s));
  int nblk = 0;
  DS_DISPATCH(dtype, T, DS_TRY(ssq_launch<T>(ctx, n, (const T*)x, s.red, &nblk)));
  DS_TRY(finish_ssq(ctx, s.red, nblk, s.out));
  return fetch(ctx, result, s.out, sizeof(double));
}

int ds_iamax(ds_ctx* ctx, int dtype, int64_t n, const void* x, int64_t* result) {
  DS_ENTER(ctx);
  if (n <= 0) {
    set_error("iamax of empty vector");
    return DS_EDIM;
  }
  Scratch s;
  DS_TRY(get_scratch(ctx, (size_t)ctx->num_sms * 8, &s));
  const int g = reduce_grid(ctx, n);
  int64_t* ri = reinterpret_cast<int64_t*>(s.red + g);
  DS_DISPATCH(dtype, T,
              iamax_kernel<T><<<g, kRedThreads, 0, ctx->stream>>>(n, (const T*)x, s.red, ri));
  iamax_finish_kernel<<<1, 32, 0, ctx->stream>>>(s.red, ri, g, s.iout);
  count_launch(ctx, 2);
  DS_CHECK_LAUNCH();
  return fetch(ctx, result, s.iout, sizeof(int64_t));
}

int ds_gemv(ds_ctx* ctx, int dtype, int64_t m, int64_t n, const void* A, int64_t lda,
            const void* x, void* y) {
  DS_ENTER(ctx);
  if (m == 0) return DS_OK;
  const GemvPlan p = gemv_plan(ctx, m, n, dtype_size(dtype));
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, p.part_bytes + 4096, &ws));
  DS_DISPATCH(dtype, T,
              DS_TRY(gemv_launch<T>(ctx, p, (const T*)A, lda, (const T*)x, (T*)y, (double*)ws,
                                    EPI_STORE, nullptr, nullptr, nullptr)));
  return DS_OK;
}

int ds_ger(ds_ctx* ctx, int dtype, int64_t m, int64_t n, const void* A, int64_t lda, double alpha,
           const void* x, const void* y, void* out, int64_t ldo) {
  DS_ENTER(ctx);
  DS_DISPATCH(dtype, T,
              DS_TRY(ger_launch<T>(ctx, m, n, (const T*)A, lda, alpha, (const T*)x, (const T*)y,
                                   (T*)out, ldo)));
  return DS_OK;
}

int ds_gemm(ds_ctx* ctx, int dtype, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
            int64_t lda, const void* B, int64_t ldb, double beta, const void* C, int64_t ldc,
            void* out, int64_t ldo) {
  DS_ENTER(ctx);
  DS_DISPATCH(dtype, T,
              DS_TRY(gemm_launch<T>(ctx, m, n, k, alpha, (const T*)A, lda, (const T*)B, ldb, beta,
                                    (const T*)C, ldc, (T*)out, ldo)));
  return DS_OK;
}

int ds_trsm_lower_unit(ds_ctx* ctx, int dtype, int64_t b, int64_t m, const void* L, int64_t ldl,
                       const void* B, int64_t ldb, void* Z, int64_t ldz) {
  DS_ENTER(ctx);
  DS_DISPATCH(dtype, T,
              DS_TRY(trsm_lower_unit_launch<T>(ctx, b, m, (const T*)L, ldl, (const T*)B, ldb,
                                               (T*)Z, ldz)));
  return DS_OK;
}

int ds_trsm_upper(ds_ctx* ctx, int dtype, int64_t b, int64_t m, const void* U, int64_t ldu,
                  const void* B, int64_t ldb, void* Z, int64_t ldz) {
  DS_ENTER(ctx);
  DS_DISPATCH(dtype, T,
              DS_TRY(trsm_upper_launch<T>(ctx, b, m, (const T*)U, ldu, (const T*)B, ldb, (T*)Z,
                                          ldz)));
  return DS_OK;
}

int ds_symmetry_check(ds_ctx* ctx, int dtype, int64_t n, const void* A, int64_t lda,
                      double* maxdiff, double* amax) {
  DS_ENTER(ctx);
  if (n == 0) {
    *maxdiff = 0.0;
    *amax = 0.0;
    return DS_OK;
  }
  Scratch s;
  DS_TRY(get_scratch(ctx, (size_t)ctx->num_sms * 16 + 64, &s));
  int nblk = 0;
  DS_DISPATCH(dtype, T, DS_TRY(symcheck_launch<T>(ctx, n, (const T*)A, lda, s.red, &nblk)));
  finish_max2_kernel<<<1, 256, 0, ctx->stream>>>(s.red, nblk, s.out);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  double h[2];
  DS_TRY(fetch(ctx, h, s.out, 2 * sizeof(double)));
  *maxdiff = h[0];
  *amax = h[1];
  return DS_OK;
}

int ds_relative_residual(ds_ctx* ctx, int dtype, int64_t n, const void* A, int64_t lda,
                         const void* x, const void* b, double* result) {
  DS_ENTER(ctx);
  const GemvPlan p = gemv_plan(ctx, n, n, dtype_size(dtype));
  const int rblocks = (int)ceil_div(std::max<int64_t>(n, 1), 256);
  const size_t es = dtype_size(dtype);
  void* ws = nullptr;
  const size_t red_off = (p.part_bytes + 255) / 256 * 256;
  const size_t r_off = red_off + ((size_t)rblocks * 3 + 64) * sizeof(double);
  const size_t o_off = (r_off + (size_t)n * es + 255) / 256 * 256;
  DS_TRY(ctx_workspace(ctx, o_off + 256 + 4 * sizeof(double) * rblocks, &ws));
  char* base = (char*)ws;
  double* part = (double*)base;
  double* red = (double*)(base + red_off);
  void* r = base + r_off;
  double* out = (double*)(base + o_off);
  int nb = 0;
  DS_DISPATCH(dtype, T,
              DS_TRY(gemv_launch<T>(ctx, p, (const T*)A, lda, (const T*)x, (T*)r, part, EPI_RESID,
                                    (const T*)b, red, &nb)));
  // ||b - Ax|| with the plain 2-norm (np.linalg.norm, core.py:207-210): sum red[2nb..3nb)
  DS_TRY(finish_sum(ctx, red + 2 * nb, nb, out));
  int nb2 = 0;
  double* red2 = red + 3 * nb + 8;
  DS_DISPATCH(dtype, T, DS_TRY(dot_launch<T>(ctx, n, (const T*)b, (const T*)b, red2, &nb2)));
  DS_TRY(finish_sum(ctx, red2, nb2, out + 1));
  double h[2];
  DS_TRY(fetch(ctx, h, out, 2 * sizeof(double)));
  const double bnorm = sqrt(h[1]);
  if (bnorm == 0.0) {
    set_error("||b|| = 0: relative residual undefined (x = 0 is exact)");
    return DS_EDEGRHS;
  }
  *result = sqrt(h[0]) / bnorm;
  return DS_OK;
}

}  // extern "C"
