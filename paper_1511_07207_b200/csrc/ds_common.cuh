// ds_common.cuh — shared device/host helpers for the densolve B200 library.
//
// Numerics notes (why the elementwise helpers below exist):
//   The reference evaluates every vector update with NumPy, i.e. each binary
//   operation rounds separately and nothing is contracted into an FMA
//   (backends.py:107 `y + alpha * x`, :126 `alpha * x`, :152-155
//   `out += alpha * np.outer(x, y)`).  The device kernels use the explicit
//   round-to-nearest intrinsics below for those updates so that, given the same
//   inputs, each element is bitwise identical to the reference's.  Only
//   reductions (dot/nrm2/gemv/gemm sums) differ, by summation order.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cmath>
#include <cstdarg>
#include <mutex>
#include <string>

#include "../../include/densolve_b200.h"

namespace ds {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// host-side error plumbing
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);

struct Status {
  int code = DS_OK;
};

#define DS_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::ds::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__,    \
                      __LINE__, cudaGetErrorString(_e));                               \
      return _e == cudaErrorMemoryAllocation ? DS_ENOMEM : DS_ECUDA;                   \
    }                                                                                  \
  } while (0)

#define DS_TRY(expr)              \
  do {                            \
    int _s = (expr);              \
    if (_s != DS_OK) return _s;   \
  } while (0)

#define DS_CHECK_LAUNCH() DS_CUDA(cudaGetLastError())

// ---------------------------------------------------------------------------
// exact NumPy-style elementwise arithmetic (one rounding per binary op)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }

// Accumulator type of reductions: fp64 for both dtypes (deterministic, and at
// least as accurate as the reference's BLAS sdot/ddot).
template <typename T>
struct Acc {
  using type = double;
};

// ---------------------------------------------------------------------------
// warp / block reductions (deterministic: fixed shuffle tree, fixed smem order)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// NaN-propagating max of absolute values (np.max propagates NaN, backends.py:118).
__device__ __forceinline__ double nanmax(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a > b ? a : b;
}
__device__ __forceinline__ double warp_nanmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; result valid in every thread.  smem must hold >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? smem[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) smem[0] = t;
  }
  __syncthreads();
  t = smem[0];
  return t;
}
__device__ __forceinline__ double block_nanmax(double v, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_nanmax(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? smem[lane] : 0.0;
    t = warp_nanmax(t);
    if (lane == 0) smem[0] = t;
  }
  __syncthreads();
  t = smem[0];
  return t;
}

// ---------------------------------------------------------------------------
// overflow-safe sum of squares: (scale, ssq) pairs with value = scale^2 * ssq.
// Restates the intent of Backend.nrm2 (backends.py:114-122: m*sqrt(dot(x/m,x/m)))
// in a single pass: partial pairs are combined to the global max scale m.
// ---------------------------------------------------------------------------
// max propagating NaN (np.max semantics)
__device__ __forceinline__ double nan_max(double a, double b) {
  return (a != a) ? a : (b != b) ? b : fmax(a, b);
}
struct Ssq {
  double scale;  // max |x| seen (NaN-propagating)
  double ssq;    // sum (x/scale)^2
};
__device__ __forceinline__ Ssq ssq_add(Ssq a, double x) {
  double ax = fabs(x);
  if (ax != ax || a.scale != a.scale) return Ssq{ax != ax ? ax : a.scale, 1.0};
  if (ax == 0.0) return a;
  if (isinf(ax) || isinf(a.scale)) return Ssq{INFINITY, 1.0};
  if (ax > a.scale) {
    double r = a.scale / ax;
    return Ssq{ax, 1.0 + a.ssq * r * r};
  }
  double r = ax / a.scale;
  return Ssq{a.scale, a.ssq + r * r};
}
__device__ __forceinline__ Ssq ssq_merge(Ssq a, Ssq b) {
  if (a.scale != a.scale) return a;
  if (b.scale != b.scale) return b;
  if (isinf(a.scale) || isinf(b.scale)) return Ssq{INFINITY, 1.0};
  if (b.scale == 0.0) return a;
  if (a.scale == 0.0) return b;
  if (a.scale >= b.scale) {
    double r = b.scale / a.scale;
    return Ssq{a.scale, a.ssq + b.ssq * r * r};
  }
  double r = a.scale / b.scale;
  return Ssq{b.scale, b.ssq + a.ssq * r * r};
}
// value of the norm, with the reference's special cases: m == 0 or non-finite -> m.
__device__ __host__ __forceinline__ double ssq_norm(double scale, double ssq) {
  if (scale == 0.0 || !(scale - scale == 0.0)) return scale;  // 0, inf or nan
  return scale * sqrt(ssq);
}
__device__ __forceinline__ Ssq warp_ssq(Ssq v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Ssq w{__shfl_xor_sync(0xffffffffu, v.scale, o), __shfl_xor_sync(0xffffffffu, v.ssq, o)};
    // combine in a lane-order-independent but deterministic way: the xor tree
    // applies the same sequence of merges in every run.
    v = (threadIdx.x & o) ? ssq_merge(w, v) : ssq_merge(v, w);
  }
  return v;
}
__device__ __forceinline__ Ssq block_ssq(Ssq v, double* smem /* >= 64 doubles */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_ssq(v);
  __syncthreads();
  if (lane == 0) {
    smem[2 * wid] = v.scale;
    smem[2 * wid + 1] = v.ssq;
  }
  __syncthreads();
  if (wid == 0) {
    Ssq t = lane < nw ? Ssq{smem[2 * lane], smem[2 * lane + 1]} : Ssq{0.0, 0.0};
    t = warp_ssq(t);
    if (lane == 0) {
      smem[0] = t.scale;
      smem[1] = t.ssq;
    }
  }
  __syncthreads();
  Ssq r{smem[0], smem[1]};
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// software grid barrier for cooperative launches (all CTAs co-resident)
// ---------------------------------------------------------------------------
// Monotonic grid barrier: the counter is zeroed before the launch; barrier #e
// completes when the counter reaches e * nblocks.  Thread 0 of each CTA releases
// the CTA's prior writes (fence + relaxed add) and acquires everyone else's.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_sync(unsigned* counter, unsigned nblocks, unsigned& epoch) {
  __syncthreads();
  epoch += 1;
  if (threadIdx.x == 0) {
    const unsigned target = epoch * nblocks;
    __threadfence();
    atomicAdd(counter, 1u);
    while (ld_acquire_u32(counter) < target) {
    }
  }
  __syncthreads();
}

inline __host__ __device__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// workspace carving helper (256-byte aligned sub-buffers of one allocation)
struct Carver {
  char* base;
  size_t off = 0;
  template <typename P>
  P* take(size_t bytes) {
    off = (off + 255) / 256 * 256;
    P* p = reinterpret_cast<P*>(base + off);
    off += bytes;
    return p;
  }
};

inline size_t dtype_size(int dtype) { return dtype == DS_F64 ? 8 : 4; }

}  // namespace ds

// ---------------------------------------------------------------------------
// context (defined in ds_context.cu)
// ---------------------------------------------------------------------------
struct ds_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  size_t smem_optin = 0;
  // grow-only scratch buffers (device), reused across calls on this context
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // small pinned host staging buffer
  void* hbuf = nullptr;
  size_t hbuf_bytes = 0;
  int64_t launches = 0;
  // LU look-ahead: a high-priority side stream for the next panel's factorization
  cudaStream_t side = nullptr;
  cudaStream_t aux = nullptr;  // low-priority stream for the swaps of already-factored L columns
  cudaStream_t copy = nullptr;  // asynchronous host->device staging (ds_upload_async)
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_c = nullptr;
  // LU trailing GEMM beside the look-ahead panel: > 0 runs the fp64 C - AB update as the
  // persistent kernel that leaves SMs [0, gemm_reserve) to the side stream (ds_lu.cu)
  int gemm_reserve = 0;
  unsigned* gemm_ctr = nullptr;  // its tile / worker counters (2 words, zeroed per launch)
  // Serialises the entry points on this context: its workspace, streams, pinned buffer
  // and events are shared state ("one solve at a time" per backend, backends.py:80-81).
  // Recursive: a GMRES workspace sink may call back into the library on this thread.
  std::recursive_mutex mu;
};

namespace ds {
int ctx_workspace(ds_ctx* ctx, size_t bytes, void** out);  // grow-only, zero-filled when (re)allocated
// Epoch of the next LL exchange (LU panel, fused Arnoldi step): unique in the process, so a
// workspace that reuses memory freed by another context can never hold a word that matches.
unsigned next_ll_epoch();
int ctx_hostbuf(ds_ctx* ctx, size_t bytes, void** out);
int ctx_begin(ds_ctx* ctx);  // cudaSetDevice
inline void count_launch(ds_ctx* ctx, int n = 1) { ctx->launches += n; }
}  // namespace ds

// Entry-point prologue: select the device and hold the context's lock until return.
#define DS_ENTER(ctx)                 \
  DS_TRY(::ds::ctx_begin(ctx));       \
  std::lock_guard<std::recursive_mutex> _ds_ctx_guard((ctx)->mu)

#define DS_DISPATCH(dtype, T, ...)                              \
  do {                                                          \
    if ((dtype) == DS_F64) {                                    \
      using T = double;                                         \
      __VA_ARGS__;                                              \
    } else if ((dtype) == DS_F32) {                             \
      using T = float;                                          \
      __VA_ARGS__;                                              \
    } else {                                                    \
      ::ds::set_error("unsupported dtype code %d", (int)(dtype)); \
      return DS_EPREC;                                          \
    }                                                           \
  } while (0)
