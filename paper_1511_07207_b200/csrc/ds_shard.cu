// ds_shard.cu — row-sharded CG across G shards (one per GPU), exchanges fused into the
// kernels over peer memory (NVLink P2P stores; CUDA IPC between processes).
//
// Restates krylov.cg_solve (/root/reference/pkg/src/densolve/krylov.py:36-72) on a
// row-sharded system, SURVEY.md §8e / BASELINE config C4 ("row-sharded across
// 1/2/4/8 B200").  Shard q owns rows [q*n_loc, (q+1)*n_loc) of A (an n_loc x n
// column-major block, zero rows past n) and of every vector.
//
// Exchange design (no NCCL on the data path, no host round trip per iteration):
//   * every shard owns one exchange region (cudaMalloc, IPC-exportable):
//       flags[G]            one monotonically increasing sequence word per SOURCE shard
//       rec[kinds][G][4]    one reduction record per source shard and kind
//       full[N]             the gathered iterate (p) — shard q's p IS full[q*n_loc ...]
//       xbuf                staging for the symmetry gate's transposed blocks
//   * a producer kernel writes its data straight into every peer's region (remote
//     stores: the all-gather of p is fused into the p-update kernel, the scalar
//     all-gathers into the kernels that finalise the per-shard records), fences at
//     system scope, then releases flags[self] = seq in every peer (st.release.sys);
//   * a consumer waits in a one-warp kernel (ld.acquire.sys poll, bounded by a
//     watchdog) before the kernel that reads the data.
//   Every shard combines the G records IN SHARD ORDER, so all shards compute
//   bitwise-identical alpha/beta/residuals and stop on the same iteration.
//   No double buffering is needed: each exchange of iteration k+1 is issued after a
//   wait that transitively orders it behind every consumer of the same buffer in
//   iteration k (p: finish(k) waits for r-records(k), which every shard publishes
//   after its GEMV(k) has read full; records likewise).
//
// Per iteration and shard:  [wait p] GEMV(partials) reduce(+p'Ap record, published by the
//   last CTA) [wait] update(x, r; the r record published by its last CTA) [wait]
//   finish(p -> own slice + every peer's slice; the last CTA releases the exchange):
//   seven launches, three of them one-warp waits.
// At G = 1 the waits, signals and record kernels vanish (the update and finish kernels
// read the local block partials directly): the fused single-GPU CG's four launches.
//
// Single process with several local shards (devices=[...]): one host thread per
// shard enqueues its shard's chunks; the chunk length follows the replicated stop
// word, so every shard enqueues the same number of iterations.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <ctime>
#include <mutex>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

constexpr int kMaxShards = DS_MAX_SHARDS;
enum { REC_B = 0, REC_PAP = 1, REC_R = 2, REC_GEN = 3, REC_KINDS = 4 };
constexpr int FLAG_BCAST = 16, FLAG_DONE = 32;  // offsets of the block-cyclic LU flag sets
constexpr int kRecW = 4;
constexpr int kShT = 256;

struct Peers {
  int G, rank;
  unsigned long long* flag[kMaxShards];  // shard t's flags (one word per source shard)
  double* rec[kMaxShards];               // shard t's records [REC_KINDS][kMaxShards][kRecW]
  char* full[kMaxShards];                // shard t's gathered vector
  char* xbuf[kMaxShards];                // shard t's staging buffer
  double* gr[kMaxShards];                // shard t's gather regions (GMRES records, rank-major)
};

// gather regions (doubles): two multi-dot record buffers (CGS pass parity) of G x kc and
// one (s2, scale, ssq) record buffer of G x 3, each written at [rank * cnt ...] by every shard
constexpr int GR_MD0 = 0, GR_MD1 = kMaxShards * 64, GR_P3 = 2 * kMaxShards * 64;
constexpr size_t kGrBytes = (size_t)(2 * kMaxShards * 64 + kMaxShards * 4) * sizeof(double);

__device__ __forceinline__ size_t rec_off(int kind, int src) {
  return ((size_t)kind * kMaxShards + src) * kRecW;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}

// one thread: release flags[self] = seq in every peer (after a system-scope fence)
__device__ __forceinline__ void signal_peers(const Peers& P, unsigned long long seq) {
  if (P.G <= 1) return;
  __threadfence_system();
  for (int t = 0; t < P.G; ++t)
    if (t != P.rank) st_release_sys(P.flag[t] + P.rank, seq);
}

// one warp: wait until every peer's word in the local flag array reached seq.  A stuck
// exchange (a dead peer) ends after `timeout_ns` with *err = 1 instead of hanging.
__global__ void sh_wait_kernel(const unsigned long long* flag, int G, int rank, unsigned long long seq,
                               int* err, unsigned long long timeout_ns) {
  const int t = threadIdx.x;
  if (t < G && t != rank) {
    const unsigned long long t0 = globaltimer_ns();
    unsigned long long v;
    while ((v = ld_acquire_sys(flag + t)) < seq) {
      if (globaltimer_ns() - t0 > timeout_ns) {
        // diagnostics for the host: the awaited sequence number and what each peer reached
        unsigned long long* dbg = reinterpret_cast<unsigned long long*>(err) + 1;
        dbg[0] = seq;
        dbg[1 + t] = v;
        __threadfence();
        atomicExch(err, 1);
        break;
      }
      __nanosleep(32);
    }
  }
}

__global__ void sh_signal_kernel(Peers P, unsigned long long seq) {
  if (threadIdx.x == 0) signal_peers(P, seq);
}

// Finalise this shard's record of `kind` from per-block partials (fixed block order),
// store it into every shard's record slot [kind][rank], then signal.
//   MODE 0: red[blk]                                   -> (sum, 0, 0)
//   MODE 1: red[3 blk], red[3 blk+1], red[3 blk+2]     -> (sum x^2, scale, ssq)
//   MODE 2: red[2 blk], red[2 blk+1], red[2 nblk+blk]  -> (sum x^2, scale, ssq)  (gemv EPI_RESID)
template <int MODE>
__global__ void __launch_bounds__(kShT) sh_publish_kernel(Peers P, const double* __restrict__ red, int nblk, int kind,
                                                          unsigned long long seq) {
  __shared__ double sm[64];
  double s = 0.0;
  Ssq q{0.0, 0.0};
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    if (MODE == 0) {
      s += red[i];
    } else if (MODE == 1) {
      s += red[3 * i];
      q = ssq_merge(q, Ssq{red[3 * i + 1], red[3 * i + 2]});
    } else {
      s += red[2 * nblk + i];
      q = ssq_merge(q, Ssq{red[2 * i], red[2 * i + 1]});
    }
  }
  s = block_sum(s, sm);
  if (MODE != 0) q = block_ssq(q, sm);
  if (threadIdx.x == 0) {
    for (int t = 0; t < P.G; ++t) {
      double* r = P.rec[t] + rec_off(kind, P.rank);
      r[0] = s;
      r[1] = q.scale;
      r[2] = q.ssq;
    }
    signal_peers(P, seq);
  }
}

// host scalars (a, b) into every shard's record [kind][rank], then signal
__global__ void sh_publish2_kernel(Peers P, double a, double b, int kind, unsigned long long seq) {
  if (threadIdx.x != 0) return;
  for (int t = 0; t < P.G; ++t) {
    double* r = P.rec[t] + rec_off(kind, P.rank);
    r[0] = a;
    r[1] = b;
  }
  signal_peers(P, seq);
}

// rank-ordered combination of G (sum, scale, ssq) records of one kind
__device__ __forceinline__ void combine_rec(const double* rec, int kind, int G, double& s, double& nrm) {
  s = 0.0;
  Ssq q{0.0, 0.0};
  for (int t = 0; t < G; ++t) {
    const double* r = rec + rec_off(kind, t);
    s += r[0];
    q = ssq_merge(q, Ssq{r[1], r[2]});
  }
  nrm = ssq_norm(q.scale, q.ssq);
}

// v (n_loc) -> own full slice and every peer's full slice at rank*n_loc
template <typename T>
__global__ void __launch_bounds__(kShT) sh_put_slice_kernel(Peers P, int64_t n_loc, const T* __restrict__ v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += (int64_t)gridDim.x * blockDim.x) {
    const T x = v[i];
    for (int t = 0; t < P.G; ++t) reinterpret_cast<T*>(P.full[t])[P.rank * n_loc + i] = x;
  }
  if (P.G > 1) __threadfence_system();
}

// a finalised local array (cnt doubles, device) into every shard's gather region at
// [off + rank * cnt], then signal (the all-gather of the GMRES records)
__global__ void sh_publish_array_kernel(Peers P, const double* __restrict__ src, int cnt, int off,
                                        unsigned long long seq) {
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    const double v = src[j];
    for (int t = 0; t < P.G; ++t) P.gr[t][off + P.rank * cnt + j] = v;
  }
  if (P.G > 1) __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) signal_peers(P, seq);
}

// ---- 1-D block-cyclic LU exchange kernels -------------------------------------------
// the owner's factored panel (rows kb..n of its column block, width w), its pivots (absolute)
// and zero-pivot flags into every peer's staging slot; then release the broadcast flag
template <typename T>
__global__ void __launch_bounds__(kShT)
    sh_bcast_panel_kernel(Peers P, const T* __restrict__ panel, int64_t ldp, int64_t mp, int64_t w,
                          const int64_t* __restrict__ piv, const int8_t* __restrict__ zero, size_t slot_off,
                          size_t piv_off, size_t zero_off, unsigned long long flag_val, unsigned* ticket) {
  const int64_t total = mp * w;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / mp, i = e - j * mp;
    const T v = panel[i + j * ldp];
    for (int t = 0; t < P.G; ++t)
      if (t != P.rank) reinterpret_cast<T*>(P.xbuf[t] + slot_off)[e] = v;
  }
  if (blockIdx.x == 0)
    for (int64_t j = threadIdx.x; j < w; j += blockDim.x)
      for (int t = 0; t < P.G; ++t)
        if (t != P.rank) {
          reinterpret_cast<int64_t*>(P.xbuf[t] + piv_off)[j] = piv[j];
          reinterpret_cast<int8_t*>(P.xbuf[t] + zero_off)[j] = zero[j];
        }
  __threadfence_system();
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence_system();
    for (int t = 0; t < P.G; ++t)
      if (t != P.rank) st_release_sys(P.flag[t] + FLAG_BCAST + P.rank, flag_val);
    *ticket = 0;
  }
}

// one flag word per peer at `off` (FLAG_DONE: every peer; single source: src >= 0)
__global__ void sh_wait_set_kernel(const unsigned long long* flag, int off, int G, int rank, int src,
                                   unsigned long long val, int* err, unsigned long long timeout_ns) {
  const int t = threadIdx.x;
  const bool mine = src >= 0 ? t == src : (t < G && t != rank);
  if (mine) {
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(flag + off + t) < val) {
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicExch(err, 1);
        break;
      }
      __nanosleep(32);
    }
  }
}

__global__ void sh_signal_set_kernel(Peers P, int off, unsigned long long val) {
  if (threadIdx.x != 0 || P.G <= 1) return;
  __threadfence_system();
  for (int t = 0; t < P.G; ++t)
    if (t != P.rank) st_release_sys(P.flag[t] + off + P.rank, val);
}

__global__ void sh_piv_offset_kernel(int64_t* piv, int64_t w, int64_t kb) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < w; j += (int64_t)gridDim.x * blockDim.x)
    piv[j] += kb;
}

__global__ void sh_any_kernel(const int8_t* z, int64_t n, int* out) {
  int a = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a |= z[i] != 0;
  a = __syncthreads_or(a);
  if (threadIdx.x == 0 && a) *out = 1;
}

struct ShCg {
  int64_t stop_it;  // gate word (Gate.stop_it)
  int32_t status;
  int32_t pad;
  double bad_val;
  double bnorm;
};

// ||b||, r0 = b - A x0 records -> res0, rs0, stop word (krylov.py:45-52)
__global__ void sh_cg_init_kernel(const double* rec, int G, ShCg* st, double* rs_hist, double* hist, double tol,
                                  int64_t cap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double bs2, bn, rs, rn;
  combine_rec(rec, REC_B, G, bs2, bn);
  combine_rec(rec, REC_R, G, rs, rn);
  st->bnorm = bn;
  st->status = DS_OK;
  st->bad_val = 0.0;
  if (bn == 0.0) {
    st->stop_it = 0;
    return;
  }
  const double res = rn / bn;
  hist[0] = res;
  rs_hist[0] = rs;
  st->stop_it = (res > tol && 0 < cap) ? cap : 0;
}

// Last-CTA helper: every CTA has stored its block partial; the CTA that arrives last
// (ticket) sees all of them (fence + atomic, the classic threadfence reduction).
__device__ __forceinline__ bool last_cta(unsigned* ticket) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// the (s2, scale, ssq) record of nblk block partials red[3 blk ..] in block order, stored into
// every shard's slot [kind][rank], then signal (== sh_publish_kernel<1>, fused into its producer)
__device__ __forceinline__ void publish_parts3(const Peers& P, const double* red, int nblk, int kind,
                                               unsigned long long seq, double* sm) {
  double s2 = 0.0;
  Ssq q{0.0, 0.0};
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    s2 += red[3 * i];
    q = ssq_merge(q, Ssq{red[3 * i + 1], red[3 * i + 2]});
  }
  s2 = block_sum(s2, sm);
  q = block_ssq(q, sm);
  if (threadIdx.x == 0) {
    for (int t = 0; t < P.G; ++t) {
      double* r = P.rec[t] + rec_off(kind, P.rank);
      r[0] = s2;
      r[1] = q.scale;
      r[2] = q.ssq;
    }
    signal_peers(P, seq);
  }
}

// alpha = rs/pAp (pAp from the shard-ordered records); x += alpha p; r -= alpha Ap;
// (r.r, scale, ssq) partials per block (krylov.py:55-61).  G > 1: the last CTA finalises this
// shard's r record and publishes it to the peers (no separate record kernel).
template <typename T>
__global__ void __launch_bounds__(kShT)
    sh_cg_update_kernel(int64_t n, Peers P, const double* __restrict__ rec, const double* __restrict__ red_pap,
                        int nblk_pap, ShCg* st, const double* __restrict__ rs_hist, T* __restrict__ x,
                        T* __restrict__ r, const T* __restrict__ p, const T* __restrict__ Ap, double* __restrict__ red,
                        Gate gate, unsigned* ticket, unsigned long long seq) {
  const int G = P.G;
  const bool skip = gated(gate);
  if (skip && G == 1) return;
  __shared__ double sm[64];
  double pAp = 0.0;
  if (!skip) {
    if (G == 1) {  // one shard: the GEMV's block partials directly (no record round trip)
      pAp = reduce_sum_partials(red_pap, nblk_pap, sm);
    } else {
      for (int t = 0; t < G; ++t) pAp += rec[rec_off(REC_PAP, t)];
    }
  }
  const bool notspd = !skip && pAp <= 0.0;
  if (notspd && blockIdx.x == 0 && threadIdx.x == 0) {  // krylov.py:57-58
    st->status = DS_ENOTSPD;
    st->bad_val = pAp;
    st->stop_it = gate.k;
  }
  if (!skip && !notspd) {
    const double alpha = rs_hist[gate.k] / pAp;
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
  if (G > 1 && last_cta(ticket)) {  // (stale partials after a stop: the consumers are gated)
    publish_parts3(P, red, gridDim.x, REC_R, seq, sm);
    if (threadIdx.x == 0) *ticket = 0;
  }
}

// GEMV stage 2 of the sharded CG (G > 1): Ap = sum of the chunk partials (chunk order),
// the block partials of p'Ap, and the last CTA publishes this shard's p'Ap record
template <typename T>
__global__ void __launch_bounds__(kShT)
    sh_cg_reduce_pap_kernel(Peers P, const double* __restrict__ part, int64_t m, int64_t nchunks, T* Ap,
                            const T* __restrict__ p, double* __restrict__ red, Gate gate, unsigned* ticket,
                            unsigned long long seq) {
  __shared__ double sm[64];
  if (!gated(gate)) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double d = 0.0;
    if (i < m) {
      double s = 0.0;
      int64_t c = 0;
      for (; c + 8 <= nchunks; c += 8) {  // the chunk order of ds_colstream_reduce_kernel
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = part[(c + u) * m + i];
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
      }
      for (; c < nchunks; ++c) s += part[c * m + i];
      const T yi = (T)s;
      Ap[i] = yi;
      d = (double)p[i] * (double)yi;
    }
    d = block_sum(d, sm);
    if (threadIdx.x == 0) red[blockIdx.x] = d;
  }
  if (last_cta(ticket)) {
    double s = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) s += red[b];
    s = block_sum(s, sm);
    if (threadIdx.x == 0) {
      for (int t = 0; t < P.G; ++t) P.rec[t][rec_off(REC_PAP, P.rank)] = s;
      signal_peers(P, seq);
      *ticket = 0;
    }
  }
}

// beta = rs_new/rs; p = r + beta p written into the own slice of full AND every peer's
// slice (the all-gather of p fused into the update); history and stop word (:62-67)
template <typename T>
__global__ void __launch_bounds__(kShT)
    sh_cg_finish_kernel(int64_t n_loc, Peers P, const double* __restrict__ rec, const double* __restrict__ red,
                        int nblk, const T* __restrict__ r, double* rs_hist, double* hist, ShCg* st, double tol,
                        int64_t cap, Gate gate, unsigned* ticket, unsigned long long seq) {
  if (gated(gate)) {
    // G > 1: still release this exchange (the peers wait for it; nothing was written)
    if (P.G > 1 && last_cta(ticket) && threadIdx.x == 0) {
      signal_peers(P, seq);
      *ticket = 0;
    }
    return;
  }
  double rs_new, nrm;
  if (P.G == 1) {  // one shard: the update's block partials directly
    __shared__ double sm[64];
    double s2 = 0.0;
    Ssq q{0.0, 0.0};
    for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
      s2 += red[3 * i];
      q = ssq_merge(q, Ssq{red[3 * i + 1], red[3 * i + 2]});
    }
    rs_new = block_sum(s2, sm);
    q = block_ssq(q, sm);
    nrm = ssq_norm(q.scale, q.ssq);
  } else {
    combine_rec(rec, REC_R, P.G, rs_new, nrm);
  }
  const int64_t k = gate.k;
  const double beta = rs_new / rs_hist[k];
  const T bt = (T)beta;
  T* p = reinterpret_cast<T*>(P.full[P.rank]) + P.rank * n_loc;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += (int64_t)gridDim.x * blockDim.x) {
    const T pv = add_rn(r[i], mul_rn(bt, p[i]));
    p[i] = pv;
    for (int t = 0; t < P.G; ++t)
      if (t != P.rank) reinterpret_cast<T*>(P.full[t])[P.rank * n_loc + i] = pv;
  }
  if (P.G > 1) __threadfence_system();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double res = nrm / st->bnorm;
    rs_hist[k + 1] = rs_new;
    hist[k + 1] = res;
    if (!(res > tol) || k + 1 >= cap) st->stop_it = k + 1;
  }
  // G > 1: the p slices of every CTA are in the peers' regions: the last CTA releases them
  if (P.G > 1 && last_cta(ticket) && threadIdx.x == 0) {
    signal_peers(P, seq);
    *ticket = 0;
  }
}

// (sum x^2, scale, ssq) partials of a local vector
template <typename T>
__global__ void __launch_bounds__(kShT) sh_parts_kernel(int64_t n, const T* __restrict__ x, double* red) {
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

// column block [c0, c0 + w) of the local row block (n_loc rows, ld lda) -> dst (ld n_loc),
// written into a peer's staging buffer (the symmetry gate's block exchange)
template <typename T>
__global__ void __launch_bounds__(kShT) sh_copy_block_kernel(int64_t n_loc, int64_t w, const T* __restrict__ A,
                                                             int64_t lda, T* __restrict__ dst) {
  const int64_t total = n_loc * w;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / n_loc, i = e - j * n_loc;
    dst[e] = A[i + j * lda];
  }
  __threadfence_system();
}

}  // namespace ds

using namespace ds;

// ---------------------------------------------------------------------------
// the shard set
// ---------------------------------------------------------------------------
struct ShardLocal {
  ds_ctx* ctx = nullptr;
  int rank = 0;
  char* region = nullptr;  // cudaMalloc'd exchange region
  size_t region_bytes = 0;
  void* sws = nullptr;     // the solver's own device buffers (grow-only, allocated before any exchange)
  size_t sws_bytes = 0;
  unsigned long long* flag = nullptr;
  double* rec = nullptr;
  double* gr = nullptr;
  char* full = nullptr;
  char* xbuf = nullptr;
  int* err = nullptr;  // watchdog word (in the region)
  Peers peers{};
  std::vector<void*> opened;  // IPC-mapped peer regions (closed on destroy)
  unsigned long long seq = 0;
  unsigned long long lu_epoch = 0;  // block-cyclic LU: flag values of earlier factorizations
};

struct ds_shardset {
  int G = 1;
  int64_t n = 0, n_loc = 0, N = 0;
  size_t elem = 8;
  size_t xbytes = 0;
  bool connected = false;
  bool broken = false;
  std::vector<ShardLocal> loc;
};

namespace {

constexpr size_t kFlagBytes = 512;  // words 0..15: exchange sequence; 16..31: LU broadcasts; 32..47: LU done
constexpr size_t kRecBytes = (size_t)REC_KINDS * kMaxShards * kRecW * sizeof(double);  // 2 KB
constexpr size_t kErrBytes = 256;

size_t round256(size_t b) { return (b + 255) / 256 * 256; }

struct Layout {
  size_t flag, rec, gr, err, full, xbuf, total;
};
Layout layout_of(const ds_shardset* s) {
  Layout L;
  L.flag = 0;
  L.rec = kFlagBytes;
  L.gr = L.rec + round256(kRecBytes);
  L.err = L.gr + round256(kGrBytes);
  L.full = L.err + kErrBytes;
  L.xbuf = L.full + round256((size_t)s->N * s->elem);
  L.total = L.xbuf + round256(std::max<size_t>(s->xbytes, 256));
  return L;
}

void bind_region(ShardLocal& S, const Layout& L, char* base) {
  S.flag = reinterpret_cast<unsigned long long*>(base + L.flag);
  S.rec = reinterpret_cast<double*>(base + L.rec);
  S.gr = reinterpret_cast<double*>(base + L.gr);
  S.err = reinterpret_cast<int*>(base + L.err);
  S.full = base + L.full;
  S.xbuf = base + L.xbuf;
}

unsigned long long watchdog_ns() {
  const char* e = getenv("DENSOLVE_SHARD_TIMEOUT_S");
  const double s = e ? atof(e) : 120.0;
  return (unsigned long long)(s * 1e9);
}

// Host barrier of the local shard threads: every shard finishes its allocations before
// any shard enqueues an exchange.  An allocation may synchronise the whole device
// (cudaMalloc of a first workspace, pinned host memory), and on a GPU shared by several
// local shards that would wait for a peer's exchange kernel spinning on this shard.
struct HostBarrier {
  std::mutex m;
  std::condition_variable cv;
  int n, arrived = 0;
  explicit HostBarrier(int n_) : n(n_) {}
  void arrive_and_wait() {
    std::unique_lock<std::mutex> lk(m);
    if (++arrived >= n) {
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return arrived >= n; });
  }
};

bool trace_on() {
  static const bool on = getenv("DENSOLVE_SHARD_TRACE") != nullptr;
  return on;
}
void trace(const ShardLocal& S, const char* what) {
  if (!trace_on()) return;
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  fprintf(stderr, "[shard %d %.6f] %s seq=%llu\n", S.rank, ts.tv_sec + 1e-9 * ts.tv_nsec, what, S.seq);
}

// ---- exchange primitives (host side, on the shard's stream) ------------------
int sh_wait(ShardLocal& S, const ds_shardset* ss) {
  trace(S, "wait");
  if (ss->G <= 1) return DS_OK;
  sh_wait_kernel<<<1, 32, 0, S.ctx->stream>>>(S.flag, ss->G, S.rank, S.seq, S.err, watchdog_ns());
  count_launch(S.ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
int sh_signal(ShardLocal& S, const ds_shardset* ss) {
  ++S.seq;
  trace(S, "signal");
  if (ss->G <= 1) return DS_OK;
  sh_signal_kernel<<<1, 32, 0, S.ctx->stream>>>(S.peers, S.seq);
  count_launch(S.ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
// a barrier over all shards (signal everyone, wait for everyone)
int sh_barrier(ShardLocal& S, const ds_shardset* ss) {
  DS_TRY(sh_signal(S, ss));
  return sh_wait(S, ss);
}
template <int MODE>
int sh_publish(ShardLocal& S, const ds_shardset* ss, const double* red, int nblk, int kind) {
  ++S.seq;
  sh_publish_kernel<MODE><<<1, kShT, 0, S.ctx->stream>>>(S.peers, red, nblk, kind, S.seq);
  count_launch(S.ctx);
  DS_CHECK_LAUNCH();
  return sh_wait(S, ss);
}

int check_watchdog(ShardLocal& S) {
  unsigned long long h[1 + 1 + kMaxShards] = {};
  DS_CUDA(cudaMemcpyAsync(h, S.err, sizeof h, cudaMemcpyDeviceToHost, S.ctx->stream));
  DS_CUDA(cudaStreamSynchronize(S.ctx->stream));
  if ((int)h[0]) {
    std::string fl;
    for (int t = 0; t < S.peers.G; ++t) fl += (t ? "," : "") + std::to_string(h[2 + t]);
    set_error("sharded solve: shard %d waited for exchange %llu past DENSOLVE_SHARD_TIMEOUT_S "
              "(peers reached [%s]; 0 = this shard or not reported)",
              S.rank, h[1], fl.c_str());
    return DS_ECUDA;
  }
  return DS_OK;
}

int vgrid(ds_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(std::max<int64_t>(n, 1), kShT), (int64_t)ctx->num_sms * 2));
}

// symmetric gate on the row-sharded matrix (krylov.py:41-44): round s compares the
// block A[rows q, cols d] (d = q + s mod G) received from shard q against the transpose
// of this shard's A[rows d, cols q]; max over shards of (max|A - A^T|, max|A|).
template <typename T>
int sh_symmetry(ShardLocal& S, ds_shardset* ss, const T* A, int64_t lda, double* md_out, double* am_out) {
  const int G = ss->G, q = S.rank;
  const int64_t n = ss->n, nl = ss->n_loc;
  auto cw = [&](int r) { return std::max<int64_t>(0, std::min<int64_t>(n, (int64_t)(r + 1) * nl) - (int64_t)r * nl); };
  double md = 0.0, am = 0.0;
  auto fold = [&](double d, double a) {
    md = (d != d) ? d : (md != md ? md : std::max(md, d));
    am = (a != a) ? a : (am != am ? am : std::max(am, a));
  };
  const int dcode = sizeof(T) == 8 ? DS_F64 : DS_F32;
  double out[2];
  trace(S, "sym round 0");
  // round 0: the diagonal block against its own transpose (the square gate kernel, each
  // symmetric pair read once; rows past n are zero padding and not compared)
  if (cw(q) > 0) {
    DS_TRY(ds_symmetry_check(S.ctx, dcode, cw(q), A + (int64_t)q * nl * lda, lda, &out[0], &out[1]));
    fold(out[0], out[1]);
  }
  trace(S, "sym round 0 done");
  // max|A| over the off-diagonal column groups too
  for (int s = 1; s < G; ++s) {
    const int d = (q + s) % G;   // this shard sends A[rows q, cols d] to shard d
    const int src = (q - s + G) % G;  // and receives A[rows src, cols q] from shard src
    if (cw(d) > 0) {
      sh_copy_block_kernel<T><<<S.ctx->num_sms * 2, kShT, 0, S.ctx->stream>>>(
          nl, cw(d), A + (int64_t)d * nl * lda, lda, reinterpret_cast<T*>(S.peers.xbuf[d]));
      count_launch(S.ctx);
      DS_CHECK_LAUNCH();
    }
    DS_TRY(sh_barrier(S, ss));
    trace(S, "sym barrier enqueued");
    // xbuf = A[rows src, cols q] (nl x cw(q), ld nl); own block A[rows q, cols src] (nl x cw(src))
    if (cw(src) > 0 && cw(q) > 0) {
      DS_TRY(ds_absdiff_transposed(S.ctx, dcode, cw(q), cw(src), A + (int64_t)src * nl * lda, lda,
                                   reinterpret_cast<const T*>(S.xbuf), nl, out));
      fold(out[0], out[1]);
      trace(S, "sym compare done");
      // max|A| of the own off-diagonal block: absdiff's second value covers the first operand
    }
    DS_TRY(sh_barrier(S, ss));  // the staging buffer may be overwritten in the next round
  }
  // max over shards: each shard's (md, am) record, combined in shard order on the host
  ++S.seq;
  sh_publish2_kernel<<<1, 32, 0, S.ctx->stream>>>(S.peers, md, am, REC_GEN, S.seq);
  count_launch(S.ctx);
  DS_CHECK_LAUNCH();
  DS_TRY(sh_wait(S, ss));
  std::vector<double> h((size_t)kMaxShards * kRecW);
  DS_CUDA(cudaMemcpyAsync(h.data(), S.rec + (size_t)REC_GEN * kMaxShards * kRecW, h.size() * sizeof(double),
                          cudaMemcpyDeviceToHost, S.ctx->stream));
  DS_CUDA(cudaStreamSynchronize(S.ctx->stream));
  DS_TRY(check_watchdog(S));
  md = 0.0;
  am = 0.0;
  for (int t = 0; t < G; ++t) fold(h[(size_t)t * kRecW], h[(size_t)t * kRecW + 1]);
  *md_out = md;
  *am_out = am;
  return DS_OK;
}

template <typename T>
int sh_cg_run(ShardLocal& S, ds_shardset* ss, const T* A, int64_t lda, const T* b, const T* x0, T* x, double tol,
              int64_t cap, int check_sym, double* h_hist, int64_t hist_cap, ds_solve_info* info,
              HostBarrier* allocated) {
  ds_ctx* ctx = S.ctx;
  const int64_t launches0 = ctx->launches;
  const int G = ss->G;
  const int64_t n = ss->n, nl = ss->n_loc;
  const double u = (sizeof(T) == 8 ? 1.1102230246251565e-16 : 5.960464477539063e-08);
  const GemvPlan gp = gemv_plan(ctx, nl, n, sizeof(T));
  const int rblocks = (int)ceil_div(std::max<int64_t>(nl, 1), 256);
  const int vg = vgrid(ctx, nl);
  size_t need = gp.part_bytes + 256;
  need += (size_t)nl * sizeof(T) * 2 + 2 * 256;  // r, Ap
  need += ((size_t)std::max(rblocks, vg) * 3 + 64) * sizeof(double) * 2 + 2 * 256;
  need += (size_t)(cap + 2) * sizeof(double) * 2 + 2 * 256;
  need += sizeof(ShCg) + 256 + 256;
  // Every allocation of the call happens here, before the first exchange: an allocation
  // that synchronises the device (cudaFree of a smaller workspace, pinned host memory)
  // would otherwise wait on a peer shard's exchange kernel sharing this GPU.
  void* ws = nullptr;
  int64_t* h_stop = nullptr;
  int ast = ctx_workspace(ctx, std::max<size_t>(need, (size_t)ctx->num_sms * 64 * sizeof(double) + 4096), &ws);
  if (ast == DS_OK) ast = ctx_hostbuf(ctx, 64, (void**)&h_stop);
  if (allocated) allocated->arrive_and_wait();
  if (ast != DS_OK) {
    ss->broken = true;  // the peers are about to wait for this shard's exchanges
    return ast;
  }
  DS_CUDA(cudaMemsetAsync(S.err, 0, kErrBytes, ctx->stream));
  if (check_sym) {
    double md = 0, am = 0;
    DS_TRY(sh_symmetry<T>(S, ss, A, lda, &md, &am));
    if (md > 10.0 * u * am) {  // krylov.py:42-44
      set_error("matrix is not symmetric");
      info->error_index = -1;
      return DS_ENOTSPD;
    }
  }
  Carver cv{(char*)ws};
  double* part = cv.take<double>(gp.part_bytes);
  T* r = cv.take<T>((size_t)nl * sizeof(T));
  T* Ap = cv.take<T>((size_t)nl * sizeof(T));
  double* red_a = cv.take<double>(((size_t)std::max(rblocks, vg) * 3 + 64) * sizeof(double));
  double* red_b = cv.take<double>(((size_t)std::max(rblocks, vg) * 3 + 64) * sizeof(double));
  double* rs_hist = cv.take<double>((size_t)(cap + 2) * sizeof(double));
  double* hist = cv.take<double>((size_t)(cap + 2) * sizeof(double));
  ShCg* st = cv.take<ShCg>(sizeof(ShCg));
  unsigned* tickets = cv.take<unsigned>(64);  // last-CTA tickets of the fused record kernels
  T* full = reinterpret_cast<T*>(S.full);
  T* p = full + (int64_t)S.rank * nl;

  // ||b|| record (krylov.py:45 -> _rhs_norm)
  sh_parts_kernel<T><<<vg, kShT, 0, ctx->stream>>>(nl, b, red_b);
  count_launch(ctx);
  DS_TRY(sh_publish<1>(S, ss, red_b, vg, REC_B));
  // x = x0.copy(); gather x into full; r = b - A x  (krylov.py:46-47)
  if (x != x0) DS_CUDA(cudaMemcpyAsync(x, x0, nl * sizeof(T), cudaMemcpyDeviceToDevice, ctx->stream));
  sh_put_slice_kernel<T><<<vg, kShT, 0, ctx->stream>>>(S.peers, nl, x);
  count_launch(ctx);
  DS_TRY(sh_signal(S, ss));
  DS_TRY(sh_wait(S, ss));
  int rb = 0;
  DS_TRY(gemv_launch<T>(ctx, gp, A, lda, full, r, part, EPI_RESID, b, red_a, &rb));
  DS_TRY(sh_publish<2>(S, ss, red_a, rb, REC_R));
  sh_cg_init_kernel<<<1, 32, 0, ctx->stream>>>(S.rec, G, st, rs_hist, hist, tol, cap);
  count_launch(ctx);
  // p = r, gathered
  sh_put_slice_kernel<T><<<vg, kShT, 0, ctx->stream>>>(S.peers, nl, r);
  count_launch(ctx);
  DS_TRY(sh_signal(S, ss));
  DS_CHECK_LAUNCH();
  DS_CUDA(cudaMemsetAsync(tickets, 0, 64, ctx->stream));
  ShCg hst;
  DS_CUDA(cudaMemcpyAsync(&hst, st, sizeof(ShCg), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hst.bnorm == 0.0) {
    DS_TRY(sh_wait(S, ss));  // keep the exchange sequence aligned with the peers
    set_error("||b|| = 0");
    return DS_EDEGRHS;
  }

  int64_t k = 0, chunk = 2;
  while (true) {
    DS_CUDA(cudaMemcpyAsync(h_stop, &st->stop_it, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA(cudaStreamSynchronize(ctx->stream));
    DS_TRY(check_watchdog(S));
    const int64_t stop_it = *h_stop;
    if (stop_it <= k || k >= cap) break;
    const int64_t kend = std::min<int64_t>(cap, k + chunk);
    for (; k < kend; ++k) {
      const Gate g{&st->stop_it, k};
      DS_TRY(sh_wait(S, ss));  // every shard's slice of p is in full
      int rb2 = 0;
      if (G == 1) {
        DS_TRY(gemv_launch<T>(ctx, gp, A, lda, full, Ap, part, EPI_DOT, p, red_a, &rb2, g));
      } else {  // stage 2 with the p'Ap record published by its last CTA
        DS_TRY(gemv_launch<T>(ctx, gp, A, lda, full, Ap, part, EPI_PARTIAL, nullptr, nullptr, nullptr, g));
        rb2 = (int)ceil_div(nl, 256);
        ++S.seq;
        sh_cg_reduce_pap_kernel<T><<<rb2, kShT, 0, ctx->stream>>>(S.peers, part, nl, gp.nchunks, Ap, p, red_a, g,
                                                                  tickets, S.seq);
        count_launch(ctx);
        DS_TRY(sh_wait(S, ss));
      }
      if (G > 1) ++S.seq;
      sh_cg_update_kernel<T><<<vg, kShT, 0, ctx->stream>>>(nl, S.peers, S.rec, red_a, rb2, st, rs_hist, x, r, p, Ap,
                                                           red_b, g, tickets + 1, S.seq);
      count_launch(ctx);
      if (G > 1) DS_TRY(sh_wait(S, ss));
      ++S.seq;  // the p exchange: released by the finish kernel's last CTA
      sh_cg_finish_kernel<T><<<vg, kShT, 0, ctx->stream>>>(nl, S.peers, S.rec, red_b, vg, r, rs_hist, hist, st,
                                                           tol, cap, g, tickets + 2, S.seq);
      count_launch(ctx);
    }
    DS_CHECK_LAUNCH();
    chunk = std::min<int64_t>(chunk * 2, 64);
  }
  DS_TRY(sh_wait(S, ss));  // the last p exchange (nothing reads it; keeps peers' writes out of the next call)
  DS_CUDA(cudaMemcpyAsync(&hst, st, sizeof(ShCg), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  DS_TRY(check_watchdog(S));
  if (hst.status == DS_ENOTSPD) {
    set_error("p'Ap = %.17g <= 0: matrix is not positive definite", hst.bad_val);
    info->error_value = hst.bad_val;
    info->error_index = hst.stop_it;
    return DS_ENOTSPD;
  }
  const int64_t iters = std::min<int64_t>(hst.stop_it, cap);
  const int64_t hl = std::min<int64_t>(iters + 1, hist_cap);
  if (h_hist && hl > 0)
    DS_CUDA(cudaMemcpyAsync(h_hist, hist, hl * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  double res = 0;
  DS_CUDA(cudaMemcpyAsync(&res, hist + iters, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  info->iterations = iters;
  info->history_len = hl;
  info->final_relative_residual = res;
  info->converged = res <= tol;  // krylov.py:68
  info->breakdown = DS_BREAKDOWN_NONE;
  info->kernel_launches = ctx->launches - launches0;
  return DS_OK;
}

// ---- row-sharded GMRES(m) (krylov.py:75-182) ------------------------------------
// The host logic of distributed.gmres_solve_sharded in C++: every exchange is an
// all-gather over the peer-memory regions (v_k slices into `full`, multi-dot records per
// CGS pass, (s2, scale, ssq) norm records), the per-shard compute is the ds_dist.cu shard
// kernels.  All shards hold identical H, Givens rotations, estimates and stop decisions.
void combine3_host(const double* parts, int G, double* s2_out, double* nrm_out) {
  double s2 = 0.0, scale = 0.0, ssq = 0.0;  // rank-ordered, as the device combine3
  for (int q = 0; q < G; ++q) {
    s2 += parts[3 * q];
    const double bs = parts[3 * q + 1], bq = parts[3 * q + 2];
    if (scale != scale) continue;
    if (bs != bs) {
      scale = bs;
      ssq = bq;
      continue;
    }
    if (std::isinf(scale) || std::isinf(bs)) {
      scale = INFINITY;
      ssq = 1.0;
      continue;
    }
    if (bs == 0.0) continue;
    if (scale == 0.0) {
      scale = bs;
      ssq = bq;
      continue;
    }
    if (scale >= bs) {
      const double r = bs / scale;
      ssq = ssq + bq * r * r;
    } else {
      const double r = scale / bs;
      const double ns = bq + ssq * r * r;
      scale = bs;
      ssq = ns;
    }
  }
  *s2_out = s2;
  *nrm_out = (scale == 0.0 || !(scale - scale == 0.0)) ? scale : scale * std::sqrt(ssq);
}

enum { GST_RS = 0, GST_BNORM = 1, GST_STATUS = 2, GST_STOP = 3, GST_BAD = 4, GST_RES = 5 };

template <typename T>
int sh_gmres_run(ShardLocal& S, ds_shardset* ss, const T* A, int64_t lda, const T* b, const T* x0, T* x, double tol,
                 int64_t cap, int64_t m, int orth, double* h_hist, int64_t hist_cap, int64_t* h_cycles,
                 int64_t cycles_cap, ds_solve_info* info, HostBarrier* allocated) {
  ds_ctx* ctx = S.ctx;
  const int64_t launches0 = ctx->launches;
  const int G = ss->G;
  const int64_t n = ss->n, nl = ss->n_loc;
  const int dt = sizeof(T) == 8 ? DS_F64 : DS_F32;
  const double u = (sizeof(T) == 8 ? 1.1102230246251565e-16 : 5.960464477539063e-08);
  const int passes = orth == DS_ORTH_CLASSICAL ? 1 : 2;
  // scratch of the ds_* shard entry points (the context workspace, reused from offset 0 by
  // each call) and this solver's own buffers: both sized here, before any exchange
  const GemvPlan gp = gemv_plan(ctx, nl, n, sizeof(T));
  const int vg = vgrid(ctx, nl);
  const size_t ws_need = std::max<size_t>(gp.part_bytes + 4096, ((size_t)vg * 64 + 64) * sizeof(double) + 4096);
  const int64_t ldv = ceil_div(std::max<int64_t>(nl, 1), 4) * 4;
  const int64_t ldh = m + 1;
  size_t need = 0;
  need += 256 + (size_t)ldv * (m + 1) * sizeof(T);      // V
  need += 256 + (size_t)ldh * m * sizeof(T) * 2;        // H, Hraw
  need += 256 + (size_t)(m + 2) * sizeof(T) * 3;        // g, cs, sn
  need += 256 + 64 * sizeof(T);                         // y
  need += 256 + (size_t)nl * sizeof(T);                 // r
  need += 256 + (64 + 64 + 16 + 64) * sizeof(double);   // hsave, est, state (16: ST_* + int64 stop mirror), md
  int ast = DS_OK;
  void* ws = nullptr;
  ast = ctx_workspace(ctx, ws_need, &ws);
  if (ast == DS_OK && need > S.sws_bytes) {
    if (S.sws) cudaFree(S.sws);
    S.sws = nullptr;
    S.sws_bytes = 0;
    if (cudaMalloc(&S.sws, need) == cudaSuccess)
      S.sws_bytes = need;
    else
      ast = DS_ENOMEM;
  }
  double* h_st = nullptr;
  if (ast == DS_OK) ast = ctx_hostbuf(ctx, 64 * sizeof(double) + kMaxShards * 3 * sizeof(double), (void**)&h_st);
  if (allocated) allocated->arrive_and_wait();
  if (ast != DS_OK) {
    ss->broken = true;
    if (ast == DS_ENOMEM) set_error("sharded GMRES: device buffers (%zu bytes) could not be allocated", need);
    return ast;
  }
  DS_CUDA(cudaMemsetAsync(S.err, 0, kErrBytes, ctx->stream));
  Carver cv{(char*)S.sws};
  T* V = cv.take<T>((size_t)ldv * (m + 1) * sizeof(T));
  T* H = cv.take<T>((size_t)ldh * m * sizeof(T));
  T* Hraw = cv.take<T>((size_t)ldh * m * sizeof(T));
  T* g = cv.take<T>((size_t)(m + 2) * sizeof(T));
  T* cs = cv.take<T>((size_t)(m + 2) * sizeof(T));
  T* sn = cv.take<T>((size_t)(m + 2) * sizeof(T));
  T* y = cv.take<T>(64 * sizeof(T));
  T* r = cv.take<T>((size_t)nl * sizeof(T));
  double* hsave = cv.take<double>(64 * sizeof(double));
  double* est = cv.take<double>(64 * sizeof(double));
  double* st = cv.take<double>(16 * sizeof(double));
  double* md = cv.take<double>(64 * sizeof(double));  // this shard's multi-dot record / (s2, scale, ssq)
  T* full = reinterpret_cast<T*>(S.full);
  double* p3_all = S.gr + GR_P3;
  double* h_p3 = h_st + 64;

  auto gather_vec = [&](const T* v) -> int {  // v (n_loc) -> every shard's full
    sh_put_slice_kernel<T><<<vg, kShT, 0, ctx->stream>>>(S.peers, nl, v);
    count_launch(ctx);
    DS_CHECK_LAUNCH();
    DS_TRY(sh_signal(S, ss));
    return sh_wait(S, ss);
  };
  auto publish = [&](const double* src, int cnt, int off) -> int {
    ++S.seq;
    sh_publish_array_kernel<<<1, 64, 0, ctx->stream>>>(S.peers, src, cnt, off, S.seq);
    count_launch(ctx);
    DS_CHECK_LAUNCH();
    return sh_wait(S, ss);
  };
  auto read_p3 = [&](double* s2, double* nrm) -> int {  // the G (s2, scale, ssq) records, host-combined
    DS_CUDA(cudaMemcpyAsync(h_p3, p3_all, (size_t)G * 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA(cudaStreamSynchronize(ctx->stream));
    DS_TRY(check_watchdog(S));
    combine3_host(h_p3, G, s2, nrm);
    return DS_OK;
  };
  auto residual = [&](double* s2, double* nrm) -> int {  // r = b - A x (krylov.py:104), its record
    DS_TRY(gather_vec(x));
    DS_TRY(ds_resid_parts(ctx, dt, nl, n, A, lda, full, b, r, md));
    DS_TRY(publish(md, 3, GR_P3));
    return read_p3(s2, nrm);
  };

  // ||b|| (krylov.py:87 -> _rhs_norm)
  DS_TRY(ds_vec_parts(ctx, dt, nl, b, md));
  DS_TRY(publish(md, 3, GR_P3));
  double s2b = 0.0, bnorm = 0.0;
  DS_TRY(read_p3(&s2b, &bnorm));
  if (bnorm == 0.0) {
    set_error("||b|| = 0");
    return DS_EDEGRHS;
  }
  const double bnorm_plain = std::sqrt(s2b);
  if (x != x0) DS_CUDA(cudaMemcpyAsync(x, x0, nl * sizeof(T), cudaMemcpyDeviceToDevice, ctx->stream));
  {
    double h0[8] = {0, bnorm, 0, 0, 0, 0, 0, 0};
    DS_CUDA(cudaMemcpyAsync(st, h0, sizeof h0, cudaMemcpyHostToDevice, ctx->stream));
  }
  std::vector<double> history;
  std::vector<int64_t> cycles;
  int64_t total = 0, resid_evals = 0;
  int breakdown = DS_BREAKDOWN_NONE;
  bool converged = false;
  const size_t vbytes = (size_t)ldv * (m + 1) * sizeof(T), hbytes = (size_t)ldh * m * sizeof(T);
  while (true) {
    double s2r = 0.0, beta = 0.0;
    DS_TRY(residual(&s2r, &beta));
    ++resid_evals;
    const double relres = beta / bnorm;
    if (total == 0) history.push_back(relres);
    if (relres <= tol) {
      converged = true;
      break;
    }
    if (total >= cap) break;
    cycles.push_back(total);
    const double start_res = relres;
    DS_CUDA(cudaMemsetAsync(V, 0, vbytes, ctx->stream));
    DS_CUDA(cudaMemsetAsync(H, 0, hbytes, ctx->stream));
    DS_CUDA(cudaMemsetAsync(Hraw, 0, hbytes, ctx->stream));
    DS_CUDA(cudaMemsetAsync(g, 0, (size_t)(m + 2) * sizeof(T), ctx->stream));
    DS_CUDA(cudaMemsetAsync(cs, 0, (size_t)(m + 2) * sizeof(T), ctx->stream));
    DS_CUDA(cudaMemsetAsync(sn, 0, (size_t)(m + 2) * sizeof(T), ctx->stream));
    {
      const double hs[3] = {0.0, (double)m, 0.0};  // status, stop, happy
      DS_CUDA(cudaMemcpyAsync(st + GST_STATUS, hs, sizeof hs, cudaMemcpyHostToDevice, ctx->stream));
      const int64_t stop64 = m;  // the GEMVs' Gate word (int64 mirror of the stop, slot 8)
      DS_CUDA(cudaMemcpyAsync(st + 8, &stop64, sizeof stop64, cudaMemcpyHostToDevice, ctx->stream));
    }
    DS_TRY(ds_gmres_shard_start(ctx, dt, nl, r, V, G, p3_all, g, st));
    // all m steps enqueued at once behind the replicated stop word: after a stop the
    // GEMVs are gated (Gate on the int64 mirror), the rest are tiny; one sync per cycle
    int64_t k = 0, chunk = m;
    const int64_t* stop64 = reinterpret_cast<const int64_t*>(st + 8);
    while (true) {
      if (k > 0) {
        DS_CUDA(cudaMemcpyAsync(h_st, st, 8 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        DS_CUDA(cudaStreamSynchronize(ctx->stream));
        DS_TRY(check_watchdog(S));
        if (h_st[GST_STOP] <= (double)k || k >= m) break;
      }
      const int64_t kend = std::min<int64_t>(m, k + chunk);
      for (; k < kend; ++k) {
        T* vk = V + k * ldv;
        T* w = V + (k + 1) * ldv;
        DS_TRY(gather_vec(vk));
        DS_TRY(gemv_launch<T>(ctx, gp, A, lda, full, w, static_cast<double*>(ws), EPI_STORE, nullptr, nullptr,
                              nullptr, Gate{stop64, k}));
        const int kc = (int)(k + 1);
        for (int ps = 0; ps < passes; ++ps) {
          const int off = ps == 0 ? GR_MD0 : GR_MD1;
          DS_TRY(ds_multidot_dev(ctx, dt, nl, V, ldv, kc, w, md));
          DS_TRY(publish(md, kc, off));
          DS_TRY(ds_cgs_update_shard(ctx, dt, nl, V, ldv, kc, w, G, S.gr + off, H + k * ldh, hsave, ps, md, st,
                                     k));
        }
        DS_TRY(publish(md, 3, GR_P3));
        DS_TRY(ds_gmres_shard_step(ctx, dt, nl, w, G, p3_all, H, Hraw, ldh, g, cs, sn, (int)k, est, st, tol, total,
                                   cap));
      }
      chunk = std::min<int64_t>(2 * chunk, 32);
    }
    DS_CUDA(cudaMemcpyAsync(h_st, st, 8 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA(cudaStreamSynchronize(ctx->stream));
    const int64_t inner = std::min<int64_t>((int64_t)h_st[GST_STOP], m);
    const bool happy = h_st[GST_BAD] != 0.0;
    {
      std::vector<double> e((size_t)std::max<int64_t>(inner, 1));
      if (inner > 0) {
        DS_CUDA(cudaMemcpyAsync(e.data(), est, inner * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        DS_CUDA(cudaStreamSynchronize(ctx->stream));
      }
      for (int64_t i = 0; i < inner; ++i) history.push_back(e[i]);
    }
    total += inner;
    DS_TRY(ds_gmres_lsq(ctx, dt, H, ldh, g, (int)inner, y, st));
    DS_CUDA(cudaMemcpyAsync(h_st, st, 8 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h_st[GST_STATUS] == (double)DS_ESINGULAR) {
      set_error("zero diagonal at row %lld", (long long)h_st[GST_RES]);
      info->error_index = (int64_t)h_st[GST_RES];
      return DS_ESINGULAR;
    }
    if (inner > 0) DS_TRY(ds_gemv_acc(ctx, dt, nl, inner, V, ldv, y, x));  // x += V y (krylov.py:167)
    double s2t = 0.0, nt = 0.0;
    DS_TRY(residual(&s2t, &nt));
    ++resid_evals;
    const double true_res = std::sqrt(s2t) / bnorm_plain;
    if (happy || history.back() <= tol || true_res <= tol) {
      history.back() = true_res;
      if (true_res <= tol || happy) {
        converged = true;
        if (happy) breakdown = DS_BREAKDOWN_HAPPY;
        break;
      }
    }
    if (total >= cap) {
      history.back() = true_res;
      break;
    }
    if (inner == m && true_res >= start_res * (1.0 - u)) {  // stagnation (krylov.py:177-180)
      history.back() = true_res;
      break;
    }
  }
  const int64_t hl = std::min<int64_t>((int64_t)history.size(), hist_cap);
  if (h_hist) std::copy(history.begin(), history.begin() + hl, h_hist);
  const int64_t cl = std::min<int64_t>((int64_t)cycles.size(), cycles_cap);
  if (h_cycles) std::copy(cycles.begin(), cycles.begin() + cl, h_cycles);
  info->iterations = total;
  info->history_len = hl;
  info->cycles_len = cl;
  info->final_relative_residual = history.back();
  info->converged = converged;
  info->breakdown = breakdown;
  info->residual_evals = resid_evals;
  info->kernel_launches = ctx->launches - launches0;
  return DS_OK;
}

// ---- 1-D block-cyclic LU (direct.py:50-84) ------------------------------------------
// Column blocks of width nb are dealt round-robin: shard q owns blocks q, q+G, ... stored
// contiguously in W (n rows, ld ldw).  Step k: the owner of block k broadcasts its factored
// panel (rows kb..n, its pivots and zero-pivot flags) into every peer's staging slot
// (parity k&1) and releases the broadcast flag; every shard applies the panel's row swaps to
// all its columns outside block k, the b-blocked TRSM of the U block row and the DMMA
// trailing update to its blocks right of k, then signals that it is done with the slot.
// Look-ahead: the owner of block k+1 updates that block first and factors it before its
// other step-k updates.  Two flag sets decouple the broadcast (one source per step) from the
// done signals (every shard), so the look-ahead owner can broadcast early.
size_t lu_slot_bytes(int64_t n, int64_t nb, size_t elem) {
  return round256((size_t)n * nb * elem) + round256((size_t)nb * 8) + round256((size_t)nb);
}

template <typename T>
int sh_lu_run(ShardLocal& S, ds_shardset* ss, T* W, int64_t ldw, int64_t nb, int64_t b, int64_t* h_piv, int* h_sing,
              HostBarrier* allocated) {
  ds_ctx* ctx = S.ctx;
  const int G = ss->G, q = S.rank;
  const int64_t n = ss->n;
  const int64_t nblocks = ceil_div(n, nb);
  const size_t slot = lu_slot_bytes(n, nb, sizeof(T));
  const int64_t nloc_blocks = nblocks > q ? ceil_div(nblocks - q, (int64_t)G) : 0;
  auto lcol = [&](int64_t k) { return (k / G) * nb; };                 // local column of (own) block k
  auto bw = [&](int64_t k) { return std::min<int64_t>(nb, n - k * nb); };
  const int64_t ncols = nloc_blocks > 0 ? lcol(q + (nloc_blocks - 1) * G) + bw(q + (nloc_blocks - 1) * G) : 0;
  // allocations (before any exchange, behind the host barrier of the local shards)
  void* ws = nullptr;
  int ast = ctx_workspace(ctx, (size_t)16 << 20, &ws);  // panel / laswp scratch of the shard kernels
  const size_t need = round256((size_t)n * 8) + round256((size_t)n) + 512;
  if (ast == DS_OK && need > S.sws_bytes) {
    if (S.sws) cudaFree(S.sws);
    S.sws = nullptr;
    S.sws_bytes = 0;
    if (cudaMalloc(&S.sws, need) == cudaSuccess)
      S.sws_bytes = need;
    else
      ast = DS_ENOMEM;
  }
  if (allocated) allocated->arrive_and_wait();
  if (ast != DS_OK) {
    ss->broken = true;
    return ast;
  }
  if (G > 1 && ss->xbytes < 2 * slot) {
    set_error("shard set staging buffer too small for the block-cyclic LU panels");
    return DS_EINVAL;
  }
  Carver cv{(char*)S.sws};
  int64_t* piv = cv.take<int64_t>((size_t)n * 8);
  int8_t* zero = cv.take<int8_t>((size_t)n);
  unsigned* ticket = cv.take<unsigned>(64);
  int* d_any = reinterpret_cast<int*>(ticket + 8);
  DS_CUDA(cudaMemsetAsync(zero, 0, (size_t)n, ctx->stream));
  DS_CUDA(cudaMemsetAsync(ticket, 0, 64, ctx->stream));
  DS_CUDA(cudaMemsetAsync(S.err, 0, kErrBytes, ctx->stream));
  const unsigned long long base = S.lu_epoch;
  const unsigned long long tmo = watchdog_ns();

  auto factor = [&](int64_t k) -> int {  // the owner's panel: rows kb..n of block k
    const int64_t kb = k * nb, w = bw(k);
    DS_TRY(lu_factor_impl<T>(ctx, n - kb, w, W + kb + lcol(k) * ldw, ldw, std::min<int64_t>(b, w), piv + kb,
                             zero + kb));
    sh_piv_offset_kernel<<<1, 256, 0, ctx->stream>>>(piv + kb, w, kb);
    count_launch(ctx);
    return DS_OK;
  };
  auto update = [&](int64_t k, const T* L, int64_t ldl, int64_t c0, int64_t c1) -> int {
    if (c1 <= c0) return DS_OK;
    const int64_t kb = k * nb, w = bw(k), cw = c1 - c0;
    for (int64_t ib = 0; ib < w; ib += b) {  // U block row, b-blocked (direct.py:80-81)
      const int64_t ibf = std::min<int64_t>(ib + b, w);
      T* U = W + (kb + ib) + c0 * ldw;
      DS_TRY(trsm_lower_unit_launch<T>(ctx, ibf - ib, cw, L + ib + ib * ldl, ldl, U, ldw, U, ldw));
      if (ibf < w)
        DS_TRY(gemm_launch<T>(ctx, w - ibf, cw, ibf - ib, -1.0, L + ibf + ib * ldl, ldl, U, ldw, 1.0,
                              W + (kb + ibf) + c0 * ldw, ldw, W + (kb + ibf) + c0 * ldw, ldw));
    }
    if (kb + w < n)  // trailing update (direct.py:82-83)
      DS_TRY(gemm_launch<T>(ctx, n - kb - w, cw, w, -1.0, L + w, ldl, W + kb + c0 * ldw, ldw, 1.0,
                            W + (kb + w) + c0 * ldw, ldw, W + (kb + w) + c0 * ldw, ldw));
    return DS_OK;
  };
  auto bcast = [&](int64_t k) -> int {  // owner: panel k into every peer's slot k&1
    if (G <= 1) return DS_OK;
    const int64_t kb = k * nb, w = bw(k);
    if (k >= 2) {  // slot k&1 held panel k-2: every peer finished step k-2
      sh_wait_set_kernel<<<1, 32, 0, ctx->stream>>>(S.flag, FLAG_DONE, G, q, -1, base + (unsigned long long)(k - 1),
                                                    S.err, tmo);
      count_launch(ctx);
    }
    const size_t so = (size_t)(k & 1) * slot;
    const size_t po = so + round256((size_t)n * nb * sizeof(T)), zo = po + round256((size_t)nb * 8);
    sh_bcast_panel_kernel<T><<<ctx->num_sms, kShT, 0, ctx->stream>>>(S.peers, W + kb + lcol(k) * ldw, ldw, n - kb, w,
                                                                      piv + kb, zero + kb, so, po, zo,
                                                                      base + (unsigned long long)(k + 1), ticket);
    count_launch(ctx);
    DS_CHECK_LAUNCH();
    return DS_OK;
  };

  if (nblocks > 0 && q == 0) DS_TRY(factor(0));
  for (int64_t k = 0; k < nblocks; ++k) {
    const int o = (int)(k % G);
    const int64_t kb = k * nb, w = bw(k);
    const T* L;
    int64_t ldl;
    if (q == o) {
      DS_TRY(bcast(k));
      L = W + kb + lcol(k) * ldw;
      ldl = ldw;
    } else {
      sh_wait_set_kernel<<<1, 32, 0, ctx->stream>>>(S.flag, FLAG_BCAST, G, q, o, base + (unsigned long long)(k + 1),
                                                    S.err, tmo);
      count_launch(ctx);
      const size_t so = (size_t)(k & 1) * slot;
      const size_t po = so + round256((size_t)n * nb * sizeof(T)), zo = po + round256((size_t)nb * 8);
      L = reinterpret_cast<const T*>(S.xbuf + so);
      ldl = n - kb;
      DS_CUDA(cudaMemcpyAsync(piv + kb, S.xbuf + po, (size_t)w * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      DS_CUDA(cudaMemcpyAsync(zero + kb, S.xbuf + zo, (size_t)w, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    // the panel's row swaps on every local column outside block k (full-row swaps, direct.py:68-70)
    if (q == o) {
      DS_TRY(laswp_range<T>(ctx, W, ldw, lcol(k), kb, kb + w, piv));
      DS_TRY(laswp_range<T>(ctx, W + (lcol(k) + w) * ldw, ldw, ncols - lcol(k) - w, kb, kb + w, piv));
    } else if (ncols > 0) {
      DS_TRY(laswp_range<T>(ctx, W, ldw, ncols, kb, kb + w, piv));
    }
    // local blocks right of k: from the first own block with index > k to the end
    int64_t kr = k + 1 + (((q - (int)((k + 1) % G)) % G + G) % G);  // first own block >= k+1
    if (kr < nblocks) {
      const int64_t c0 = lcol(kr);
      if (kr == k + 1) {  // look-ahead: this shard owns block k+1
        DS_TRY(update(k, L, ldl, c0, c0 + bw(kr)));
        DS_TRY(factor(k + 1));
        DS_TRY(update(k, L, ldl, c0 + bw(kr), ncols));
      } else {
        DS_TRY(update(k, L, ldl, c0, ncols));
      }
    }
    if (G > 1) {  // done with the slot of panel k
      sh_signal_set_kernel<<<1, 32, 0, ctx->stream>>>(S.peers, FLAG_DONE, base + (unsigned long long)(k + 1));
      count_launch(ctx);
    }
    DS_CHECK_LAUNCH();
  }
  DS_CUDA(cudaMemsetAsync(d_any, 0, sizeof(int), ctx->stream));
  sh_any_kernel<<<1, 256, 0, ctx->stream>>>(zero, n, d_any);
  count_launch(ctx);
  if (h_piv) DS_CUDA(cudaMemcpyAsync(h_piv, piv, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaMemcpyAsync(h_sing, d_any, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  DS_TRY(check_watchdog(S));
  S.lu_epoch = base + (unsigned long long)nblocks;
  return DS_OK;
}

// run fn(i) for every local shard: inline for one, one host thread per shard otherwise;
// the first failing shard's status and message are returned
template <typename F>
int for_each_local(ds_shardset* ss, F fn) {
  const int L = (int)ss->loc.size();
  if (L == 1) return fn(0);
  std::vector<int> st(L, DS_OK);
  std::vector<std::string> msg(L);
  std::vector<std::thread> th;
  for (int i = 0; i < L; ++i)
    th.emplace_back([&, i] {
      st[i] = fn(i);
      if (st[i] != DS_OK) msg[i] = ds_last_error();
    });
  for (auto& t : th) t.join();
  // a failed exchange (watchdog) explains the other shards' errors: report it first
  for (int pass = 0; pass < 2; ++pass)
    for (int i = 0; i < L; ++i)
      if (st[i] != DS_OK && (pass == 1 || st[i] == DS_ECUDA)) {
        set_error("%s", msg[i].c_str());
        return st[i];
      }
  return DS_OK;
}

// Every kernel a shard launches while peers may be spinning on an exchange is loaded up
// front: with lazy module loading (the CUDA 12 default) the first launch of a kernel
// loads its module and waits for the device — on a GPU shared by several shards that
// wait would include a peer's exchange kernel waiting for this very shard.
template <typename T>
void shard_kernel_list(std::vector<const void*>& f) {
  f.push_back((const void*)sh_publish_kernel<0>);
  f.push_back((const void*)sh_publish_kernel<1>);
  f.push_back((const void*)sh_publish_kernel<2>);
  f.push_back((const void*)sh_put_slice_kernel<T>);
  f.push_back((const void*)sh_cg_update_kernel<T>);
  f.push_back((const void*)sh_cg_finish_kernel<T>);
  f.push_back((const void*)sh_cg_reduce_pap_kernel<T>);
  f.push_back((const void*)sh_bcast_panel_kernel<T>);
  f.push_back((const void*)sh_parts_kernel<T>);
  f.push_back((const void*)sh_copy_block_kernel<T>);
}
int preload_kernels() {
  std::vector<const void*> f = {(const void*)sh_wait_kernel, (const void*)sh_signal_kernel,
                                (const void*)sh_publish2_kernel, (const void*)sh_cg_init_kernel,
                                (const void*)sh_publish_array_kernel, (const void*)sh_wait_set_kernel,
                                (const void*)sh_signal_set_kernel, (const void*)sh_piv_offset_kernel,
                                (const void*)sh_any_kernel};
  shard_kernel_list<double>(f);
  shard_kernel_list<float>(f);
  cudaFuncAttributes a;
  for (const void* p : f) DS_CUDA(cudaFuncGetAttributes(&a, p));
  DS_TRY(preload_sharded_kernels_blas());
  DS_TRY(preload_dense_kernels_blas());
  DS_TRY(preload_lu_kernels());
  return preload_sharded_kernels_dist();
}

int connect_peers(ds_shardset* ss, const std::vector<char*>& bases) {
  const Layout L = layout_of(ss);
  for (auto& S : ss->loc) {
    S.peers.G = ss->G;
    S.peers.rank = S.rank;
    for (int t = 0; t < ss->G; ++t) {
      char* b = bases[t];
      S.peers.flag[t] = reinterpret_cast<unsigned long long*>(b + L.flag);
      S.peers.rec[t] = reinterpret_cast<double*>(b + L.rec);
      S.peers.full[t] = b + L.full;
      S.peers.xbuf[t] = b + L.xbuf;
      S.peers.gr[t] = reinterpret_cast<double*>(b + L.gr);
    }
  }
  ss->connected = true;
  return DS_OK;
}

}  // namespace

extern "C" {

int ds_shardset_create(int nlocal, ds_ctx* const* ctxs, const int* ranks, int nshards, int dtype, int64_t n,
                       int64_t xbuf_bytes, ds_shardset** out) {
  if (nlocal < 1 || nshards < 1 || nshards > kMaxShards || nlocal > nshards || n < 1 || !ctxs || !ranks) {
    set_error("bad shard set: %d local of %d shards (max %d), n=%lld", nlocal, nshards, kMaxShards, (long long)n);
    return DS_EINVAL;
  }
  if (dtype != DS_F64 && dtype != DS_F32) {
    set_error("unsupported dtype code %d", dtype);
    return DS_EPREC;
  }
  auto* ss = new ds_shardset();
  ss->G = nshards;
  ss->n = n;
  ss->n_loc = ceil_div(n, nshards);
  ss->N = ss->n_loc * nshards;
  ss->elem = dtype_size(dtype);
  ss->xbytes = nshards > 1 ? (size_t)std::max<int64_t>(0, xbuf_bytes) : 0;
  const Layout L = layout_of(ss);
  for (int i = 0; i < nlocal; ++i) {
    int pst = ctx_begin(ctxs[i]);
    if (pst == DS_OK) pst = preload_kernels();  // per device
    if (pst != DS_OK) {
      for (auto& s2 : ss->loc) cudaFree(s2.region);
      delete ss;
      return pst;
    }
  }
  for (int i = 0; i < nlocal; ++i) {
    ShardLocal S;
    S.ctx = ctxs[i];
    S.rank = ranks[i];
    if (S.rank < 0 || S.rank >= nshards) {
      set_error("bad shard rank %d", S.rank);
      delete ss;
      return DS_EINVAL;
    }
    int st = ctx_begin(S.ctx);
    if (st != DS_OK) {
      delete ss;
      return st;
    }
    // plain cudaMalloc: exportable through CUDA IPC and mappable by peers
    cudaError_t e = cudaMalloc(&S.region, L.total);
    if (e != cudaSuccess) {
      set_error("shard exchange region (%zu bytes): %s", L.total, cudaGetErrorString(e));
      for (auto& s2 : ss->loc) cudaFree(s2.region);
      delete ss;
      return DS_ENOMEM;
    }
    cudaMemset(S.region, 0, L.total);
    S.region_bytes = L.total;
    bind_region(S, L, S.region);
    ss->loc.push_back(std::move(S));
  }
  cudaDeviceSynchronize();
  *out = ss;
  return DS_OK;
}

int ds_shardset_info(const ds_shardset* ss, int64_t* n_loc, int64_t* N) {
  if (!ss) {
    set_error("null shard set");
    return DS_EINVAL;
  }
  *n_loc = ss->n_loc;
  *N = ss->N;
  return DS_OK;
}

int ds_shardset_connect_local(ds_shardset* ss) {
  // every shard is in this process: peer pointers are the regions themselves
  if ((int)ss->loc.size() != ss->G) {
    set_error("connect_local needs all %d shards in this process", ss->G);
    return DS_EINVAL;
  }
  std::vector<char*> bases(ss->G, nullptr);
  for (auto& S : ss->loc) bases[S.rank] = S.region;
  for (auto& S : ss->loc) {
    DS_TRY(ctx_begin(S.ctx));
    for (auto& P : ss->loc) {
      if (P.ctx->device == S.ctx->device) continue;
      int can = 0;
      DS_CUDA(cudaDeviceCanAccessPeer(&can, S.ctx->device, P.ctx->device));
      if (!can) {
        set_error("device %d cannot access peer device %d (no P2P path)", S.ctx->device, P.ctx->device);
        return DS_ECUDA;
      }
      const cudaError_t e = cudaDeviceEnablePeerAccess(P.ctx->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) DS_CUDA(e);
      cudaGetLastError();
    }
  }
  return connect_peers(ss, bases);
}

int ds_shardset_ipc_handle(ds_shardset* ss, unsigned char* h_out) {
  if (ss->loc.size() != 1) {
    set_error("IPC export is for one local shard per process");
    return DS_EINVAL;
  }
  DS_TRY(ctx_begin(ss->loc[0].ctx));
  cudaIpcMemHandle_t h;
  DS_CUDA(cudaIpcGetMemHandle(&h, ss->loc[0].region));
  static_assert(sizeof(cudaIpcMemHandle_t) == DS_SHARD_HANDLE_BYTES, "IPC handle size");
  memcpy(h_out, &h, sizeof h);
  return DS_OK;
}

int ds_shardset_connect_ipc(ds_shardset* ss, const unsigned char* h_all) {
  if (ss->loc.size() != 1) {
    set_error("IPC connect is for one local shard per process");
    return DS_EINVAL;
  }
  ShardLocal& S = ss->loc[0];
  DS_TRY(ctx_begin(S.ctx));
  std::vector<char*> bases(ss->G, nullptr);
  for (int t = 0; t < ss->G; ++t) {
    if (t == S.rank) {
      bases[t] = S.region;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, h_all + (size_t)t * DS_SHARD_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    DS_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    S.opened.push_back(p);
    bases[t] = (char*)p;
  }
  return connect_peers(ss, bases);
}

int ds_shardset_destroy(ds_shardset* ss) {
  if (!ss) return DS_OK;
  for (auto& S : ss->loc) {
    if (ctx_begin(S.ctx) != DS_OK) continue;
    cudaStreamSynchronize(S.ctx->stream);
    for (void* p : S.opened) cudaIpcCloseMemHandle(p);
    if (S.region) cudaFree(S.region);
    if (S.sws) cudaFree(S.sws);
  }
  delete ss;
  return DS_OK;
}

int ds_shardset_gather(ds_shardset* ss, int dtype, const void* const* d_loc, void* h_out) {
  if (!ss || !ss->connected) {
    set_error("shard set is not connected");
    return DS_EINVAL;
  }
  if (dtype_size(dtype) != ss->elem) {
    set_error("dtype does not match the shard set");
    return DS_EPREC;
  }
  const int st = for_each_local(ss, [&](int i) -> int {
    ShardLocal& S = ss->loc[i];
    DS_ENTER(S.ctx);
    DS_CUDA(cudaMemsetAsync(S.err, 0, kErrBytes, S.ctx->stream));
    DS_DISPATCH(dtype, T, {
      sh_put_slice_kernel<T><<<vgrid(S.ctx, ss->n_loc), kShT, 0, S.ctx->stream>>>(S.peers, ss->n_loc,
                                                                                  (const T*)d_loc[i]);
      count_launch(S.ctx);
      DS_CHECK_LAUNCH();
    });
    DS_TRY(sh_barrier(S, ss));
    if (i == 0)
      DS_CUDA(cudaMemcpyAsync(h_out, S.full, (size_t)ss->n * ss->elem, cudaMemcpyDeviceToHost, S.ctx->stream));
    DS_TRY(sh_barrier(S, ss));  // nobody overwrites full before the copy finished
    DS_CUDA(cudaStreamSynchronize(S.ctx->stream));
    return check_watchdog(S);
  });
  if (st == DS_ECUDA) ss->broken = true;
  return st;
}

int ds_lu_block_cyclic(ds_shardset* ss, int dtype, void* const* d_W, int64_t ldw, int64_t nb, int64_t b,
                       int64_t* h_piv, int32_t* h_singular) {
  if (!ss || !ss->connected) {
    set_error("shard set is not connected");
    return DS_EINVAL;
  }
  if (ss->broken) {
    set_error("shard set is unusable after an earlier failed exchange; create a new one");
    return DS_ECUDA;
  }
  if (dtype_size(dtype) != ss->elem) {
    set_error("dtype does not match the shard set");
    return DS_EPREC;
  }
  if (nb < 1 || b < 1 || ldw < ss->n) {
    set_error("invalid block-cyclic LU configuration (nb=%lld, b=%lld, ldw=%lld)", (long long)nb, (long long)b,
              (long long)ldw);
    return DS_EINVAL;
  }
  const int L = (int)ss->loc.size();
  std::vector<int> sing(L, 0);
  HostBarrier allocated(L);
  const int st = for_each_local(ss, [&](int i) -> int {
    ShardLocal& S = ss->loc[i];
    const int e = ctx_begin(S.ctx);
    if (e != DS_OK) {
      allocated.arrive_and_wait();
      return e;
    }
    std::lock_guard<std::recursive_mutex> guard(S.ctx->mu);
    if (dtype == DS_F64)
      return sh_lu_run<double>(S, ss, (double*)d_W[i], ldw, nb, b, i == 0 ? h_piv : nullptr, &sing[i], &allocated);
    return sh_lu_run<float>(S, ss, (float*)d_W[i], ldw, nb, b, i == 0 ? h_piv : nullptr, &sing[i], &allocated);
  });
  if (h_singular) *h_singular = sing.empty() ? 0 : sing[0];
  if (st == DS_ECUDA) ss->broken = true;
  return st;
}

int ds_gmres_sharded(ds_shardset* ss, int dtype, void* const* d_A, int64_t lda, const void* const* d_b,
                     const void* const* d_x0, void* const* d_x, double tol, int64_t max_it, int64_t restart_m,
                     int orth, double* h_hist, int64_t hist_cap, int64_t* h_cycles, int64_t cycles_cap,
                     ds_solve_info* info) {
  if (!ss || !ss->connected) {
    set_error("shard set is not connected");
    return DS_EINVAL;
  }
  if (ss->broken) {
    set_error("shard set is unusable after an earlier failed exchange; create a new one");
    return DS_ECUDA;
  }
  if (dtype_size(dtype) != ss->elem) {
    set_error("dtype does not match the shard set");
    return DS_EPREC;
  }
  if (!(tol > 0) || max_it < 1 || restart_m < 1 || lda < ss->n_loc ||
      (orth != DS_ORTH_MODIFIED && orth != DS_ORTH_CLASSICAL)) {
    set_error("invalid sharded GMRES configuration");
    return DS_EINVAL;
  }
  if (ss->G == 1) {
    // one shard holds every row: there is nothing to exchange, and the single-GPU solver's
    // fused step (GEMV + one-cluster orthogonalisation chained by PDL) is the same
    // arithmetic with fewer launches than the shard kernels
    return ds_gmres(ss->loc[0].ctx, dtype, ss->n, d_A[0], lda, d_b[0], d_x0[0], d_x[0], tol, max_it, restart_m,
                    orth, h_hist, hist_cap, h_cycles, cycles_cap, nullptr, nullptr, info);
  }
  if (restart_m > 63) {  // the shard kernels keep one Hessenberg column (<= 64 entries) in shared memory
    set_error("restart_m = %lld exceeds the sharded GMRES limit of 63", (long long)restart_m);
    return DS_EINVAL;
  }
  const int L = (int)ss->loc.size();
  std::vector<ds_solve_info> infos(L);
  HostBarrier allocated(L);
  const int st = for_each_local(ss, [&](int i) -> int {
    ShardLocal& S = ss->loc[i];
    const int e = ctx_begin(S.ctx);
    if (e != DS_OK) {
      allocated.arrive_and_wait();
      return e;
    }
    std::lock_guard<std::recursive_mutex> guard(S.ctx->mu);
    infos[i] = ds_solve_info{};
    infos[i].error_index = -1;
    const bool first = i == 0;
    if (dtype == DS_F64)
      return sh_gmres_run<double>(S, ss, (const double*)d_A[i], lda, (const double*)d_b[i], (const double*)d_x0[i],
                                  (double*)d_x[i], tol, max_it, restart_m, orth, first ? h_hist : nullptr, hist_cap,
                                  first ? h_cycles : nullptr, cycles_cap, &infos[i], &allocated);
    return sh_gmres_run<float>(S, ss, (const float*)d_A[i], lda, (const float*)d_b[i], (const float*)d_x0[i],
                               (float*)d_x[i], tol, max_it, restart_m, orth, first ? h_hist : nullptr, hist_cap,
                               first ? h_cycles : nullptr, cycles_cap, &infos[i], &allocated);
  });
  *info = infos[0];
  if (st == DS_ECUDA) ss->broken = true;
  return st;
}

int ds_cg_sharded(ds_shardset* ss, int dtype, void* const* d_A, int64_t lda, const void* const* d_b,
                  const void* const* d_x0, void* const* d_x, double tol, int64_t max_it, int check_sym,
                  double* h_hist, int64_t hist_cap, ds_solve_info* info) {
  if (!ss || !ss->connected) {
    set_error("shard set is not connected");
    return DS_EINVAL;
  }
  if (ss->broken) {
    set_error("shard set is unusable after an earlier failed exchange; create a new one");
    return DS_ECUDA;
  }
  if (dtype_size(dtype) != ss->elem) {
    set_error("dtype does not match the shard set");
    return DS_EPREC;
  }
  if (!(tol > 0) || max_it < 1 || lda < ss->n_loc) {
    set_error("invalid sharded CG configuration");
    return DS_EINVAL;
  }
  const int L = (int)ss->loc.size();
  std::vector<ds_solve_info> infos(L);
  HostBarrier allocated(L);
  const int st = for_each_local(ss, [&](int i) -> int {
    ShardLocal& S = ss->loc[i];
    const int e = ctx_begin(S.ctx);
    if (e != DS_OK) {
      allocated.arrive_and_wait();
      return e;
    }
    std::lock_guard<std::recursive_mutex> guard(S.ctx->mu);
    infos[i] = ds_solve_info{};
    infos[i].error_index = -1;
    if (dtype == DS_F64)
      return sh_cg_run<double>(S, ss, (const double*)d_A[i], lda, (const double*)d_b[i], (const double*)d_x0[i],
                               (double*)d_x[i], tol, max_it, check_sym, i == 0 ? h_hist : nullptr, hist_cap,
                               &infos[i], &allocated);
    return sh_cg_run<float>(S, ss, (const float*)d_A[i], lda, (const float*)d_b[i], (const float*)d_x0[i],
                            (float*)d_x[i], tol, max_it, check_sym, i == 0 ? h_hist : nullptr, hist_cap, &infos[i],
                            &allocated);
  });
  *info = infos[0];
  if (st == DS_ECUDA) ss->broken = true;
  return st;
}

}  // extern "C"
