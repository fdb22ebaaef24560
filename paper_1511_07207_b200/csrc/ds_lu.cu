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
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <vector>

#include <map>
#include <mutex>
#include <tuple>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

namespace ds {

// 128 threads: a panel CTA (<= 32 regs/thread) then fits beside two trailing-GEMM
// CTAs (240 regs x 128 threads each) on one SM, so the look-ahead panel running on
// the side stream does not evict half of the GEMM's occupancy.
constexpr int kPanelThreads = 128;
// register-row panel kernel: TPR threads per row (2 or 4), <= kPanelRegThreads threads
constexpr int kPanelRegThreads = 512;

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
  unsigned* bar;       // grid barrier counter (zeroed before each launch)
  double* cand_v;      // [2][grid]  candidate |value| per CTA, double-buffered by column parity
  int64_t* cand_i;     // [2][grid]  candidate row per CTA
  void* cand_row;      // [2][grid][kPanelMaxW] the candidate rows' panel values (smem kernel)
  void* diag_row;      // [2][kPanelMaxW] row i's values before the swap (smem kernel)
  void* rowP;          // global kernel: pivot row
  void* rowI;          // global kernel: row i before the swap
  int per;             // rows per CTA
  int ldt;             // smem tile leading dimension
  uint64_t* ll_hdr;    // smem kernel: [2][grid][kHdrWords] LL candidate headers
  uint64_t* ll_row;    // smem kernel: [2][grid][kPanelMaxW * words/value] LL candidate rows
  uint64_t* ll_diag;   // smem kernel: [2][kPanelMaxW * words/value] LL row i
  unsigned seq;        // per-context panel launch counter (LL epochs)
  int backoff;         // poller kernel: __nanosleep between failed LL polls (0 = spin)
  unsigned long long* trace;  // optional [grid][ncol][4] %globaltimer stamps (DENSOLVE_PANEL_TRACE)
};


constexpr int kPanelMaxW = 64;

// Block-wide first-max argmax (np.argmax(np.abs(.)) semantics); result in thread 0.
__device__ __forceinline__ void block_argmax(double& bv, int64_t& bi, double* sv, int64_t* si) {
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
  }
}

// Every thread loads at most a few of the G published candidates (one L2 round
// trip for G <= blockDim.x), then a block-wide first-max reduction in a fixed
// order => the identical pivot in every CTA; returned in s_piv.
__device__ __forceinline__ void reduce_candidates(const PanelArgs& a, int par, int64_t i,
                                                  int64_t* s_piv, double* sv, int64_t* si) {
  const unsigned G = gridDim.x;
  double bv = -1.0;
  int64_t bi = INT64_MAX;
  for (unsigned b0 = threadIdx.x; b0 < G; b0 += 2 * blockDim.x) {
    const unsigned b1 = b0 + blockDim.x;  // both loads issued before either compare
    const double v0 = __ldcg(a.cand_v + par * G + b0);
    const int64_t i0 = __ldcg(a.cand_i + par * G + b0);
    double v1 = -1.0;
    int64_t i1 = INT64_MAX;
    if (b1 < G) {
      v1 = __ldcg(a.cand_v + par * G + b1);
      i1 = __ldcg(a.cand_i + par * G + b1);
    }
    if (piv_better(v0, i0, bv, bi)) {
      bv = v0;
      bi = i0;
    }
    if (piv_better(v1, i1, bv, bi)) {
      bv = v1;
      bi = i1;
    }
  }
  block_argmax(bv, bi, sv, si);
  if (threadIdx.x == 0) *s_piv = bi == INT64_MAX ? i : bi;
  __syncthreads();
}

// ---- LL exchange words: 32 data bits + a 32-bit epoch flag in one aligned 8-byte
// word.  An 8-byte store is single-copy atomic, so a reader that sees the
// expected flag also sees that store's data: no fence, no atomic, no separate
// barrier.  Epochs are unique per (panel launch, column) and the buffers are
// double-buffered by column parity (a CTA can only be one column ahead of the
// slowest reader).
__device__ __forceinline__ void ll_store(uint64_t* p, uint32_t data, uint32_t flag) {
  const uint64_t w = ((uint64_t)flag << 32) | data;
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;\n" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ uint64_t ll_load(const uint64_t* p) {
  uint64_t w;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ bool ll_ok(uint64_t w, uint32_t flag) { return (uint32_t)(w >> 32) == flag; }

template <typename T>
struct LLVal;  // words per value
template <>
struct LLVal<double> {
  static constexpr int W = 2;
  __device__ static void put(uint64_t* p, double v, uint32_t f) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    ll_store(p, (uint32_t)b, f);
    ll_store(p + 1, (uint32_t)(b >> 32), f);
  }
  __device__ static double get(const uint64_t* w) {
    return __longlong_as_double((long long)((w[0] & 0xffffffffull) | (w[1] << 32)));
  }
};
template <>
struct LLVal<float> {
  static constexpr int W = 1;
  __device__ static void put(uint64_t* p, float v, uint32_t f) { ll_store(p, __float_as_uint(v), f); }
  __device__ static float get(const uint64_t* w) { return __uint_as_float((uint32_t)w[0]); }
};

// First-max argmax over the CTA: keys are the IEEE bits of |v| (monotone for
// v >= 0, NaN canonicalised above +inf so it wins like np.argmax), reduced with
// two redux.sync max passes; ties go to the lowest row (a redux.sync min over the
// top lanes); the warp records are then combined by every thread in the same order
// (one barrier).  `none` candidates carry key 0 and row INT64_MAX.
__device__ __forceinline__ unsigned long long piv_key(double v) {
  return v != v ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(v);
}
__device__ __forceinline__ void cta_argmax_key(unsigned long long& key, int64_t& idx,
                                               unsigned long long* wk, int64_t* wi) {
  const unsigned hi = (unsigned)(key >> 32);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned lo = hi == mhi ? (unsigned)key : 0u;
  const unsigned mlo = __reduce_max_sync(0xffffffffu, lo);
  const bool top = hi == mhi && (unsigned)key == mlo;
  // rows < 2^31 - 1; INT64_MAX (none) maps to 0xffffffff
  const unsigned widx = __reduce_min_sync(0xffffffffu, top ? (unsigned)min(idx, (int64_t)0xffffffff) : 0xffffffffu);
  const unsigned long long wkey = ((unsigned long long)mhi << 32) | mlo;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    wk[wid] = wkey;
    wi[wid] = widx == 0xffffffffu ? INT64_MAX : (int64_t)widx;
  }
  __syncthreads();  // the poller-warp panel reaches it with every warp at the same code location
  // every warp combines the nw warp records itself (lane w reads record w): the same
  // reduction in every warp, no second barrier
  const int nw = (int)(blockDim.x >> 5);
  const unsigned long long k2 = lane < nw ? wk[lane] : 0ull;
  const int64_t i2 = lane < nw ? wi[lane] : INT64_MAX;
  const unsigned h2 = (unsigned)(k2 >> 32);
  const unsigned mh2 = __reduce_max_sync(0xffffffffu, h2);
  const unsigned l2 = h2 == mh2 ? (unsigned)k2 : 0u;
  const unsigned ml2 = __reduce_max_sync(0xffffffffu, l2);
  const bool top2 = h2 == mh2 && (unsigned)k2 == ml2;
  const unsigned mi2 = __reduce_min_sync(0xffffffffu, top2 ? (unsigned)min(i2, (int64_t)0xffffffff) : 0xffffffffu);
  key = ((unsigned long long)mh2 << 32) | ml2;
  idx = mi2 == 0xffffffffu ? INT64_MAX : (int64_t)mi2;
}

// Panel factorization, one row per thread held in REGISTERS (rows <= 256 per CTA,
// i.e. m <= 148 * 256).  The register row is kept rotated: y[k] is the current
// value of panel column c + k, so every column runs the same straight-line code
// (static register indices): the update touches y[1..63], then column c retires
// into the shared-memory array Ls (the final L / U values of columns < c) and the
// row shifts by one.  Per column every CTA publishes, as LL words, its local
// candidate header (|v|, row; one 128-byte line per CTA) and the candidate row

// Forward-progress watchdog of the panel kernels' LL spin loops.  The exchange needs every
// CTA of the panel grid resident at once; the host asserts that with the occupancy
// calculator before each plain launch (panel_launch) and otherwise takes the cooperative
// kernel.  Should residency still fail (another context, MPS partitioning), a poll would
// spin forever: after 10 s of wall time (%globaltimer) the kernel traps instead, which the
// host sees as a CUDA error (DS_ECUDA -> RuntimeError), not a hung device.
struct SpinGuard {
  unsigned n = 0;
  unsigned long long t0 = 0;
  __device__ __forceinline__ void tick() {
    if ((++n & 4095u) == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t0 == 0)
        t0 = now;
      else if (now - t0 > 10000000000ull)
        __trap();
    }
  }
};
// (written by the owning thread); the owner of row i publishes row i.  Every CTA
// polls the G headers (the only grid-wide synchronisation), reduces them in a
// fixed order (the same first-max pivot everywhere), polls the winner's row and
// row i, and every thread swaps / scales / rank-1-updates its own row (NumPy
// rounding: bitwise the reference).
constexpr int kHdrWords = 16;  // |v| (2 words), row (1 word), padding to a 128-byte line
template <typename T, int TPR>
__global__ void __launch_bounds__(kPanelRegThreads, 1) lu_panel_smem_kernel(T* __restrict__ W, PanelArgs a) {
  constexpr int PW = kPanelMaxW / TPR;  // panel columns per thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Ls = reinterpret_cast<T*>(smem_raw);  // [ncol][ldt]: retired columns
  __shared__ unsigned long long wk[2][kPanelRegThreads / 32];
  __shared__ int64_t wi[2][kPanelRegThreads / 32];
  __shared__ __align__(16) T stage[2][kPanelMaxW];  // candidate row / diagonal row, columns >= c
  __shared__ __align__(16) T prow[kPanelMaxW];       // winner row, column order
  __shared__ __align__(16) T drow[kPanelMaxW];       // row i, column order
  __shared__ __align__(16) T prs[kPanelMaxW + 2];    // prs[k] = prow[c + k] (0 past the panel)
  __shared__ __align__(16) T drs[kPanelMaxW + 2];    // drs[k] = drow[c + k]
  constexpr int VW = LLVal<T>::W;
  const unsigned G = gridDim.x;
  const int per = a.per, ldt = a.ldt;
  const int64_t my_lo = a.kb + (int64_t)blockIdx.x * per;
  const int64_t my_hi = min(a.n, my_lo + per);
  const int nr = (int)(my_hi - my_lo);
  const int ncol = (int)(a.bf - a.kb);
  uint64_t* hdr = a.ll_hdr;    // [2][G][kHdrWords]
  uint64_t* rows = a.ll_row;   // [2][G][kPanelMaxW * VW]
  uint64_t* diag = a.ll_diag;  // [2][kPanelMaxW * VW]
  const int RW = kPanelMaxW * VW;
  const int t = threadIdx.x, nt = blockDim.x;
  const int r = t / TPR, q = t % TPR;  // my row, my column slice [q * PW, (q + 1) * PW)
  const bool mine = r < nr;
  const bool lead = mine && q == 0;  // holds the current column c in y[0]
  const int64_t g = my_lo + r;
  const int lead_lane = (t & 31) & ~(TPR - 1);

  // y[k] = current value of panel column c + q * PW + k of my row (rotated view)
  T y[PW];
#pragma unroll
  for (int k = 0; k < PW; ++k) {
    const int j = q * PW + k;
    y[k] = (mine && j < ncol) ? W[g + (a.kb + j) * a.ld] : T(0);
  }

  auto publish_header = [&](int cc, unsigned long long bk, int64_t bi) {
    if (t == 0) {
      const uint32_t ep = a.seq * 128u + (uint32_t)cc + 1u;
      uint64_t* h = hdr + ((size_t)(cc & 1) * G + blockIdx.x) * kHdrWords;
      ll_store(h, (uint32_t)bk, ep);
      ll_store(h + 1, (uint32_t)(bk >> 32), ep);
      ll_store(h + 2, bi == INT64_MAX ? 0xffffffffu : (uint32_t)bi, ep);
    }
  };
  // candidate row and row kb + cc: the owners stage their register slices (columns >= cc)
  auto publish_rows = [&](int cc, int64_t bi) {
    const int par = cc & 1;
    const uint32_t ep = a.seq * 128u + (uint32_t)cc + 1u;
    const int64_t ii = a.kb + cc;
    if (mine && g == bi) {
#pragma unroll
      for (int k = 0; k < PW; ++k) stage[0][q * PW + k] = y[k];
    }
    if (mine && g == ii) {
#pragma unroll
      for (int k = 0; k < PW; ++k) stage[1][q * PW + k] = y[k];
    }
    __syncthreads();
    if (G == 1) return;  // a single CTA reads its candidate straight from shared memory
    for (int j = t; j < ncol; j += nt) {
      if (bi != INT64_MAX) {
        const T v = j < cc ? Ls[j * ldt + (int)(bi - my_lo)] : stage[0][j - cc];
        LLVal<T>::put(rows + ((size_t)par * G + blockIdx.x) * RW + j * VW, v, ep);
      }
      if (ii >= my_lo && ii < my_hi) {
        const T v = j < cc ? Ls[j * ldt + (int)(ii - my_lo)] : stage[1][j - cc];
        LLVal<T>::put(diag + (size_t)par * RW + j * VW, v, ep);
      }
    }
  };

  unsigned long long cand_k;  // this CTA's candidate of the current column
  int64_t cand_i;
  {
    unsigned long long bk = lead ? piv_key(fabs((double)y[0])) : 0ull;
    int64_t bi = lead ? g : INT64_MAX;
    cta_argmax_key(bk, bi, wk[0], wi[0]);
    if (G > 1) publish_header(0, bk, bi);
    publish_rows(0, bi);
    cand_k = bk;
    cand_i = bi;
  }
  for (int c = 0; c < ncol; ++c) {
    const int64_t i = a.kb + c;
    const int par = c & 1;
    const uint32_t ep = a.seq * 128u + (uint32_t)c + 1u;
    const long long t_c = clock64();
    // ---- poll the G headers, reduce (ties -> lowest row)
    unsigned long long gk = 0ull;
    int64_t gi = INT64_MAX;
    for (int b = t; G > 1 && b < (int)G; b += nt) {
      const uint64_t* h = hdr + ((size_t)par * G + b) * kHdrWords;
      uint64_t x0, x1, x2;
      SpinGuard sg;
      do {
        x0 = ll_load(h);
        x1 = ll_load(h + 1);
        x2 = ll_load(h + 2);
        sg.tick();
      } while (!(ll_ok(x0, ep) && ll_ok(x1, ep) && ll_ok(x2, ep)));
      const unsigned long long k2 = (x0 & 0xffffffffull) | (x1 << 32);
      const int64_t i2 = (uint32_t)x2 == 0xffffffffu ? INT64_MAX : (int64_t)(uint32_t)x2;
      if (k2 > gk || (k2 == gk && i2 < gi)) {
        gk = k2;
        gi = i2;
      }
    }
    const long long t_d = clock64();
    if (G > 1) {
      cta_argmax_key(gk, gi, wk[1], wi[1]);
    } else {  // one CTA: its own candidate is the pivot
      gk = cand_k;
      gi = cand_i;
    }
    const long long t_e = clock64();
    const int64_t p = gi == INT64_MAX ? i : gi;
    const int win = gi == INT64_MAX ? -1 : (int)((gi - a.kb) / per);
    // ---- the winner's row and row i (LL polls), in column order and rotated by c
    {
      const uint64_t* pr = rows + ((size_t)par * G + (win < 0 ? 0 : win)) * RW;
      const uint64_t* dr = diag + (size_t)par * RW;
      for (int j = t; j < c + kPanelMaxW + 2; j += nt) {
        if (j < ncol && G == 1) {  // single CTA: rows from shared memory (published by publish_rows)
          const int64_t pi_ = gi == INT64_MAX ? i : gi;
          const T pv = j < c ? Ls[j * ldt + (int)(pi_ - my_lo)] : stage[0][j - c];
          const T dv = j < c ? Ls[j * ldt + (int)(i - my_lo)] : stage[1][j - c];
          drow[j] = dv;
          prow[j] = gi == INT64_MAX ? dv : pv;
          if (j >= c) {
            drs[j - c] = dv;
            prs[j - c] = prow[j];
          }
        } else if (j < ncol) {
          uint64_t pw[VW], dw[VW];
          SpinGuard sg;
          while (true) {
            sg.tick();
            bool ok = true;
#pragma unroll
            for (int qq = 0; qq < VW; ++qq) {
              pw[qq] = win < 0 ? ((uint64_t)ep << 32) : ll_load(pr + j * VW + qq);
              dw[qq] = ll_load(dr + j * VW + qq);
              ok = ok && ll_ok(pw[qq], ep) && ll_ok(dw[qq], ep);
            }
            if (ok) break;
          }
          const T dv = LLVal<T>::get(dw);
          const T pv = win < 0 ? dv : LLVal<T>::get(pw);
          drow[j] = dv;
          prow[j] = pv;
          if (j >= c) {
            drs[j - c] = dv;
            prs[j - c] = pv;
          }
        } else if (j >= c) {
          drs[j - c] = T(0);
          prs[j - c] = T(0);
        }
      }
    }
    if (blockIdx.x == 0 && t == 0) a.piv[i] = p;  // piv[i] = v (direct.py:67)
    __syncthreads();
    const long long t_f = clock64();
    const T aii = prow[c];
    const bool zero = aii == T(0);
    long long t_f1 = 0, t_f2 = 0, t_f3 = 0;
    if (zero && blockIdx.x == 0 && t == 0) a.zero_cols[i] = 1;  // direct.py:71-74
    // retired columns j < c of rows i and p: one column per thread
    if (p != i)
      for (int j = t; j < c; j += nt) {
        if (i >= my_lo && i < my_hi) Ls[j * ldt + (int)(i - my_lo)] = prow[j];
        if (p >= my_lo && p < my_hi) Ls[j * ldt + (int)(p - my_lo)] = drow[j];
      }
    // ---- swap (direct.py:68-70, restricted to the panel)
    if (mine && p != i && (g == i || g == p)) {
#pragma unroll
      for (int k = 0; k < PW; ++k) y[k] = g == i ? prs[q * PW + k] : drs[q * PW + k];
    }
    // ---- reciprocal scale (the lead thread) and the update of column c + 1 first
    const bool act = mine && g > i && !zero;
    T l = T(0);
    if (lead && act) {
      l = mul_rn(div_rn(T(1), aii), y[0]);
      y[0] = l;
      if (PW > 1) y[1] = sub_rn(y[1], mul_rn(l, prs[1]));
    }
    l = __shfl_sync(0xffffffffu, l, lead_lane);
    if (lead) Ls[c * ldt + r] = y[0];  // retire column c
    if (a.trace) t_f1 = clock64();
    unsigned long long bk = 0ull;
    int64_t bi = INT64_MAX;
    if (c + 1 < ncol) {
      // next column's candidate (rows >= i + 1): column c + 1 is y[1] of the lead (PW > 1)
      const T nx = PW > 1 ? y[1 % PW] : T(0);
      if (lead && g > i) {
        bk = piv_key(fabs((double)nx));
        bi = g;
      }
    }
    if (PW == 1) {  // TPR == 64 is not used; keep the generic path well-defined
      bk = 0ull;
      bi = INT64_MAX;
    }
    if (c + 1 < ncol) {
      cta_argmax_key(bk, bi, wk[0], wi[0]);
      if (G > 1) publish_header(c + 1, bk, bi);  // the exchange of column c + 1 starts here
      cand_k = bk;
      cand_i = bi;
    }
    if (a.trace) t_f2 = clock64();
    // ---- rest of the rank-1 update of my slice (direct.py:75-79), then rotate by one
    if (act) {
#pragma unroll
      for (int k = 0; k < PW; ++k) {
        const int j = q * PW + k;
        if (j >= 2) y[k] = sub_rn(y[k], mul_rn(l, prs[j]));
      }
    }
    {
      const T carry = __shfl_down_sync(0xffffffffu, y[0], 1);
#pragma unroll
      for (int k = 0; k + 1 < PW; ++k) y[k] = y[k + 1];
      y[PW - 1] = q == TPR - 1 ? T(0) : carry;
    }
    if (a.trace) t_f3 = clock64();
    if (c + 1 < ncol) publish_rows(c + 1, bi);
    if (a.trace && t == 0) {
      const long long t_g = clock64();
      unsigned long long* tr = a.trace + (size_t)blockIdx.x * 8;
      tr[2] += t_d - t_c;  // header poll
      tr[3] += t_e - t_d;  // argmax of the headers
      tr[4] += t_f - t_e;  // row poll + barrier
      tr[0] += t_f1 - t_f;  // swap, scale
      tr[1] += t_f2 - t_f1;  // next column's CTA argmax + header publish
      tr[5] += t_f3 - t_f2;  // rank-1 update, rotate
      tr[6] += t_g - t_f3;   // publish rows
    }
  }
  __syncthreads();
  for (int idx = t; idx < ncol * nr; idx += nt) {
    const int j = idx / nr, rr = idx % nr;
    W[(my_lo + rr) + (a.kb + j) * a.ld] = Ls[j * ldt + rr];
  }
}

// Poller-warp panel (default for <= 224 rows per CTA): warp 0 of every CTA is a
// dedicated exchange warp with no rows; warps 1..7 hold one row per thread (the
// whole 64-column row rotated in registers).  Per column the row warps meet
// ONCE (the CTA argmax of the next column's candidate); right after it the
// candidate's owner publishes the header (signed value + row) and the candidate
// row and row i+1 as LL words, BEFORE the rank-1 update of the column: the rows
// go out with that update still pending, and the poller applies it to the two
// received rows (same mul/sub, same order: bitwise what the owner would have
// computed).  So the G-wide exchange latency overlaps the update.  The poller
// polls the headers, reduces them with warp REDUX, computes the reciprocal of
// the pivot while the row poll is in flight, fills CTA-shared, column-parity
// double-buffered row copies and hands them to the row warps through an
// mbarrier.  Same arithmetic and pivots as lu_panel_smem_kernel (bitwise the
// reference, direct.py:59-79).
__device__ __forceinline__ void warp_argmax_key(unsigned long long& key, int64_t& idx) {
  const unsigned hi = (unsigned)(key >> 32);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned lo = hi == mhi ? (unsigned)key : 0u;
  const unsigned mlo = __reduce_max_sync(0xffffffffu, lo);
  const bool top = hi == mhi && (unsigned)key == mlo;
  const unsigned widx = __reduce_min_sync(0xffffffffu, top ? (unsigned)min(idx, (int64_t)0xffffffff) : 0xffffffffu);
  key = ((unsigned long long)mhi << 32) | mlo;
  idx = widx == 0xffffffffu ? INT64_MAX : (int64_t)widx;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra WAIT_%=;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

constexpr int kPanelWarpThreads = 256;              // 1 poller warp + 7 row warps
constexpr int kPanelWarpRows = kPanelWarpThreads - 32;
constexpr int kRot = kPanelMaxW + 2;                // rotated row copies, zero padded

template <typename T>
__global__ void __launch_bounds__(kPanelWarpThreads, 1) lu_panel_warp_kernel(T* __restrict__ W, PanelArgs a) {
  constexpr int PW = kPanelMaxW;
  constexpr int VW = LLVal<T>::W;
  constexpr int NW = kPanelWarpThreads / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Ls = reinterpret_cast<T*>(smem_raw);  // [ncol][ldt]: retired columns
  __shared__ unsigned long long wk[2][NW];
  __shared__ int64_t wi[2][NW];
  __shared__ __align__(16) T pabs[2][kPanelMaxW];  // [column parity]: pivot row, column order
  __shared__ __align__(16) T dabs[2][kPanelMaxW];  // row i before the swap, column order
  __shared__ __align__(16) T prot[2][kRot];        // prot[k] = pivot row[c + k], zero padded
  __shared__ __align__(16) T drot[2][kRot];        // drot[k] = row i[c + k]
  __shared__ __align__(16) T wstage[NW][2][2 * kPanelMaxW];  // per row warp: rows being published
  __shared__ int64_t s_piv[2];
  __shared__ T s_rcp[2];
  __shared__ __align__(8) uint64_t s_bar;  // poller -> row warps, one phase per column
  const unsigned G = gridDim.x;
  const int per = a.per, ldt = a.ldt;
  const int64_t my_lo = a.kb + (int64_t)blockIdx.x * per;
  const int64_t my_hi = min(a.n, my_lo + per);
  const int nr = (int)(my_hi - my_lo);
  const int ncol = (int)(a.bf - a.kb);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const bool poller = wid == 0;
  const int r = t - 32;  // my row (row warps)
  const bool mine = r >= 0 && r < nr;
  const int64_t g = my_lo + r;
  uint64_t* hdr = a.ll_hdr;    // [2][G][kHdrWords]
  uint64_t* rows = a.ll_row;   // [2][G][kPanelMaxW * VW]
  uint64_t* diag = a.ll_diag;  // [2][kPanelMaxW * VW]
  const int RW = kPanelMaxW * VW;
  if (t == 0) mbar_init(&s_bar, 32);  // every lane of the exchange warp arrives (releases its own writes)

  __syncthreads();  // mbarrier initialised
  // One loop for both roles, so that every warp reaches the CTA-wide barrier of the candidate
  // argmax (cta_argmax_key) at the same code location: the exchange warp (no rows, its
  // candidate is "none") polls and hands over column c, the row warps swap / scale, then all
  // meet in the argmax of column c + 1, then the row warps publish it and finish the update.
  T y[PW];  // y[k] = current value of panel column c + k of my row (zeros in the exchange warp)
#pragma unroll
  for (int k = 0; k < PW; ++k) y[k] = (mine && k < ncol) ? W[g + (a.kb + k) * a.ld] : T(0);
  // column cc's CTA candidate ci and row kb + cc go out as LL words.  y[0] holds
  // column `base` (cc == base: current rows; cc == base + 1: the candidate's
  // column cc is current, columns > cc still miss column base's update).
  auto publish = [&](int cc, int base, int64_t ci) {
    const int par = cc & 1;
    const uint32_t ep = a.seq * 128u + (uint32_t)cc + 1u;
    const int64_t ii = a.kb + cc;
    const bool has_c = ci != INT64_MAX;
    const bool has_d = ii >= my_lo && ii < my_hi;
    const int cw = has_c ? 1 + ((int)(ci - my_lo) >> 5) : -1;
    const int dw = has_d ? 1 + ((int)(ii - my_lo) >> 5) : -1;
    if (has_c ? (mine && g == ci) : t == 32) {
      uint64_t* h = hdr + ((size_t)par * G + blockIdx.x) * kHdrWords;
      const T hv = cc == base ? y[0] : y[1];
      const unsigned long long b = (unsigned long long)__double_as_longlong(has_c ? (double)hv : 0.0);
      ll_store(h, (uint32_t)b, ep);
      ll_store(h + 1, (uint32_t)(b >> 32), ep);
      ll_store(h + 2, has_c ? (uint32_t)ci : 0xffffffffu, ep);
    }
    if (wid == cw || wid == dw) {
      if (mine && (g == ci || g == ii)) {  // y[k] -> slot base + k (slots < cc are not read)
        T* st = wstage[wid][g == ci ? 0 : 1] + base;
#pragma unroll
        for (int k = 0; k < PW; ++k) st[k] = y[k];
        if (g == ci && g == ii) {
          T* st2 = wstage[wid][1] + base;
#pragma unroll
          for (int k = 0; k < PW; ++k) st2[k] = y[k];
        }
      }
      __syncwarp();
      for (int j = lane; j < ncol; j += 32) {
        if (wid == cw) {
          const T v = j < cc ? Ls[j * ldt + (int)(ci - my_lo)] : wstage[wid][0][j];
          LLVal<T>::put(rows + ((size_t)par * G + blockIdx.x) * RW + j * VW, v, ep);
        }
        if (wid == dw) {
          const T v = j < cc ? Ls[j * ldt + (int)(ii - my_lo)] : wstage[wid][1][j];
          LLVal<T>::put(diag + (size_t)par * RW + j * VW, v, ep);
        }
      }
      __syncwarp();
    }
  };

  bool prev_zero = false;  // exchange warp: column c - 1 had a zero pivot (its update was skipped)
  {
    unsigned long long ck = mine ? piv_key(fabs((double)y[0])) : 0ull;
    int64_t ci = mine ? g : INT64_MAX;
    cta_argmax_key(ck, ci, wk[0], wi[0]);
    if (!poller) publish(0, 0, ci);
  }
  for (int c = 0; c < ncol; ++c) {
    const int64_t i = a.kb + c;
    const int par = c & 1;
    // row-warp state carried across the argmax
    const T* pr = prot[par];
    bool act = false;
    T l = T(0);
    long long tr_c = 0, tr_e2 = 0, tr_f = 0;
    if (poller) {
      // ======== exchange warp
      const uint32_t ep = a.seq * 128u + (uint32_t)c + 1u;
      const long long t_c = a.trace ? clock64() : 0;
      // ---- pivot: poll the G headers, reduce (first max, ties -> lowest row)
      unsigned long long gk = 0ull;
      int64_t gi = INT64_MAX;
      double gv = 0.0;
      {
        // up to kHdrPerLane headers per lane, all loads in flight at once; re-poll the
        // ones not yet published
        constexpr int kHdrPerLane = 5;  // G <= 160
        uint64_t x[kHdrPerLane][3];
        unsigned pending = 0;
#pragma unroll
        for (int s2 = 0; s2 < kHdrPerLane; ++s2)
          if (lane + 32 * s2 < (int)G) pending |= 1u << s2;
        SpinGuard sg;
        while (pending) {
          sg.tick();
#pragma unroll
          for (int s2 = 0; s2 < kHdrPerLane; ++s2)
            if (pending >> s2 & 1u) {
              const uint64_t* h = hdr + ((size_t)par * G + lane + 32 * s2) * kHdrWords;
              x[s2][0] = ll_load(h);
              x[s2][1] = ll_load(h + 1);
              x[s2][2] = ll_load(h + 2);
            }
#pragma unroll
          for (int s2 = 0; s2 < kHdrPerLane; ++s2)
            if ((pending >> s2 & 1u) && ll_ok(x[s2][0], ep) && ll_ok(x[s2][1], ep) && ll_ok(x[s2][2], ep))
              pending &= ~(1u << s2);
          if (pending && a.backoff) __nanosleep(a.backoff);
        }
#pragma unroll
        for (int s2 = 0; s2 < kHdrPerLane; ++s2)
          if (lane + 32 * s2 < (int)G) {
            const double v = __longlong_as_double((long long)((x[s2][0] & 0xffffffffull) | (x[s2][1] << 32)));
            const int64_t i2 = (uint32_t)x[s2][2] == 0xffffffffu ? INT64_MAX : (int64_t)(uint32_t)x[s2][2];
            const unsigned long long k2 = i2 == INT64_MAX ? 0ull : piv_key(fabs(v));
            if (k2 > gk || (k2 == gk && i2 < gi)) {
              gk = k2;
              gi = i2;
              gv = v;
            }
          }
      }
      const unsigned long long mk = gk;
      const int64_t mi = gi;
      warp_argmax_key(gk, gi);
      const unsigned src = __ballot_sync(0xffffffffu, mk == gk && mi == gi);
      gv = __shfl_sync(0xffffffffu, gv, src ? __ffs(src) - 1 : 0);
      const long long t_d = a.trace ? clock64() : 0;
      const int64_t p = gi == INT64_MAX ? i : gi;
      const int win = gi == INT64_MAX ? -1 : (int)((gi - a.kb) / per);
      // ---- the winner's row and row i; column c - 1's pending update applied here
      const uint64_t* prow_ll = rows + ((size_t)par * G + (win < 0 ? 0 : win)) * RW;
      const uint64_t* drow_ll = diag + (size_t)par * RW;
      T rcp = div_rn(T(1), (T)gv);  // overlaps the row poll
      const T* pprev = pabs[par ^ 1];  // column c - 1's pivot row
      T pv[2], dv[2];  // columns lane and lane + 32
      {
        uint64_t pw[2][VW], dw[2][VW];
        unsigned pending = (lane < ncol ? 1u : 0u) | (lane + 32 < ncol ? 2u : 0u);
        SpinGuard sg;
        while (pending) {
          sg.tick();
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2)
            if (pending >> s2 & 1u) {
              const int j = lane + 32 * s2;
#pragma unroll
              for (int qq = 0; qq < VW; ++qq) {
                pw[s2][qq] = win < 0 ? ((uint64_t)ep << 32) : ll_load(prow_ll + j * VW + qq);
                dw[s2][qq] = ll_load(drow_ll + j * VW + qq);
              }
            }
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2)
            if (pending >> s2 & 1u) {
              bool ok = true;
#pragma unroll
              for (int qq = 0; qq < VW; ++qq) ok = ok && ll_ok(pw[s2][qq], ep) && ll_ok(dw[s2][qq], ep);
              if (ok) pending &= ~(1u << s2);
            }
          if (pending && a.backoff) __nanosleep(a.backoff);
        }
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          dv[s2] = LLVal<T>::get(dw[s2]);
          pv[s2] = win < 0 ? dv[s2] : LLVal<T>::get(pw[s2]);
        }
      }
      if (c > 0 && !prev_zero) {
        // the owners published before column c - 1's update: v -= l * u for columns > c,
        // l = the row's own column c - 1 (its multiplier), u = column c - 1's pivot row
        const int jl = c - 1;
        const T lp = __shfl_sync(0xffffffffu, jl < 32 ? pv[0] : pv[1], jl & 31);
        const T ld_ = __shfl_sync(0xffffffffu, jl < 32 ? dv[0] : dv[1], jl & 31);
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          const int j = lane + 32 * s2;
          if (j > c && j < ncol) {
            const T up = pprev[j];
            dv[s2] = sub_rn(dv[s2], mul_rn(ld_, up));
            pv[s2] = win < 0 ? dv[s2] : sub_rn(pv[s2], mul_rn(lp, up));
          }
        }
      }
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        const int j = lane + 32 * s2;
        if (j < ncol) {
          pabs[par][j] = pv[s2];
          dabs[par][j] = dv[s2];
          if (j >= c) {
            prot[par][j - c] = pv[s2];
            drot[par][j - c] = dv[s2];
          }
        }
      }
      for (int k = ncol - c + lane; k < kRot; k += 32) {  // zero pad past the panel
        prot[par][k] = T(0);
        drot[par][k] = T(0);
      }
      __syncwarp();
      const T aii = prot[par][0];
      if (gi == INT64_MAX) rcp = div_rn(T(1), aii);
      prev_zero = aii == T(0);
      if (lane == 0) {
        s_piv[par] = p;
        s_rcp[par] = rcp;
        if (blockIdx.x == 0) {
          a.piv[i] = p;                         // piv[i] = v (direct.py:67)
          if (prev_zero) a.zero_cols[i] = 1;    // direct.py:71-74
        }
      }
      __syncwarp();
      mbar_arrive(&s_bar);
      if (a.trace && t == 0) {
        unsigned long long* tr = a.trace + (size_t)blockIdx.x * 8;
        tr[2] += t_d - t_c;         // header poll + reduce
        tr[4] += clock64() - t_d;   // row poll + handoff
      }
    } else {
      // ======== row warps
      tr_c = a.trace ? clock64() : 0;
      mbar_wait(&s_bar, (unsigned)par);
      tr_e2 = a.trace ? clock64() : 0;
      const T* pa = pabs[par];
      const T* da = dabs[par];
      const T* dr = drot[par];
      const int64_t p = s_piv[par];
      const T aii = pr[0];
      const bool zero = aii == T(0);
      // ---- swap (direct.py:68-70, restricted to the panel): retired columns by the
      // owning warps, the register rows by their threads
      if (p != i) {
        if (i >= my_lo && i < my_hi && wid == 1 + ((int)(i - my_lo) >> 5))
          for (int j = lane; j < c; j += 32) Ls[j * ldt + (int)(i - my_lo)] = pa[j];
        if (p >= my_lo && p < my_hi && wid == 1 + ((int)(p - my_lo) >> 5))
          for (int j = lane; j < c; j += 32) Ls[j * ldt + (int)(p - my_lo)] = da[j];
        if (mine && (g == i || g == p)) {
          const T* src = g == i ? pr : dr;
#pragma unroll
          for (int k = 0; k < PW; ++k) y[k] = src[k];
        }
      }
      // ---- reciprocal scale and the update of column c + 1 first
      act = mine && g > i && !zero;
      if (act) {
        l = mul_rn(s_rcp[par], y[0]);
        y[0] = l;
        y[1] = sub_rn(y[1], mul_rn(l, pr[1]));
      }
      if (mine) Ls[c * ldt + r] = y[0];  // retire column c
      tr_f = a.trace ? clock64() : 0;
    }
    // ---- next column's CTA candidate (rows >= i + 1): the one CTA-wide barrier, then its
    // header and rows go out before the rest of the update
    if (c + 1 < ncol) {
      const bool cand = !poller && mine && g > i;
      unsigned long long ck = cand ? piv_key(fabs((double)y[1])) : 0ull;
      int64_t ci = cand ? g : INT64_MAX;
      cta_argmax_key(ck, ci, wk[(c + 1) & 1], wi[(c + 1) & 1]);
      if (!poller) publish(c + 1, c, ci);
    }
    if (!poller) {
      const long long tr_g = a.trace ? clock64() : 0;
      // ---- rest of the rank-1 update (direct.py:75-79), then rotate by one
      if (act) {
#pragma unroll
        for (int k = 2; k < PW; ++k) y[k] = sub_rn(y[k], mul_rn(l, pr[k]));
      }
#pragma unroll
      for (int k = 0; k + 1 < PW; ++k) y[k] = y[k + 1];
      y[PW - 1] = T(0);
      if (a.trace && t == 32) {
        const long long t_h = clock64();
        unsigned long long* tr = a.trace + (size_t)blockIdx.x * 8;
        tr[3] += tr_e2 - tr_c;  // wait for the handoff
        tr[0] += tr_f - tr_e2;  // swap, scale
        tr[1] += tr_g - tr_f;   // next column's CTA argmax + publish
        tr[5] += t_h - tr_g;    // update, rotate
      }
    }
  }
  __syncthreads();
  for (int idx = t; idx < ncol * nr; idx += blockDim.x) {
    const int j = idx / nr, rr = idx % nr;
    W[(my_lo + rr) + (a.kb + j) * a.ld] = Ls[j * ldt + rr];
  }
}

// Fallback for panels too large for shared memory (e.g. the unblocked b = n
// factorization): rows stay in global memory (L2), two grid barriers per column.
template <typename T>
__global__ void __launch_bounds__(kPanelThreads) lu_panel_global_kernel(T* __restrict__ W, PanelArgs a) {
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  __shared__ int64_t s_piv;
  const unsigned G = gridDim.x;
  const int64_t per = a.per;
  const int64_t my_lo = a.kb + (int64_t)blockIdx.x * per;
  const int64_t my_hi = min(a.n, my_lo + per);
  const int64_t nr = my_hi - my_lo;
  const int64_t ncol = a.bf - a.kb;
  T* rowP = reinterpret_cast<T*>(a.rowP);
  T* rowI = reinterpret_cast<T*>(a.rowI);
  unsigned epoch = 0;
  for (int64_t c = 0; c < ncol; ++c) {
    const int64_t i = a.kb + c;
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t r = max(my_lo, i) + threadIdx.x; r < my_hi; r += blockDim.x) {
      const double v = fabs((double)W[r + i * a.ld]);
      if (piv_better(v, r, bv, bi)) {
        bv = v;
        bi = r;
      }
    }
    block_argmax(bv, bi, sv, si);
    if (threadIdx.x == 0) {
      a.cand_v[blockIdx.x] = bv;
      a.cand_i[blockIdx.x] = bi;
    }
    grid_sync(a.bar, G, epoch);
    reduce_candidates(a, 0, i, &s_piv, sv, si);
    const int64_t p = s_piv;
    if (blockIdx.x == 0) {
      if (threadIdx.x == 0) a.piv[i] = p;
      for (int64_t j = threadIdx.x; j < ncol; j += blockDim.x) {
        rowP[j] = __ldcg(W + p + (a.kb + j) * a.ld);
        rowI[j] = __ldcg(W + i + (a.kb + j) * a.ld);
      }
    }
    grid_sync(a.bar, G, epoch);
    if (p != i) {
      if (i >= my_lo && i < my_hi)
        for (int64_t j = threadIdx.x; j < ncol; j += blockDim.x) W[i + (a.kb + j) * a.ld] = __ldcg(rowP + j);
      if (p >= my_lo && p < my_hi)
        for (int64_t j = threadIdx.x; j < ncol; j += blockDim.x) W[p + (a.kb + j) * a.ld] = __ldcg(rowI + j);
    }
    __syncthreads();
    const T aii = __ldcg(rowP + c);
    if (aii == T(0)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) a.zero_cols[i] = 1;
    } else {
      const T recip = div_rn(T(1), aii);
      const int64_t u0 = max(my_lo, i + 1);
      const int64_t nu = my_hi - u0;
      for (int64_t r = u0 + threadIdx.x; r < my_hi; r += blockDim.x)
        W[r + i * a.ld] = mul_rn(recip, W[r + i * a.ld]);
      __syncthreads();
      const int64_t w = ncol - c - 1;
      if (nu > 0)
        for (int64_t idx = threadIdx.x; idx < w * nu; idx += blockDim.x) {
          const int64_t j = i + 1 + idx / nu, r = u0 + idx % nu;
          W[r + j * a.ld] = sub_rn(W[r + j * a.ld], mul_rn(W[r + i * a.ld], __ldcg(rowP + (j - a.kb))));
        }
    }
    (void)nr;
  }
}

// laswp (K11): the swaps piv[kb..bf) applied, in order, to columns outside the
// panel.  A one-thread kernel first folds the swap sequence into its net
// permutation of the affected rows ({kb..bf-1} U {piv[k]}): pairs (dst, src)
// meaning "row dst receives the original row src".  The gather kernel then
// moves every affected element of a column at once (all loads before all
// stores, no dependent chains); rows kb..bf-1 of a column are contiguous.
// Parallel plan for cnt <= kPlanMax (256 threads).  Swap k exchanges positions
// k and s_k >= k, so position k is final after step k: the slots s_k are
// resolved in parallel (rows outside the panel are deduplicated into compact
// slots cnt + r, first occurrence first), only the swap replay itself is a
// serial loop over shared memory, and the (dst, src) compaction is a warp
// ballot scan.  Same output layout as the serial kernel.
constexpr int kPlanMax = 512;
__global__ void __launch_bounds__(256)
    laswp_plan_kernel(int64_t kb, int64_t bf, const int64_t* __restrict__ piv, int64_t* pairs,
                      int* npairs) {
  __shared__ int64_t P[kPlanMax];         // pivot rows
  __shared__ int64_t home[2 * kPlanMax];  // row label of each slot
  __shared__ int64_t orig[2 * kPlanMax];  // content (original row) of each slot after the swaps
  __shared__ int S[kPlanMax];             // slot swapped with position k
  __shared__ int rank[kPlanMax];          // compact index of an outside row (first occurrence)
  __shared__ int s_nout;
  // outside rows -> their first position k: an open-addressing table (load <= 1/2), so the
  // first-occurrence test is O(cnt) instead of a scan of all earlier pivots per entry
  constexpr int kH = 2 * kPlanMax;
  __shared__ unsigned long long hkey[kH];
  __shared__ int hfirst[kH];
  const int cnt = (int)(bf - kb);
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < kH; i += blockDim.x) {
    hkey[i] = ~0ull;
    hfirst[i] = INT_MAX;
  }
  for (int k = tid; k < cnt; k += blockDim.x) P[k] = piv[kb + k];
  __syncthreads();
  auto slot_of = [&](unsigned long long key) {
    unsigned h = (unsigned)((key * 0x9E3779B97F4A7C15ull) >> 40) & (kH - 1);
    while (hkey[h] != key) h = (h + 1) & (kH - 1);
    return h;
  };
  for (int k = tid; k < cnt; k += blockDim.x) {
    if (P[k] < bf) continue;
    const unsigned long long key = (unsigned long long)P[k];
    unsigned h = (unsigned)((key * 0x9E3779B97F4A7C15ull) >> 40) & (kH - 1);
    while (true) {
      const unsigned long long prev = atomicCAS(&hkey[h], ~0ull, key);
      if (prev == ~0ull || prev == key) {
        atomicMin(&hfirst[h], k);
        break;
      }
      h = (h + 1) & (kH - 1);
    }
  }
  __syncthreads();
  // first occurrence of each outside row
  for (int k = tid; k < cnt; k += blockDim.x)
    rank[k] = P[k] >= bf && hfirst[slot_of((unsigned long long)P[k])] == k ? 1 : 0;
  __syncthreads();
  if (tid < 32) {  // exclusive scan of the first-occurrence flags
    int base = 0;
    for (int k0 = 0; k0 < cnt; k0 += 32) {
      const int k = k0 + lane;
      const int f = k < cnt ? rank[k] : 0;
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if (k < cnt) rank[k] = f ? base + __popc(m & ((1u << lane) - 1)) : -1;
      base += __popc(m);
    }
    if (lane == 0) s_nout = base;
  }
  __syncthreads();
  for (int k = tid; k < cnt; k += blockDim.x) {
    const int64_t p = P[k];
    int slot;
    if (p < bf) {
      slot = (int)(p - kb);
    } else {
      int r = rank[k];
      if (r < 0) {
        r = rank[hfirst[slot_of((unsigned long long)p)]];
      } else {
        home[cnt + r] = p;
        orig[cnt + r] = p;
      }
      slot = cnt + r;
    }
    S[k] = slot;
    home[k] = kb + k;
    orig[k] = kb + k;
  }
  __syncthreads();
  if (tid == 0) {  // replay the swaps (direct.py:68-70 applied to row labels)
    for (int k = 0; k < cnt; ++k) {
      const int sk = S[k];
      if (sk != k) {
        const int64_t t = orig[k];
        orig[k] = orig[sk];
        orig[sk] = t;
      }
    }
  }
  __syncthreads();
  if (tid < 32) {  // compact the moved slots into (dst, src) pairs
    const int tot = cnt + s_nout;
    int64_t* dst = pairs + 4 * cnt;
    int64_t* src = pairs + 6 * cnt;
    int base = 0;
    for (int q0 = 0; q0 < tot; q0 += 32) {
      const int q = q0 + lane;
      const bool mv = q < tot && orig[q] != home[q];
      const unsigned m = __ballot_sync(0xffffffffu, mv);
      if (mv) {
        const int o = base + __popc(m & ((1u << lane) - 1));
        dst[o] = home[q];
        src[o] = orig[q];
      }
      base += __popc(m);
    }
    if (lane == 0) *npairs = base;
  }
}

__global__ void laswp_plan_serial_kernel(int64_t kb, int64_t bf, const int64_t* __restrict__ piv,
                                  int64_t* pairs /* [8*cnt] */, int* npairs) {
  // one warp; the working maps live in shared memory (cnt <= kLaswpSmem), else in `pairs`
  extern __shared__ int64_t sm[];
  const int cnt = (int)(bf - kb);
  const int lane = threadIdx.x;
  const bool in_smem = cnt <= 1024;
  int64_t* orig_in = in_smem ? sm : pairs;                 // [cnt]
  int64_t* out_rows = in_smem ? sm + cnt : pairs + 2 * cnt;  // [cnt]
  int64_t* out_orig = in_smem ? sm + 2 * cnt : pairs + 3 * cnt;
  __shared__ int s_nout;
  __shared__ int64_t s_piv[1024];
  for (int k = lane; k < cnt && k < 1024; k += 32) s_piv[k] = piv[kb + k];
  for (int k = lane; k < cnt; k += 32) orig_in[k] = kb + k;
  if (lane == 0) s_nout = 0;
  __syncwarp();
  for (int k = 0; k < cnt; ++k) {
    const int64_t p = k < 1024 ? s_piv[k] : piv[kb + k];
    if (p == kb + k) continue;
    int64_t* op;
    if (p < bf) {
      op = &orig_in[p - kb];
    } else {
      const int nout = s_nout;
      int f = -1;
      for (int q0 = 0; q0 < nout && f < 0; q0 += 32) {
        const int q = q0 + lane;
        const unsigned m = __ballot_sync(0xffffffffu, q < nout && out_rows[q] == p);
        if (m) f = q0 + __ffs(m) - 1;
      }
      if (f < 0) {
        f = nout;
        if (lane == 0) {
          out_rows[f] = p;
          out_orig[f] = p;
          s_nout = nout + 1;
        }
      }
      op = &out_orig[f];
    }
    __syncwarp();
    if (lane == 0) {
      const int64_t t = orig_in[k];
      orig_in[k] = *op;
      *op = t;
    }
    __syncwarp();
  }
  // compact into (dst, src) pairs: dst at pairs+4cnt, src at pairs+6cnt
  if (lane == 0) {
    int64_t* dst = pairs + 4 * cnt;
    int64_t* src = pairs + 6 * cnt;
    int np = 0;
    for (int k = 0; k < cnt; ++k)
      if (orig_in[k] != kb + k) {
        dst[np] = kb + k;
        src[np] = orig_in[k];
        ++np;
      }
    for (int q = 0; q < s_nout; ++q)
      if (out_orig[q] != out_rows[q]) {
        dst[np] = out_rows[q];
        src[np] = out_orig[q];
        ++np;
      }
    *npairs = np;
  }
}

// One CTA per group of `cols` columns: every affected element of those columns
// is first read into shared memory, then written to its destination row.
template <typename T>
__global__ void __launch_bounds__(256)
    laswp_gather_kernel(T* W, int64_t ld, int64_t c_lo, int64_t c_hi, int cols,
                        const int64_t* __restrict__ dst, const int64_t* __restrict__ src,
                        const int* __restrict__ npairs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* buf = reinterpret_cast<T*>(smem_raw);  // [cols][np]
  const int np = *npairs;
  const int64_t c0 = c_lo + (int64_t)blockIdx.x * cols;
  const int nc = (int)min((int64_t)cols, c_hi - c0);
  // thread <-> pair (rows kb..bf-1 of the plan are contiguous: coalesced), loop over columns
  for (int t = threadIdx.x; t < np; t += blockDim.x) {
    const int64_t s_ = src[t];
    T v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = q < nc ? W[s_ + (c0 + q) * ld] : T(0);  // 8 loads in flight
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < nc) buf[q * np + t] = v[q];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < np; t += blockDim.x) {
    const int64_t d_ = dst[t];
    for (int q = 0; q < nc; ++q) W[d_ + (c0 + q) * ld] = buf[q * np + t];
  }
}

struct SwapPlan {
  int64_t* pairs = nullptr;
  int* np = nullptr;
  int64_t cnt = 0;
};

int laswp_plan(ds_ctx* ctx, int64_t kb, int64_t bf, const int64_t* piv, SwapPlan& sp) {
  sp.cnt = bf - kb;
  if (sp.cnt <= kPlanMax) {
    laswp_plan_kernel<<<1, 256, 0, ctx->stream>>>(kb, bf, piv, sp.pairs, sp.np);
  } else {
    const size_t smem = sp.cnt <= 1024 ? (size_t)3 * sp.cnt * sizeof(int64_t) : 0;
    laswp_plan_serial_kernel<<<1, 32, smem, ctx->stream>>>(kb, bf, piv, sp.pairs, sp.np);
  }
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

template <typename T>
int laswp_apply(ds_ctx* ctx, T* W, int64_t ld, int64_t c_lo, int64_t c_hi, const SwapPlan& sp) {
  if (c_hi <= c_lo) return DS_OK;
  // np <= 2*cnt; size the column group so the staging buffer stays <= 192 KB
  const int64_t npmax = 2 * sp.cnt;
  const int cols = (int)std::max<int64_t>(1, std::min<int64_t>(8, (192 * 1024) / (npmax * (int64_t)sizeof(T))));  // <= 8 (kernel unroll)
  const size_t smem = (size_t)cols * npmax * sizeof(T);
  static size_t attr[2] = {0, 0};
  size_t& done = attr[sizeof(T) == 8 ? 1 : 0];
  if (smem > 48 * 1024 && smem > done) {
    DS_CUDA(cudaFuncSetAttribute(laswp_gather_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(200 * 1024)));
    done = 200 * 1024;
  }
  const unsigned grid = (unsigned)ceil_div(c_hi - c_lo, cols);
  laswp_gather_kernel<T><<<grid, 256, smem, ctx->stream>>>(W, ld, c_lo, c_hi, cols, sp.pairs + 4 * sp.cnt,
                                                           sp.pairs + 6 * sp.cnt, sp.np);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

// bytes of the per-launch panel scratch carved in panel_launch (with 256-B alignment slack)
template <typename T>
size_t panel_scratch_bytes(int64_t b) {
  return 256 + 2 * 1024 * 16 + sizeof(T) * (2 * 1024 * kPanelMaxW + 2 * kPanelMaxW) +
         2 * sizeof(T) * (size_t)std::max<int64_t>(b, 1) + sizeof(uint64_t) * 2 * 1024 * kHdrWords +
         sizeof(uint64_t) * 2 * 1024 * kPanelMaxW * 2 + sizeof(uint64_t) * 2 * kPanelMaxW * 2 + 16 * 256;
}

// Can all g CTAs of a panel kernel be resident at once (the LL exchange's forward-progress
// condition)?  Occupancy per (kernel, block, smem) is cached; the kernel attributes are set
// first so the query sees the opted-in shared memory.
static bool panel_fits_resident(ds_ctx* ctx, void* kfn, int nthr, size_t smem, size_t smem_cap, int64_t g,
                                bool f64) {
  static std::mutex mu;
  static std::map<std::tuple<void*, int, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(kfn, nthr, smem);
  auto it = cache.find(key);
  if (it == cache.end()) {
    (void)f64;
    (void)smem_cap;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, nthr, smem) != cudaSuccess) {
      cudaGetLastError();
      per_sm = 0;
    }
    it = cache.emplace(key, per_sm).first;
  }
  return (int64_t)it->second * ctx->num_sms >= g;
}

template <typename T>
int panel_launch(ds_ctx* ctx, T* W, int64_t n, int64_t ld, int64_t kb, int64_t bf, int64_t* piv,
                 int8_t* zero_cols, char* scratch) {
  const int64_t rows = n - kb, ncol = bf - kb;
  PanelArgs a;
  a.n = n;
  a.ld = ld;
  a.kb = kb;
  a.bf = bf;
  a.piv = piv;
  a.zero_cols = zero_cols;
  Carver cv{scratch};
  a.bar = cv.take<unsigned>(256);
  a.cand_v = cv.take<double>(sizeof(double) * 2 * 1024);
  a.cand_i = cv.take<int64_t>(sizeof(int64_t) * 2 * 1024);
  a.cand_row = cv.take<T>(sizeof(T) * 2 * 1024 * kPanelMaxW);
  a.diag_row = cv.take<T>(sizeof(T) * 2 * kPanelMaxW);
  a.rowP = cv.take<T>(sizeof(T) * ncol);
  a.rowI = cv.take<T>(sizeof(T) * ncol);
  a.ll_hdr = cv.take<uint64_t>(sizeof(uint64_t) * 2 * 1024 * kHdrWords);
  a.ll_row = cv.take<uint64_t>(sizeof(uint64_t) * 2 * 1024 * kPanelMaxW * 2);
  a.ll_diag = cv.take<uint64_t>(sizeof(uint64_t) * 2 * kPanelMaxW * 2);
  a.seq = next_ll_epoch();
  a.trace = nullptr;
  static const int backoff = [] {
    const char* e = getenv("DENSOLVE_PANEL_BACKOFF");
    return e ? atoi(e) : 0;
  }();
  a.backoff = backoff;
  const size_t smem_cap = std::min<size_t>(ctx->smem_optin, 220 * 1024) - 2048;
  // shared-memory path: rows split over <= num_sms CTAs, >= 16 rows each
  if (ncol <= kPanelMaxW) {
    // rows per CTA: at least `target` (fewer CTAs leave SMs to the concurrent look-ahead GEMM)
    static int64_t target = [] {
      const char* e = getenv("DENSOLVE_PANEL_ROWS");
      return e ? std::max<int64_t>(16, atoll(e)) : (int64_t)256;
    }();
    // kernel choice (measured per column, n = 16384): the poller-warp kernel wins for
    // 2..40 CTAs of <= 224 rows (2.9 vs 3.3 us at G = 10); the CTA-synchronous
    // register-row kernel for one CTA (shared memory only) and for the tall panels.
    // DENSOLVE_PANEL_KERNEL = 1 / 2 forces one of them.
    static const int force = [] {
      const char* e = getenv("DENSOLVE_PANEL_KERNEL");
      return e ? atoi(e) : 0;
    }();
    static const int64_t kWarpMaxG = [] {  // tuning knob
      const char* e = getenv("DENSOLVE_PANEL_WARP_MAXG");
      return e ? (int64_t)atoll(e) : (int64_t)40;
    }();
    const int64_t gw = ceil_div(rows, (int64_t)kPanelWarpRows);
    const bool warp_k = force == 1 ? gw <= (int64_t)ctx->num_sms : force == 2 ? false : (gw >= 2 && gw <= kWarpMaxG);
    int64_t g = warp_k ? gw : std::min<int64_t>((int64_t)ctx->num_sms, ceil_div(rows, target));
    int64_t per = ceil_div(rows, g);
    g = ceil_div(rows, per);
    const int ldt = (int)(per | 1);
    const size_t smem = (size_t)ncol * ldt * sizeof(T);
    const int tpr = warp_k ? 1 : per <= kPanelRegThreads / 4 ? 4 : 2;
    const int nthr_pre = warp_k ? (int)(32 + ceil_div(per, 32) * 32)
                                : (int)std::max<int64_t>(ceil_div(per * tpr, 32) * 32, ceil_div(g, 32) * 32);
    void* kfn_pre = warp_k     ? (void*)lu_panel_warp_kernel<T>
                    : tpr == 4 ? (void*)lu_panel_smem_kernel<T, 4>
                               : (void*)lu_panel_smem_kernel<T, 2>;
    static bool attr_set[2] = {false, false};
    if (!attr_set[sizeof(T) == 8 ? 1 : 0]) {
      DS_CUDA(cudaFuncSetAttribute(lu_panel_smem_kernel<T, 2>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap));
      DS_CUDA(cudaFuncSetAttribute(lu_panel_smem_kernel<T, 4>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap));
      // <= 256 rows x 64 columns of retired values (131.6 KB) beside ~26 KB of static buffers
      DS_CUDA(cudaFuncSetAttribute(lu_panel_warp_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)std::min<size_t>(smem_cap, 160 * 1024)));
      attr_set[sizeof(T) == 8 ? 1 : 0] = true;
    }
    if (smem <= smem_cap && per * tpr <= kPanelRegThreads &&
        panel_fits_resident(ctx, kfn_pre, nthr_pre, smem, smem_cap, g, sizeof(T) == 8)) {
      a.per = (int)per;
      a.ldt = ldt;
      const int nthr = warp_k ? (int)(32 + ceil_div(per, 32) * 32)
                             : (int)std::max<int64_t>(ceil_div(per * tpr, 32) * 32, ceil_div(g, 32) * 32);
      void* kfn = warp_k     ? (void*)lu_panel_warp_kernel<T>
                  : tpr == 4 ? (void*)lu_panel_smem_kernel<T, 4>
                             : (void*)lu_panel_smem_kernel<T, 2>;
      const char* tr = getenv("DENSOLVE_PANEL_TRACE");  // debug: per-phase timestamps of one panel
      const bool tracing = tr && atoll(tr) == kb;
      if (tracing) {
        DS_CUDA(cudaMalloc((void**)&a.trace, sizeof(unsigned long long) * g * 8));
        DS_CUDA(cudaMemsetAsync(a.trace, 0, sizeof(unsigned long long) * g * 8, ctx->stream));
      }
      void* args[] = {(void*)&W, (void*)&a};
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (tracing) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, ctx->stream);
      }
      // a plain launch: grid <= #SMs at one CTA per SM, so every CTA becomes resident once
      // any concurrent (look-ahead) GEMM CTAs retire; a cooperative launch costs ~10x
      // more host time per panel
      DS_CUDA(cudaLaunchKernel(kfn, dim3((unsigned)g), dim3((unsigned)nthr), args, smem, ctx->stream));
      count_launch(ctx);
      if (tracing) {
        cudaEventRecord(e1, ctx->stream);
        std::vector<unsigned long long> h((size_t)g * 8);
        DS_CUDA(cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
        DS_CUDA(cudaStreamSynchronize(ctx->stream));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaFree(a.trace);
        a.trace = nullptr;
        double mean[7] = {}, mx[7] = {};
        for (int64_t b = 0; b < g; ++b)
          for (int k = 0; k < 7; ++k) {
            mean[k] += (double)h[b * 8 + k] / g / ncol;
            mx[k] = std::max(mx[k], (double)h[b * 8 + k] / ncol);
          }
        fprintf(stderr, "[panel trace] kb=%lld rows=%lld G=%lld per=%lld: %.2f us/column (events); cycles/column "
                "mean(max) [poller kernel: 0 swap+scale, 1 next argmax+publish, 2 poller hdr poll, 3 row-warp wait, "
                "4 poller row poll, 5 update; cta kernel: 0 swap+scale, 1 next argmax, 2 hdr poll, 3 hdr argmax, 4 row "
                "poll+sync, 5 update, 6 publish rows]: %.0f(%.0f) %.0f(%.0f) %.0f(%.0f) %.0f(%.0f) %.0f(%.0f) %.0f(%.0f) "
                "%.0f(%.0f) [tpr %d, %d threads]\n",
                (long long)kb, (long long)rows, (long long)g, (long long)per, 1e3 * ms / ncol, mean[0], mx[0],
                mean[1], mx[1], mean[2], mx[2], mean[3], mx[3], mean[4], mx[4], mean[5], mx[5], mean[6], mx[6],
                tpr, nthr);
      }
      return DS_OK;
    }
  }
  static int mb[2] = {0, 0};
  int& m = mb[sizeof(T) == 8 ? 1 : 0];
  if (m == 0) {
    DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, lu_panel_global_kernel<T>, kPanelThreads, 0));
    if (m < 1) m = 1;
  }
  DS_CUDA(cudaMemsetAsync(a.bar, 0, 256, ctx->stream));
  int64_t g = std::min<int64_t>(ceil_div(rows, 64), (int64_t)ctx->num_sms);
  g = std::max<int64_t>(1, g);
  int64_t per = ceil_div(rows, g);
  g = ceil_div(rows, per);
  a.per = (int)per;
  a.ldt = 0;
  void* args[] = {(void*)&W, (void*)&a};
  DS_CUDA(cudaLaunchCooperativeKernel((void*)lu_panel_global_kernel<T>, dim3((unsigned)g),
                                      dim3(kPanelThreads), args, 0, ctx->stream));
  count_launch(ctx);
  return DS_OK;
}

// Internal outer block: the reference's b-wide panels are kept (pivot search,
// swaps, scaling and rank-1 updates inside each b-panel, then TRSM + GEMM on the
// rest of the outer panel), but the trailing matrix is updated once per NB-wide
// outer panel with a K = NB GEMM.  Exact-arithmetic identical to the reference
// (same pivots), different rounding grouping in the trailing update.
static int64_t outer_block(int64_t b, int64_t n) {
  static const int64_t nb_target = [] {
    const char* e = getenv("DENSOLVE_LU_NB");  // tuning knob; default 512
    return e ? std::max<int64_t>(64, atoll(e)) : (int64_t)512;
  }();
  if (b >= nb_target || b >= n) return std::min<int64_t>(b, n);
  return std::min<int64_t>(n, b * std::max<int64_t>(1, nb_target / b));
}

// Factor the m x w (m >= w) column-major panel W in place: rows [0, m), columns
// [0, w).  m == w is the square factorization of ds_lu_factor.
//
// Look-ahead: after panel k's swaps and U01 are formed, the next outer panel's
// NB columns get their trailing update first; the factorization of panel k+1
// (cooperative panel kernels, inner TRSM/GEMM) is then enqueued on a
// high-priority side stream while the bulk trailing GEMM of panel k runs on the
// main stream (disjoint columns), and the main stream waits for it before
// applying panel k+1's swaps.
static bool lu_lookahead_enabled() {
  const char* e = getenv("DENSOLVE_LU_LOOKAHEAD");
  return !(e && e[0] == '0');
}

template <typename T>
int lu_factor_impl(ds_ctx* ctx, int64_t m, int64_t w, T* W, int64_t ld, int64_t b, int64_t* d_piv,
                   int8_t* d_zero) {
  void* ws = nullptr;
  const int64_t NB = outer_block(b, w);
  const size_t scratch_bytes = panel_scratch_bytes<T>(b);
  DS_TRY(ctx_workspace(ctx, scratch_bytes + 2 * sizeof(int64_t) * 8 * (size_t)NB + 4096, &ws));
  Carver cvs{(char*)ws};
  char* scratch = cvs.take<char>(scratch_bytes);
  SwapPlan sp_in, sp_out;
  sp_in.pairs = cvs.take<int64_t>(sizeof(int64_t) * 8 * (size_t)NB);
  sp_in.np = cvs.take<int>(64);
  sp_out.pairs = cvs.take<int64_t>(sizeof(int64_t) * 8 * (size_t)NB);
  sp_out.np = cvs.take<int>(64);

  const bool lookahead = lu_lookahead_enabled() && w > NB && m >= 2048;
  if (lookahead && !ctx->side) {
    int lo = 0, hi = 0;
    DS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    DS_CUDA(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, hi));
    DS_CUDA(cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, lo));
    DS_CUDA(cudaEventCreateWithFlags(&ctx->ev_a, cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&ctx->ev_b, cudaEventDisableTiming));
    DS_CUDA(cudaEventCreateWithFlags(&ctx->ev_c, cudaEventDisableTiming));
  }
  // tile / worker counters of the SM-reserving trailing GEMM (allocated once per context,
  // outside the enqueue sequence)
  if (lookahead && !ctx->gemm_ctr) DS_CUDA(cudaMalloc((void**)&ctx->gemm_ctr, 2 * sizeof(unsigned)));
  // swap plans of the L-column swaps (aux stream): one per outer panel, kept
  // alive until the aux stream drains
  const int64_t nouter = ceil_div(w, NB);
  int64_t* left_pairs = nullptr;
  int* left_np = nullptr;
  if (lookahead) {
    DS_CUDA(cudaMallocAsync((void**)&left_pairs, sizeof(int64_t) * 8 * (size_t)NB * nouter, ctx->stream));
    DS_CUDA(cudaMallocAsync((void**)&left_np, sizeof(int) * 64 * nouter, ctx->stream));
  }

  // factor the outer panel [kb, bf) with the reference's b-wide blocking
  auto factor_outer = [&](int64_t kb, int64_t bf) -> int {
    for (int64_t ib = kb; ib < bf; ib += b) {
      const int64_t ibf = std::min<int64_t>(ib + b, bf);
      DS_TRY(panel_launch<T>(ctx, W, m, ld, ib, ibf, d_piv, d_zero, scratch));
      if (ib == kb && ibf == bf) continue;  // no columns of the outer panel outside this b-panel
      DS_TRY(laswp_plan(ctx, ib, ibf, d_piv, sp_in));
      DS_TRY(laswp_apply<T>(ctx, W, ld, kb, ib, sp_in));
      DS_TRY(laswp_apply<T>(ctx, W, ld, ibf, bf, sp_in));
      if (ibf < bf) {
        T* U = W + ib + ibf * ld;
        DS_TRY(trsm_lower_unit_launch<T>(ctx, ibf - ib, bf - ibf, W + ib + ib * ld, ld, U, ld, U, ld));
        DS_TRY(gemm_launch<T>(ctx, m - ibf, bf - ibf, ibf - ib, -1.0, W + ibf + ib * ld, ld, U, ld, 1.0,
                              W + ibf + ibf * ld, ld, W + ibf + ibf * ld, ld));
      }
    }
    return DS_OK;
  };
  // U01 = L00^-1 A01 and A11 -= L10 U01 for trailing columns [c0, c1)
  // U01 of the outer panel in one launch (fp64, b = 64, whole 64-row blocks); bitwise the
  // TRSM / GEMM chain below.  DENSOLVE_LU_U01_FUSED=0 keeps the chain.
  static const bool u01_fused = [] {
    const char* e = getenv("DENSOLVE_LU_U01_FUSED");
    return !(e && e[0] == '0');
  }();
  auto outer_update = [&](int64_t kb, int64_t bf, int64_t c0, int64_t c1, int reserve, bool fuse = false) -> int {
    if (c1 <= c0) return DS_OK;
    if (fuse && sizeof(T) == 8 && u01_fused && b == 64 && (bf - kb) % 64 == 0) {
      DS_TRY(u01_fused_launch(ctx, reinterpret_cast<double*>(W), ld, kb, (int)((bf - kb) / 64), c0, c1));
    } else
    for (int64_t ib = kb; ib < bf; ib += b) {
      const int64_t ibf = std::min<int64_t>(ib + b, bf);
      T* Ur = W + ib + c0 * ld;
      DS_TRY(trsm_lower_unit_launch<T>(ctx, ibf - ib, c1 - c0, W + ib + ib * ld, ld, Ur, ld, Ur, ld));
      if (ibf < bf)
        DS_TRY(gemm_launch<T>(ctx, bf - ibf, c1 - c0, ibf - ib, -1.0, W + ibf + ib * ld, ld, Ur, ld, 1.0,
                              W + ibf + c0 * ld, ld, W + ibf + c0 * ld, ld));
    }
    ctx->gemm_reserve = reserve;
    const int rc = gemm_launch<T>(ctx, m - bf, c1 - c0, bf - kb, -1.0, W + bf + kb * ld, ld, W + kb + c0 * ld, ld,
                                  1.0, W + bf + c0 * ld, ld, W + bf + c0 * ld, ld);
    ctx->gemm_reserve = 0;
    return rc;
  };
  // SMs kept free of the trailing GEMM while the look-ahead factorization of the outer panel
  // [bf, bf2) runs on the side stream (0: none).  Only where the GEMM on the remaining SMs is
  // predicted to finish within the side stream's time (the tail of the factorization, where
  // the chain of panels is the critical path): there every side-stream launch would otherwise
  // wait for trailing-GEMM CTAs to retire.  Model: 33 TFLOP/s DMMA, ~4.5 us per panel column.
  static const double reserve_ratio = [] {
    const char* e = getenv("DENSOLVE_LU_RESERVE");  // tuning knob: 0 disables
    return e ? atof(e) : 1.0;
  }();
  auto side_reserve = [&](int64_t bf, int64_t bf2) -> int {
    if (reserve_ratio <= 0 || sizeof(T) != 8) return 0;
    const int64_t rows = m - bf, nsm = ctx->num_sms;
    const int64_t gw = ceil_div(rows, (int64_t)kPanelWarpRows);
    const int64_t gp = (gw >= 2 && gw <= 40) ? gw : std::min<int64_t>(nsm, ceil_div(rows, (int64_t)256));
    const int64_t r = gp + 4;
    if (r > nsm - 16) return 0;
    const double t_gemm = 2.0 * (double)(m - bf) * (double)(w - bf2) * (double)NB / (33e12 * (double)(nsm - r) / nsm);
    const double t_side = (double)(bf2 - bf) * 4.5e-6;
    return t_gemm <= reserve_ratio * t_side ? (int)r : 0;
  };

  DS_TRY(factor_outer(0, std::min<int64_t>(NB, w)));
  // debug timeline (DENSOLVE_LU_TIMELINE=1): an event on the main stream per outer panel
  // plus host enqueue times; printed at the end
  const bool timeline = getenv("DENSOLVE_LU_TIMELINE") != nullptr;
  std::vector<cudaEvent_t> tev;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> side_ev;  // look-ahead panel factorizations
  std::vector<double> thost;
  auto host_us = [] {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
  };
  auto mark = [&] {
    if (!timeline) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, ctx->stream);
    tev.push_back(e);
    thost.push_back(host_us());
  };
  mark();
  for (int64_t kb = 0; kb < w; kb += NB) {
    mark();
    const int64_t bf = std::min<int64_t>(kb + NB, w);
    // swaps of the whole outer panel on the columns outside it.  The L columns
    // [0, kb) are never read again by the factorization, so with look-ahead
    // their swaps run on the low-priority aux stream, overlapped with the GEMMs.
    SwapPlan op = sp_out;
    if (lookahead && kb > 0) {  // per-panel plan buffer: the aux stream reads it later
      const int64_t kq = kb / NB;
      op.pairs = left_pairs + (size_t)kq * 8 * NB;
      op.np = left_np + kq * 64;
    }
    if (kb > 0 || bf < w) DS_TRY(laswp_plan(ctx, kb, bf, d_piv, op));
    if (lookahead && kb > 0) {
      DS_CUDA(cudaEventRecord(ctx->ev_c, ctx->stream));
      DS_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_c, 0));
      cudaStream_t main = ctx->stream;
      ctx->stream = ctx->aux;
      const int rc = laswp_apply<T>(ctx, W, ld, 0, kb, op);
      ctx->stream = main;
      DS_TRY(rc);
    } else {
      DS_TRY(laswp_apply<T>(ctx, W, ld, 0, kb, op));
    }
    if (bf >= w) break;
    const int64_t bf2 = std::min<int64_t>(bf + NB, w);
    // the look-ahead columns [bf, bf2) get their swaps and update first: that is the
    // only work between this panel and the next panel's factorization
    DS_TRY(laswp_apply<T>(ctx, W, ld, bf, bf2, op));
    DS_TRY(outer_update(kb, bf, bf, bf2, 0, true));  // the look-ahead columns: on the panel chain
    if (lookahead) {
      DS_CUDA(cudaEventRecord(ctx->ev_a, ctx->stream));
      DS_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_a, 0));
      cudaStream_t main = ctx->stream;
      ctx->stream = ctx->side;
      cudaEvent_t s0 = nullptr, s1 = nullptr;
      if (timeline) {
        cudaEventCreate(&s0);
        cudaEventCreate(&s1);
        cudaEventRecord(s0, ctx->side);
      }
      const int rc = factor_outer(bf, bf2);
      if (timeline) {
        cudaEventRecord(s1, ctx->side);
        side_ev.push_back({s0, s1});
      }
      ctx->stream = main;
      DS_TRY(rc);
      DS_CUDA(cudaEventRecord(ctx->ev_b, ctx->side));
      // the rest of the trailing matrix (disjoint columns) overlaps the next panel
      DS_TRY(laswp_apply<T>(ctx, W, ld, bf2, w, op));
      DS_TRY(outer_update(kb, bf, bf2, w, side_reserve(bf, bf2)));
      DS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_b, 0));
    } else {
      DS_TRY(laswp_apply<T>(ctx, W, ld, bf2, w, op));
      DS_TRY(outer_update(kb, bf, bf2, w, 0));
      DS_TRY(factor_outer(bf, bf2));
    }
  }
  mark();
  if (timeline && tev.size() > 1) {
    cudaEventSynchronize(tev.back());
    const double hend = host_us();
    std::vector<std::pair<float, int>> d;
    float tot = 0;
    for (size_t k = 1; k < tev.size(); ++k) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tev[k - 1], tev[k]);
      d.push_back({ms, (int)k - 1});
      tot += ms;
    }
    std::sort(d.begin(), d.end(), [](auto& x, auto& y) { return x.first > y.first; });
    fprintf(stderr, "[lu timeline] n=%lld steps=%zu device %.2f ms, host enqueue %.2f ms, host total %.2f ms; slowest:",
            (long long)w, d.size(), tot, (thost.back() - thost.front()) / 1e3, (hend - thost.front()) / 1e3);
    for (size_t k = 0; k < std::min<size_t>(6, d.size()); ++k)
      fprintf(stderr, " #%d %.2f ms (enq at %.2f ms)", d[k].second, d[k].first,
              (thost[d[k].second] - thost.front()) / 1e3);
    fprintf(stderr, "\n[lu timeline] per outer panel (ms):");
    for (size_t k = 1; k < tev.size(); ++k) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tev[k - 1], tev[k]);
      fprintf(stderr, " %.2f", ms);
    }
    fprintf(stderr, "\n[lu timeline] look-ahead panel factorization on the side stream (ms):");
    for (auto& pe : side_ev) {
      float ms = 0;
      cudaEventElapsedTime(&ms, pe.first, pe.second);
      fprintf(stderr, " %.2f", ms);
      cudaEventDestroy(pe.first);
      cudaEventDestroy(pe.second);
    }
    fprintf(stderr, "\n");
    for (auto e : tev) cudaEventDestroy(e);
  }
  if (lookahead) {
    DS_CUDA(cudaEventRecord(ctx->ev_c, ctx->aux));
    DS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_c, 0));
    DS_CUDA(cudaFreeAsync(left_pairs, ctx->stream));
    DS_CUDA(cudaFreeAsync(left_np, ctx->stream));
  }
  return DS_OK;
}
// Load (lazy module loading) every kernel the block-cyclic LU shards launch, before any shard
// waits on a peer (see ds_shard.cu): a first launch that loads a module waits for the device.
int preload_lu_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {(const void*)lu_panel_smem_kernel<double, 2>, (const void*)lu_panel_smem_kernel<double, 4>,
                       (const void*)lu_panel_smem_kernel<float, 2>,  (const void*)lu_panel_smem_kernel<float, 4>,
                       (const void*)lu_panel_warp_kernel<double>,     (const void*)lu_panel_warp_kernel<float>,
                       (const void*)lu_panel_global_kernel<double>,   (const void*)lu_panel_global_kernel<float>,
                       (const void*)laswp_plan_kernel,                (const void*)laswp_plan_serial_kernel,
                       (const void*)laswp_gather_kernel<double>,      (const void*)laswp_gather_kernel<float>};
  for (const void* f : fns) DS_CUDA(cudaFuncGetAttributes(&a, f));
  return DS_OK;
}
template int lu_factor_impl<double>(ds_ctx*, int64_t, int64_t, double*, int64_t, int64_t, int64_t*, int8_t*);
template int lu_factor_impl<float>(ds_ctx*, int64_t, int64_t, float*, int64_t, int64_t, int64_t*, int8_t*);

// apply swaps piv[k0..k1) (absolute rows) to ncols columns of W
template <typename T>
int laswp_range(ds_ctx* ctx, T* W, int64_t ld, int64_t ncols, int64_t k0, int64_t k1, const int64_t* d_piv) {
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, sizeof(int64_t) * 8 * (size_t)(k1 - k0) + 1024, &ws));
  Carver cv{(char*)ws};
  SwapPlan sp;
  sp.pairs = cv.take<int64_t>(sizeof(int64_t) * 8 * (size_t)(k1 - k0));
  sp.np = cv.take<int>(64);
  DS_TRY(laswp_plan(ctx, k0, k1, d_piv, sp));
  return laswp_apply<T>(ctx, W, ld, 0, ncols, sp);
}
template int laswp_range<double>(ds_ctx*, double*, int64_t, int64_t, int64_t, int64_t, const int64_t*);
template int laswp_range<float>(ds_ctx*, float*, int64_t, int64_t, int64_t, int64_t, const int64_t*);

// ----------------------------------------------------------------------------
// pivots -> gather permutation: idx = apply_pivots(piv, arange(n))  (core.py:94-100)
// ----------------------------------------------------------------------------
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
#ifndef DS_TRSV_DEPTH
#define DS_TRSV_DEPTH 3
#endif
constexpr int kTrsvDepth = DS_TRSV_DEPTH;  // earlier blocks in flight per CTA during the fold

// TRANS (upper only): solve with U = M^T, i.e. U[i,j] = M[j + i*ld] (the
// backward sweep of cholesky_solve on L^T, direct.py:166-171, without forming L^T).
//
// One CTA per 64-row block, blocks taken in sweep order from an atomic ticket (a CTA
// only ever waits on blocks with smaller tickets, which are resident or done).
//   * Unknowns are published as LL words (32 data bits + flag per 8-byte word, the
//     buffer zeroed per launch): a reader polls the words themselves, so no fence and
//     no counter round trip sits on the chain.
//   * Before any wait a CTA stages its diagonal tile and the tile of the preceding
//     block in shared memory, and inverts the diagonal tile in fp64 (one thread per
//     column).  Then it folds in all earlier blocks (batched LL reads per block, next
//     block's matrix values prefetched), the preceding block from shared memory as soon
//     as its unknowns appear, and finishes with y = D^-1 (b - sums): one 64 x 64 product.
//   * Summation order is fixed (each column always goes to the same warp / lane, in
//     sweep order): results are bitwise reproducible run to run.  They differ from the
//     reference's row-by-row substitution (direct.py:123-152) by rounding only.
template <typename T, bool TRANS>
__device__ __forceinline__ void trsv_stage_tile(T (*tile)[kTrsvNB + 1], const T* __restrict__ M, int64_t ld,
                                                int64_t r0, int nr, int64_t c0, int nc) {
  // tile[r][c] = U[r0 + r, c0 + c]
  for (int e = threadIdx.x; e < kTrsvNB * kTrsvNB; e += kTrsvThreads) {
    const int fast = e % kTrsvNB, slow = e / kTrsvNB;
    const int r = TRANS ? slow : fast, c = TRANS ? fast : slow;
    if (r < nr && c < nc) tile[r][c] = TRANS ? M[(c0 + c) + (r0 + r) * ld] : M[(r0 + r) + (c0 + c) * ld];
  }
}

// LL words: each 8-byte word carries 32 data bits and a 32-bit flag (1; the buffer is zeroed
// per launch), so a reader polling the word needs no fence: fp64 values use two words.
template <typename T>
__device__ __forceinline__ void trsv_ll_write(uint64_t* p, T v) {
  uint64_t bits = sizeof(T) == 8 ? (uint64_t)__double_as_longlong((double)v) : (uint64_t)__float_as_uint((float)v);
  const uint64_t w0 = (1ull << 32) | (bits & 0xffffffffull);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;\n" ::"l"(p), "l"(w0) : "memory");
  if (sizeof(T) == 8) {
    const uint64_t w1 = (1ull << 32) | (bits >> 32);
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;\n" ::"l"(p + 1), "l"(w1) : "memory");
  }
}
template <typename T>
__device__ __forceinline__ T trsv_ll_read(const uint64_t* p) {
  uint64_t w0, w1 = 0;
  do {
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w0) : "l"(p) : "memory");
  } while ((w0 >> 32) != 1u);
  if (sizeof(T) == 8) {
    do {
      asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w1) : "l"(p + 1) : "memory");
    } while ((w1 >> 32) != 1u);
    return (T)__longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
  }
  return (T)__uint_as_float((unsigned)(w0 & 0xffffffffull));
}


template <typename T, bool LOWER, bool UNIT, bool TRANS = false>
__global__ void __launch_bounds__(kTrsvThreads)
    trsv_kernel(int64_t n, const T* __restrict__ M, int64_t ld, const T* __restrict__ rhs,
                T* out, int* ticket, uint64_t* __restrict__ ll) {
  extern __shared__ __align__(16) unsigned char trsv_smem[];
  T (*dg)[kTrsvNB + 1] = reinterpret_cast<T (*)[kTrsvNB + 1]>(trsv_smem);
  T (*pv)[kTrsvNB + 1] = dg + kTrsvNB;  // tile of the previous block in the sweep
  constexpr int NW = kTrsvThreads / 32;
  __shared__ int s_blk;
  __shared__ double part[NW][kTrsvNB];
  __shared__ T xs[kTrsvNB];
  __shared__ double rv[kTrsvNB];
  __shared__ double rdiag[kTrsvNB];
  double (*dinv)[kTrsvNB + 1] = reinterpret_cast<double (*)[kTrsvNB + 1]>(pv + kTrsvNB);
  const int64_t nblk = ceil_div(n, kTrsvNB);
  if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1);
  __syncthreads();
  const int64_t t = s_blk;
  const int64_t bi = LOWER ? t : nblk - 1 - t;
  const int64_t r0 = bi * kTrsvNB;
  const int nr = (int)min((int64_t)kTrsvNB, n - r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  trsv_stage_tile<T, TRANS>(dg, M, ld, r0, nr, r0, nr);
  int64_t cprev = 0;
  int ncprev = 0;
  if (t > 0) {
    const int64_t bj = LOWER ? t - 1 : nblk - t;
    cprev = bj * kTrsvNB;
    ncprev = (int)min((int64_t)kTrsvNB, n - cprev);
    trsv_stage_tile<T, TRANS>(pv, M, ld, r0, nr, cprev, ncprev);
  }
  // rhs of my row (threads < 64), loaded before any wait
  const T bme = threadIdx.x < nr ? rhs[r0 + threadIdx.x] : T(0);
  // D^-1 of the diagonal block in fp64 (unit: the stored diagonal is ignored), one thread
  // per column, before any wait: off the critical path of the sweep
  __syncthreads();
  if (threadIdx.x < kTrsvNB) rdiag[threadIdx.x] = (UNIT || threadIdx.x >= nr) ? 1.0 : 1.0 / (double)dg[threadIdx.x][threadIdx.x];
  __syncthreads();
  if (threadIdx.x < nr) {
    const int j = threadIdx.x;
    if (LOWER) {
      for (int i = 0; i < nr; ++i) {
        double v = 0.0;
        if (i >= j) {
          v = i == j ? 1.0 : 0.0;
          for (int k = j; k < i; ++k) v = fma(-(double)dg[i][k], dinv[k][j], v);
          v *= rdiag[i];
        }
        dinv[i][j] = v;
      }
    } else {
      for (int i = nr - 1; i >= 0; --i) {
        double v = 0.0;
        if (i <= j) {
          v = i == j ? 1.0 : 0.0;
          for (int k = i + 1; k <= j; ++k) v = fma(-(double)dg[i][k], dinv[k][j], v);
          v *= rdiag[i];
        }
        dinv[i][j] = v;
      }
    }
  }
  if (threadIdx.x < kTrsvNB) {  // padding rows / columns of a partial block stay zero
    for (int i = nr; i < kTrsvNB; ++i) dinv[i][threadIdx.x] = 0.0;
    if (threadIdx.x >= nr)
      for (int i = 0; i < kTrsvNB; ++i) dinv[i][threadIdx.x] = 0.0;
  }
  // non-TRANS: thread owns rows 2 lane, 2 lane + 1; warp owns the columns c = warp (mod NW)
  // TRANS:     thread owns the columns c = lane (mod 32); warp owns rows warp + NW j
  const int ra = 2 * lane, rb = 2 * lane + 1;
  double a0 = 0.0, a1 = 0.0;
  double at[kTrsvNB / NW];
#pragma unroll
  for (int j = 0; j < kTrsvNB / NW; ++j) at[j] = 0.0;
  // blocks solved before the preceding one, in sweep order.  Per block, a warp reads the
  // unknowns it needs as LL words in ONE batch (spinning only while that block is still
  // being solved: no per-block handshake, no fence anywhere on the chain) and the matrix
  // values of the NEXT block are loaded before the current block's unknowns are
  // validated, so HBM latency overlaps the wait.
  //   non-TRANS: warp w owns columns c0 + w + NW j (j < 8) of each block; lane j < 8 reads
  //              unknown j and broadcasts it; the thread's rows are 2 lane, 2 lane + 1.
  //   TRANS:     lane l owns columns c0 + l, c0 + l + 32; warp w owns rows w + NW j.
  if (t > 1) {
    auto block_col0 = [&](int64_t sidx) -> int64_t { return (LOWER ? sidx : nblk - 1 - sidx) * kTrsvNB; };
    constexpr int CPW = kTrsvNB / NW;  // columns per warp per block (non-TRANS)
    // kTrsvDepth blocks in flight per CTA: block sidx lives in slot sidx % kTrsvDepth, its
    // matrix values and LL words issued kTrsvDepth blocks ahead (static slot indices: the
    // loop is unrolled by the depth)
    // kept in T until the FMA: a conversion right after the load would wait for it and
    // serialise the prefetch (fp32)
    T mv[kTrsvDepth][2 * CPW];
    uint64_t xw0[kTrsvDepth][2], xw1[kTrsvDepth][2];
    auto issue = [&](int64_t sidx, T (&m)[2 * CPW], uint64_t (&w0)[2], uint64_t (&w1)[2]) {
      const int64_t c0 = block_col0(sidx);
      const int nc = (int)min((int64_t)kTrsvNB, n - c0);
      if (!TRANS) {
#pragma unroll
        for (int j = 0; j < CPW; ++j) {
          const int c = warp + NW * j;
          const T* col = M + (c0 + c) * ld + r0;
          m[2 * j] = (c < nc && ra < nr) ? col[ra] : T(0);
          m[2 * j + 1] = (c < nc && rb < nr) ? col[rb] : T(0);
        }
        const int c = warp + NW * (lane & (CPW - 1));
        const uint64_t* p = ll + 2 * (c0 + min(c, nc - 1));
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w0[0]) : "l"(p) : "memory");
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w1[0]) : "l"(p + 1) : "memory");
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = lane + 32 * h;
#pragma unroll
          for (int j = 0; j < CPW; ++j) {
            const int r = warp + NW * j;
            m[h * CPW + j] = (c < nc && r < nr) ? M[(c0 + c) + (r0 + r) * ld] : T(0);
          }
          const uint64_t* p = ll + 2 * (c0 + min(c, nc - 1));
          asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w0[h]) : "l"(p) : "memory");
          asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w1[h]) : "l"(p + 1) : "memory");
        }
      }
    };
    auto validate = [&](int64_t sidx, int h, uint64_t (&w0)[2], uint64_t (&w1)[2]) -> double {
      // re-poll the LL words of my unknown until both carry the flag
      const int64_t c0 = block_col0(sidx);
      const int nc = (int)min((int64_t)kTrsvNB, n - c0);
      const int c = TRANS ? lane + 32 * h : warp + NW * (lane & (CPW - 1));
      const uint64_t* p = ll + 2 * (c0 + min(c, nc - 1));
      while ((w0[h] >> 32) != 1u)
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w0[h]) : "l"(p) : "memory");
      if (sizeof(T) == 8) {
        while ((w1[h] >> 32) != 1u)
          asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w1[h]) : "l"(p + 1) : "memory");
        return __longlong_as_double((long long)((w1[h] << 32) | (w0[h] & 0xffffffffull)));
      }
      return (double)__uint_as_float((unsigned)(w0[h] & 0xffffffffull));
    };
    const int64_t nfold = t - 1;  // blocks folded here (all but the preceding one)
#pragma unroll
    for (int d = 0; d < kTrsvDepth; ++d)
      if (d < nfold) issue(d, mv[d], xw0[d], xw1[d]);
    for (int64_t s0 = 0; s0 < nfold; s0 += kTrsvDepth) {
#pragma unroll
      for (int d = 0; d < kTrsvDepth; ++d) {
        const int64_t sidx = s0 + d;
        if (sidx < nfold) {
          // the slot is consumed in place and refilled after its FMAs (a copy out of the slot
          // before the refill waited on the slot's loads)
          T (&cur)[2 * CPW] = mv[d];
          uint64_t (&cw0)[2] = xw0[d];
          uint64_t (&cw1)[2] = xw1[d];
          if (!TRANS) {
            const double xmine = validate(sidx, 0, cw0, cw1);
#pragma unroll
            for (int j = 0; j < CPW; ++j) {
              const double xv = __shfl_sync(0xffffffffu, xmine, j);
              a0 = fma((double)cur[2 * j], xv, a0);
              a1 = fma((double)cur[2 * j + 1], xv, a1);
            }
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double xv = validate(sidx, h, cw0, cw1);
#pragma unroll
              for (int j = 0; j < CPW; ++j) at[j] = fma((double)cur[h * CPW + j], xv, at[j]);
            }
          }
          if (sidx + kTrsvDepth < nfold) issue(sidx + kTrsvDepth, mv[d], xw0[d], xw1[d]);  // refill the slot
        }
      }
    }
  }
  if (t > 0) {  // the preceding block: its unknowns arrive as LL words, then its staged tile
    if (threadIdx.x < ncprev) xs[threadIdx.x] = trsv_ll_read<T>(ll + 2 * (cprev + threadIdx.x));
    __syncthreads();
    if (!TRANS) {
      for (int c = warp; c < ncprev; c += NW) {
        const double xv = (double)xs[c];
        if (ra < nr) a0 = fma((double)pv[ra][c], xv, a0);
        if (rb < nr) a1 = fma((double)pv[rb][c], xv, a1);
      }
    } else {
      for (int c = lane; c < ncprev; c += 32) {
        const double xv = (double)xs[c];
#pragma unroll
        for (int j = 0; j < kTrsvNB / NW; ++j) {
          const int r = warp + NW * j;
          if (r < nr) at[j] = fma((double)pv[r][c], xv, at[j]);
        }
      }
    }
  }
  if (!TRANS) {
    part[warp][ra] = a0;
    part[warp][rb] = a1;
  } else {
#pragma unroll
    for (int j = 0; j < kTrsvNB / NW; ++j) {
      const double v = warp_sum(at[j]);
      if (lane == 0) part[0][warp + NW * j] = v;
    }
  }
  __syncthreads();
  // r = b - (off-diagonal sums) in fp64, then y = D^-1 r with the inverse computed before
  // any wait: the chain step is one 64 x 64 product from shared memory
  if (threadIdx.x < kTrsvNB) {
    double off = 0.0;
    for (int q = 0; q < (TRANS ? 1 : NW); ++q) off += part[q][threadIdx.x];
    rv[threadIdx.x] = threadIdx.x < nr ? (double)bme - off : 0.0;
  }
  __syncthreads();
  {
    const int i = threadIdx.x % kTrsvNB, g = threadIdx.x / kTrsvNB;
    constexpr int KG = kTrsvNB / (kTrsvThreads / kTrsvNB);
    double p = 0.0;
#pragma unroll
    for (int k = g * KG; k < (g + 1) * KG; ++k) p = fma(dinv[i][k], rv[k], p);
    part[g][i] = p;
  }
  __syncthreads();
  if (threadIdx.x < nr) {
    const int i = threadIdx.x;
    double y = part[0][i];
    for (int g = 1; g < kTrsvThreads / kTrsvNB; ++g) y += part[g][i];
    const T yt = (T)y;
    // the next block's critical path reads these LL words (no fence, no counter round trip)
    trsv_ll_write<T>(ll + 2 * (r0 + i), yt);
    out[r0 + i] = yt;
  }
}

template <typename T>
static int trsv_smem_bytes() {  // diagonal tile + previous block's tile (T) + D^-1 (fp64)
  return (int)(2 * kTrsvNB * (kTrsvNB + 1) * sizeof(T) + kTrsvNB * (kTrsvNB + 1) * sizeof(double));
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
int trsv_upper_trans_launch(ds_ctx* ctx, int64_t n, const T* M, int64_t ld, const T* rhs, T* out,
                            char* scratch) {
  if (n == 0) return DS_OK;
  const int64_t nblk = ceil_div(n, kTrsvNB);
  int* ticket = (int*)scratch;
  uint64_t* ll = (uint64_t*)(scratch + 512);
  DS_CUDA(cudaMemsetAsync(scratch, 0, trsv_scratch_bytes(n), ctx->stream));
  const int sm = trsv_smem_bytes<T>();
  DS_CUDA(cudaFuncSetAttribute(trsv_kernel<T, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  trsv_kernel<T, false, false, true><<<(unsigned)nblk, kTrsvThreads, sm, ctx->stream>>>(
      n, M, ld, rhs, out, ticket, ll);
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}
template int trsv_upper_trans_launch<double>(ds_ctx*, int64_t, const double*, int64_t, const double*,
                                             double*, char*);
template int trsv_upper_trans_launch<float>(ds_ctx*, int64_t, const float*, int64_t, const float*,
                                            float*, char*);

template <typename T>
int trsv_launch(ds_ctx* ctx, int64_t n, const T* M, int64_t ld, const T* rhs, T* out, bool lower,
                bool unit, char* scratch) {
  if (n == 0) return DS_OK;
  const int64_t nblk = ceil_div(n, kTrsvNB);
  int* ticket = (int*)scratch;
  uint64_t* ll = (uint64_t*)(scratch + 512);
  DS_CUDA(cudaMemsetAsync(scratch, 0, trsv_scratch_bytes(n), ctx->stream));
  const int sm = trsv_smem_bytes<T>();
  if (lower && unit) {
    DS_CUDA(cudaFuncSetAttribute(trsv_kernel<T, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    trsv_kernel<T, true, true><<<(unsigned)nblk, kTrsvThreads, sm, ctx->stream>>>(n, M, ld, rhs, out, ticket, ll);
  } else if (lower) {
    DS_CUDA(cudaFuncSetAttribute(trsv_kernel<T, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    trsv_kernel<T, true, false><<<(unsigned)nblk, kTrsvThreads, sm, ctx->stream>>>(n, M, ld, rhs, out, ticket, ll);
  } else {
    DS_CUDA(cudaFuncSetAttribute(trsv_kernel<T, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    trsv_kernel<T, false, false><<<(unsigned)nblk, kTrsvThreads, sm, ctx->stream>>>(n, M, ld, rhs, out, ticket, ll);
  }
  count_launch(ctx);
  DS_CHECK_LAUNCH();
  return DS_OK;
}

template int trsv_launch<double>(ds_ctx*, int64_t, const double*, int64_t, const double*, double*,
                                 bool, bool, char*);
template int trsv_launch<float>(ds_ctx*, int64_t, const float*, int64_t, const float*, float*, bool,
                                bool, char*);

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
int lu_solve_impl(ds_ctx* ctx, int64_t n, const T* LU, int64_t ld, const int* h_idx, const T* b, T* x) {
  void* ws = nullptr;
  const size_t need = (size_t)n * (sizeof(int) + sizeof(T) * 2) + trsv_scratch_bytes(n) + 8 * 256;
  DS_TRY(ctx_workspace(ctx, need, &ws));
  Carver cv{(char*)ws};
  int* idx = cv.take<int>((size_t)n * sizeof(int));
  T* pb = cv.take<T>((size_t)n * sizeof(T));
  T* y = cv.take<T>((size_t)n * sizeof(T));
  char* scratch = cv.take<char>(trsv_scratch_bytes(n));
  DS_CUDA(cudaMemcpyAsync(idx, h_idx, (size_t)n * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  gather_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, ctx->stream>>>(
      n, idx, b, pb);
  count_launch(ctx, 1);
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
  DS_ENTER(ctx);
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
  DS_DISPATCH(dtype, T, rc = lu_factor_impl<T>(ctx, n, n, (T*)A, lda, nb, d_piv, d_zero));
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
  DS_ENTER(ctx);
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
  DS_DISPATCH(dtype, T, rc = lu_factor_impl<T>(ctx, n, n, (T*)A, lda, nb, d_piv, d_zero));
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
  DS_ENTER(ctx);
  if (n == 0) return DS_OK;
  // gather permutation idx = apply_pivots(piv, arange(n)) (core.py:94-100): the swap
  // sequence is inherently serial, so it is composed here on the host (n int swaps)
  // into the context's pinned buffer and shipped with one copy
  int* h_idx = nullptr;
  DS_TRY(ctx_hostbuf(ctx, (size_t)n * sizeof(int), (void**)&h_idx));
  for (int64_t i = 0; i < n; ++i) h_idx[i] = (int)i;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t p = h_piv[k];
    if (p < 0 || p >= n) {
      set_error("lu_solve: pivot %lld at row %lld out of range", (long long)p, (long long)k);
      return DS_EINVAL;
    }
    if (p != k) std::swap(h_idx[k], h_idx[p]);
  }
  int rc = DS_OK;
  DS_DISPATCH(dtype, T, rc = lu_solve_impl<T>(ctx, n, (const T*)LU, lda, h_idx, (const T*)b, (T*)x));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));  // also keeps h_idx alive until the copy ran
  return rc;
}

int ds_forward_substitution(ds_ctx* ctx, int dtype, int64_t n, const void* L, int64_t ldl,
                            const void* b, void* y, int unit_diagonal, int64_t* h_bad_row) {
  DS_ENTER(ctx);
  if (h_bad_row) *h_bad_row = -1;
  if (n == 0) return DS_OK;
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, trsv_scratch_bytes(n) + 512, &ws));
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
  DS_ENTER(ctx);
  if (h_bad_row) *h_bad_row = -1;
  if (n == 0) return DS_OK;
  void* ws = nullptr;
  DS_TRY(ctx_workspace(ctx, trsv_scratch_bytes(n) + 512, &ws));
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
