// ds_kernels.cuh — internal launchers shared by the op contract and the solvers.
#pragma once
#include "ds_common.cuh"

namespace ds {

// ---- GEMV ------------------------------------------------------------------
// y = A x for a column-major m x n matrix, streamed once from HBM.
// Stage 1 (ds_colstream_mv_kernel): grid (row tiles, column chunks); each CTA streams an
//   (R x C) tile with 128-bit loads, x chunk staged in shared memory by a bulk
//   async copy (cp.async.bulk, the 1-D TMA path), fp64 accumulation.
// Stage 2 (ds_colstream_reduce_kernel): sums the chunk partials in fixed chunk order (bitwise
//   deterministic) and applies a fused epilogue.
enum GemvEpi : int {
  EPI_STORE = 0,      // y = A x
  EPI_DOT = 1,        // y = A x ; block partial of dot(v, y) -> part (CG p'Ap)
  EPI_RESID = 2,      // y = b - A x (axpy(-1, Ax, b)); block partial (ssq of y, plain sum y^2)
  EPI_AXPY_INTO = 3,  // y = y + (A x)   (GMRES x += V y, krylov.py:167)
  EPI_DOT2 = 4,       // y = A x ; block partials of dot(v, y) -> red[blk], dot(y, y) -> red[nblk + blk]
                      //   (BiCGSTAB t's and t't, krylov.py:230-231)
  EPI_PARTIAL = 5,    // stage 1 only: the chunk partials stay in `part` for a consumer
                      //   kernel that sums them itself (GMRES cluster orthogonalisation)
};

// Device-side loop gate: solver kernels of iteration k return immediately once
// *stop_it <= k, so the host can enqueue iterations speculatively and only
// synchronise once per chunk (device-side convergence control).
struct Gate {
  const int64_t* stop_it;
  int64_t k;
};
__device__ __forceinline__ bool gated(const Gate& g) {
  return g.stop_it != nullptr && *((volatile const int64_t*)g.stop_it) <= g.k;
}

// Programmatic dependent launch (PDL): a kernel launched with the programmatic
// stream-serialization attribute may start while its predecessor still runs; it
// must wait here before touching the predecessor's results (no-op without PDL).
// launch_dependents lets the NEXT kernel start launching (it still waits for this
// grid's completion at its own pdl_wait).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

struct GemvPlan {
  int64_t m, n;
  int rows_per_cta;  // multiple of 32*VEC
  int64_t chunk;     // columns per CTA
  int64_t nchunks;
  int64_t rowtiles;
  size_t part_bytes;  // workspace for partials
};

GemvPlan gemv_plan(ds_ctx* ctx, int64_t m, int64_t n, size_t elem);

// Stage 1 only, launched with the PDL attribute (the GMRES cluster path: the
// orthogonalisation kernel that follows sums the partials itself).
template <typename T>
int gemv_partial_pdl_launch(ds_ctx* ctx, const GemvPlan& p, const T* A, int64_t lda, const T* x, double* part,
                            Gate stop);
// Wide-CTA stage 1 for small matrices (~one CTA per SM, 4 column groups per CTA, one
// partial per row per CTA), launched with the PDL attribute (the GMRES cluster path).
GemvPlan gemv_wide_plan(ds_ctx* ctx, int64_t m, int64_t n, size_t elem);
template <typename T>
int gemv_partial_wide_pdl_launch(ds_ctx* ctx, const GemvPlan& p, const T* A, int64_t lda, const T* x, double* part,
                                 Gate stop);
// Launch stage 1 + 2.  `part` must have plan.part_bytes; `red` (for EPI_DOT /
// EPI_RESID) receives per-block reduction partials (see reduce_blocks()).
template <typename T>
int gemv_launch(ds_ctx* ctx, const GemvPlan& p, const T* A, int64_t lda, const T* x, T* y,
                double* part, GemvEpi epi, const T* v, double* red, int* red_blocks,
                Gate gate = Gate{nullptr, 0});

// ---- deterministic two-stage reductions of per-block partials ----------------
// Each reduction producer writes `nblk` partial records; consumers read them
// back in block order.  Layouts:
//   dot:  red[blk]                         (plain sums)
//   ssq:  red[2*blk], red[2*blk+1]        (scale, ssq)
__device__ __forceinline__ double reduce_sum_partials(const double* red, int nblk, double* smem) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) s += red[i];
  return block_sum(s, smem);
}

// ---- level-1 -----------------------------------------------------------------
int reduce_grid(ds_ctx* ctx, int64_t n);  // blocks used by reduction kernels

template <typename T>
int dot_launch(ds_ctx* ctx, int64_t n, const T* x, const T* y, double* red, int* nblk);
template <typename T>
int ssq_launch(ds_ctx* ctx, int64_t n, const T* x, double* red, int* nblk);
// final stage: out[0] = sum(red[0..nblk)) ; out may be device memory
int finish_sum(ds_ctx* ctx, const double* red, int nblk, double* out);
int finish_ssq(ds_ctx* ctx, const double* red, int nblk, double* out /* norm */);

template <typename T>
int axpy_launch(ds_ctx* ctx, int64_t n, double alpha, const T* x, const T* y, T* out);
template <typename T>
int scal_launch(ds_ctx* ctx, int64_t n, double alpha, const T* x, T* out);

// symmetric gate (krylov.py:41-44): red receives 2*nblk partials (maxdiff, amax)
template <typename T>
int symcheck_launch(ds_ctx* ctx, int64_t n, const T* A, int64_t lda, double* red, int* nblk);

// ---- level-3 (LU building blocks) ---------------------------------------------
template <typename T>
int gemm_launch(ds_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const T* A,
                int64_t lda, const T* B, int64_t ldb, double beta, const T* C, int64_t ldc, T* out,
                int64_t ldo);
// C -= A B on the tiles of C holding some row >= column (C square-indexed from
// its top-left corner): the lower-triangle SYRK update of the Cholesky path.
template <typename T>
int gemm_sub_lower_launch(ds_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, int64_t lda,
                          const T* B, int64_t ldb, T* C, int64_t ldc);
template <typename T>
int trsm_lower_unit_launch(ds_ctx* ctx, int64_t b, int64_t m, const T* L, int64_t ldl, const T* B,
                           int64_t ldb, T* Z, int64_t ldz);
template <typename T>
int trsm_upper_launch(ds_ctx* ctx, int64_t b, int64_t m, const T* U, int64_t ldu, const T* B,
                      int64_t ldb, T* Z, int64_t ldz);
// U01 of an outer LU panel in one launch (fp64, b = 64): for the columns [c0, c1) of W and
// the nblk 64-row blocks starting at row kb, block by block: the unit-lower TRSM of the
// block's rows, then the update of the outer panel's rows below it (the K = 64 DMMA chain of
// gemm64 from C).  Bitwise equal to the trsm_lower_unit_cols64 / gemm launch chain.
int u01_fused_launch(ds_ctx* ctx, double* W, int64_t ld, int64_t kb, int nblk, int64_t c0, int64_t c1);
template <typename T>
int ger_launch(ds_ctx* ctx, int64_t m, int64_t n, const T* A, int64_t lda, double alpha,
               const T* x, const T* y, T* out, int64_t ldo);

// ---- triangular vector solves (ds_lu.cu) -------------------------------------
// scratch: trsv_scratch_bytes(n) (ticket, done counter, 16 B of LL words per unknown)
inline size_t trsv_scratch_bytes(int64_t n) { return 512 + 16 * (size_t)(n > 0 ? n : 1); }
template <typename T>
int trsv_launch(ds_ctx* ctx, int64_t n, const T* M, int64_t ld, const T* rhs, T* out, bool lower,
                bool unit, char* scratch);
template <typename T>
int trsv_upper_trans_launch(ds_ctx* ctx, int64_t n, const T* M, int64_t ld, const T* rhs, T* out,
                            char* scratch);

// ---- lazy-loading guard of the row-sharded solver (ds_shard.cu) ----------------
int preload_sharded_kernels_blas();
int preload_dense_kernels_blas();
int preload_lu_kernels();
template <typename T>
int lu_factor_impl(ds_ctx* ctx, int64_t m, int64_t w, T* W, int64_t ld, int64_t b, int64_t* d_piv, int8_t* d_zero);
template <typename T>
int laswp_range(ds_ctx* ctx, T* W, int64_t ld, int64_t ncols, int64_t k0, int64_t k1, const int64_t* d_piv);
int preload_sharded_kernels_dist();

}  // namespace ds
