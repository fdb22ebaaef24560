// ds_comm.cu — NCCL inside the library for the row-sharded Krylov iterations.
//
// The row-sharded CG exchanges per iteration an all-gather of p
// (n_loc values per rank) and all-gathers of the per-rank reduction records
// (p'Ap, then (r'r, scale, ssq)); every rank combines the records in rank order
// on the device (ds_dist.cu), so all ranks take identical decisions.  Driving
// those collectives from Python costs ~0.2 ms of host time per iteration; here a
// whole chunk of iterations is enqueued from C++ on the context's stream: four
// kernels + three ncclAllGather per iteration, no host synchronisation.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"): inside a torch process
// that resolves to the NCCL torch already loaded; nccl.h supplies the types.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "ds_common.cuh"
#include "ds_kernels.cuh"

struct ds_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
};

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

int nccl_load() {
  std::call_once(g_nccl_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
    if (g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllGather) g_nccl.h = h;
  });
  if (!g_nccl.h) {
    ds::set_error("NCCL (libnccl.so.2) could not be loaded");
    return DS_ECUDA;
  }
  return DS_OK;
}

#define DS_NCCL(call)                                                                       \
  do {                                                                                      \
    const ncclResult_t _r = (call);                                                         \
    if (_r != ncclSuccess) {                                                                \
      ds::set_error("NCCL error %d (%s) at %s:%d", (int)_r,                                 \
                    g_nccl.GetErrorString ? g_nccl.GetErrorString(_r) : "?", __FILE__, __LINE__); \
      return DS_ECUDA;                                                                      \
    }                                                                                       \
  } while (0)

}  // namespace

extern "C" {

int ds_comm_unique_id(unsigned char* out) {
  DS_TRY(nccl_load());
  ncclUniqueId id;
  DS_NCCL(g_nccl.GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == DS_COMM_ID_BYTES, "ncclUniqueId size");
  memcpy(out, &id, sizeof id);
  return DS_OK;
}

int ds_comm_create(ds_ctx* ctx, int nranks, int rank, const unsigned char* id, ds_comm** out) {
  DS_ENTER(ctx);
  DS_TRY(nccl_load());
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    ds::set_error("bad communicator rank %d of %d", rank, nranks);
    return DS_EINVAL;
  }
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  ds_comm* c = new ds_comm();
  c->rank = rank;
  c->nranks = nranks;
  const ncclResult_t r = g_nccl.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    ds::set_error("ncclCommInitRank failed: %s", g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
    return DS_ECUDA;
  }
  *out = c;
  return DS_OK;
}

int ds_comm_destroy(ds_comm* c) {
  if (!c) return DS_OK;
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  delete c;
  return DS_OK;
}

int ds_cg_shard_iterations(ds_ctx* ctx, ds_comm* comm, int dtype, int64_t n_loc, int64_t n, const void* A_blk,
                           int64_t lda, void* full, void* x, void* r, void* p, void* Ap, double* d_state,
                           double* d_hist, double* d_pap, double* d_pap_all, double* d_parts, double* d_rparts,
                           double tol, int64_t cap, int64_t k0, int64_t k1) {
  DS_ENTER(ctx);
  if (!comm) {
    ds::set_error("null communicator");
    return DS_EINVAL;
  }
  const ncclDataType_t vt = dtype == DS_F64 ? ncclFloat64 : ncclFloat32;
  const int G = comm->nranks;
  for (int64_t k = k0; k < k1; ++k) {
    DS_NCCL(g_nccl.AllGather(p, full, (size_t)n_loc, vt, comm->comm, ctx->stream));        // p -> all ranks
    DS_TRY(ds_gemv(ctx, dtype, n_loc, n, A_blk, lda, full, Ap));                             // my rows of A p
    DS_TRY(ds_dot_dev(ctx, dtype, n_loc, p, Ap, d_pap));                                      // my p'Ap
    DS_NCCL(g_nccl.AllGather(d_pap, d_pap_all, 1, ncclFloat64, comm->comm, ctx->stream));
    DS_TRY(ds_cg_shard_update(ctx, dtype, n_loc, G, d_pap_all, d_state, k, x, r, p, Ap, d_parts));
    DS_NCCL(g_nccl.AllGather(d_parts, d_rparts, 3, ncclFloat64, comm->comm, ctx->stream));
    DS_TRY(ds_cg_shard_finish(ctx, dtype, n_loc, G, d_rparts, d_state, k, r, p, d_hist, tol, cap));
  }
  return DS_OK;
}

}  // extern "C"
