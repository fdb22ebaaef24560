// ds_context.cu — context, memory, staging and error plumbing of the C ABI.
//
// Replaces the Backend staging seam (backends.py:94-100: stage_in/stage_out,
// "preserved for a future accelerator backend") with real
// host<->device transfers, and the F-order coercion of core.py:82-87.
#include <atomic>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "ds_common.cuh"

namespace ds {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int ctx_begin(ds_ctx* ctx) {
  if (!ctx) {
    set_error("null context");
    return DS_EINVAL;
  }
  DS_CUDA(cudaSetDevice(ctx->device));
  return DS_OK;
}

int ctx_workspace(ds_ctx* ctx, size_t bytes, void** out) {
  if (bytes > ctx->ws_bytes) {
    if (ctx->ws) {
      DS_CUDA(cudaStreamSynchronize(ctx->stream));
      DS_CUDA(cudaFree(ctx->ws));
      ctx->ws = nullptr;
      ctx->ws_bytes = 0;
    }
    size_t want = bytes < (1u << 20) ? (1u << 20) : bytes;
    DS_CUDA(cudaMalloc(&ctx->ws, want));
    // the LL exchange buffers carved from it are polled before their first write
    DS_CUDA(cudaMemsetAsync(ctx->ws, 0, want, ctx->stream));
    ctx->ws_bytes = want;
  }
  *out = ctx->ws;
  return DS_OK;
}

unsigned next_ll_epoch() {
  static std::atomic<unsigned> ctr{0};
  return ++ctr;
}

int ctx_hostbuf(ds_ctx* ctx, size_t bytes, void** out) {
  if (bytes > ctx->hbuf_bytes) {
    if (ctx->hbuf) {
      DS_CUDA(cudaStreamSynchronize(ctx->stream));
      DS_CUDA(cudaFreeHost(ctx->hbuf));
      ctx->hbuf = nullptr;
      ctx->hbuf_bytes = 0;
    }
    size_t want = bytes < 4096 ? 4096 : bytes;
    DS_CUDA(cudaMallocHost(&ctx->hbuf, want));
    ctx->hbuf_bytes = want;
  }
  *out = ctx->hbuf;
  return DS_OK;
}

// C-order host matrix (row stride ld_src) staged contiguously, transposed to F-order.
template <typename T>
__global__ void transpose_kernel(const T* __restrict__ src, int64_t rows, int64_t cols,
                                 int64_t ld_src, T* __restrict__ dst, int64_t ld_dst) {
  __shared__ T tile[32][33];
  int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * ld_src + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[r + c * ld_dst] = tile[threadIdx.x][i];
  }
}

}  // namespace ds

using namespace ds;

extern "C" {

const char* ds_last_error(void) { return g_err; }

const char* ds_version(void) { return "densolve_b200 0.1.0 (sm_100a)"; }

int ds_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *out = n;
  return DS_OK;
}

int ds_ctx_create(int device, ds_ctx** out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    set_error("no CUDA device available (cudaGetDeviceCount: %s)", cudaGetErrorString(e));
    return DS_ECUDA;
  }
  if (device < 0 || device >= n) {
    set_error("device %d out of range (have %d)", device, n);
    return DS_EINVAL;
  }
  ds_ctx* c = new ds_ctx();
  c->device = device;
  DS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  DS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) {
    set_error("device %d (%s, sm_%d%d) is not Blackwell sm_100; this library is sm_100a-only",
              device, prop.name, prop.major, prop.minor);
    delete c;
    return DS_ECUDA;
  }
  c->num_sms = prop.multiProcessorCount;
  c->smem_optin = prop.sharedMemPerBlockOptin;
  DS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->own_stream = true;
  {  // keep up to 32 GiB of freed operand memory in the pool (ds_malloc / ds_free)
    cudaMemPool_t pool;
    DS_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = 32ull << 30;
    DS_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  *out = c;
  return DS_OK;
}

int ds_ctx_destroy(ds_ctx* ctx) {
  if (!ctx) return DS_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->gemm_ctr) cudaFree(ctx->gemm_ctr);
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  if (ctx->hbuf) cudaFreeHost(ctx->hbuf);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->ev_c) cudaEventDestroy(ctx->ev_c);
  if (ctx->ev_a) cudaEventDestroy(ctx->ev_a);
  if (ctx->ev_b) cudaEventDestroy(ctx->ev_b);
  delete ctx;
  return DS_OK;
}

int ds_ctx_set_stream(ds_ctx* ctx, void* stream) {
  DS_ENTER(ctx);
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (stream == nullptr) {
    if (!ctx->own_stream) {
      DS_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
    }
    return DS_OK;
  }
  if (ctx->own_stream) DS_CUDA(cudaStreamDestroy(ctx->stream));
  ctx->stream = (cudaStream_t)stream;
  ctx->own_stream = false;
  return DS_OK;
}

int ds_ctx_synchronize(ds_ctx* ctx) {
  DS_ENTER(ctx);
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

int ds_ctx_kernel_launches(ds_ctx* ctx, int64_t* out) {
  if (!ctx) return DS_EINVAL;
  *out = ctx->launches;
  return DS_OK;
}

// Device buffers come from the device's stream-ordered memory pool with an unlimited
// release threshold: a multi-GB operand freed and re-allocated between solves is
// recycled without a cudaMalloc / cudaFree round trip (no implicit device sync).
int ds_malloc(ds_ctx* ctx, size_t bytes, void** out) {
  DS_ENTER(ctx);
  *out = nullptr;
  if (bytes == 0) bytes = 16;
  DS_CUDA(cudaMallocAsync(out, bytes, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));  // the buffer is usable on any stream on return
  return DS_OK;
}

int ds_free(ds_ctx* ctx, void* p) {
  DS_ENTER(ctx);
  if (p) DS_CUDA(cudaFreeAsync(p, ctx->stream));
  return DS_OK;
}

int ds_host_alloc(size_t bytes, void** out) {
  *out = nullptr;
  DS_CUDA(cudaMallocHost(out, bytes ? bytes : 16));
  return DS_OK;
}

int ds_host_free(void* p) {
  if (p) DS_CUDA(cudaFreeHost(p));
  return DS_OK;
}

int ds_host_register(void* p, size_t bytes) {
  DS_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterDefault));
  return DS_OK;
}

int ds_host_unregister(void* p) {
  DS_CUDA(cudaHostUnregister(p));
  return DS_OK;
}

int ds_memcpy_h2d(ds_ctx* ctx, void* dst, const void* src, size_t bytes) {
  DS_ENTER(ctx);
  if (bytes == 0) return DS_OK;
  DS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

int ds_memcpy_d2h(ds_ctx* ctx, void* dst, const void* src, size_t bytes) {
  DS_ENTER(ctx);
  if (bytes == 0) return DS_OK;
  DS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

int ds_memcpy_d2d(ds_ctx* ctx, void* dst, const void* src, size_t bytes) {
  DS_ENTER(ctx);
  if (bytes == 0) return DS_OK;
  DS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  return DS_OK;
}

int ds_memset(ds_ctx* ctx, void* dst, int value, size_t bytes) {
  DS_ENTER(ctx);
  if (bytes == 0) return DS_OK;
  DS_CUDA(cudaMemsetAsync(dst, value, bytes, ctx->stream));
  return DS_OK;
}

// Asynchronous staging on the context's copy stream (created on first use): the upload
// of the next solve's operands overlaps the current solve.  The caller guarantees the
// destination is not in use by pending work; ds_wait_event orders a later solve after it.
int ds_upload_async(ds_ctx* ctx, int dtype, const void* src, int64_t rows, int64_t cols, int64_t ld_host,
                    void* dst, int64_t ld_dev, void** event_out) {
  DS_ENTER(ctx);
  *event_out = nullptr;
  if (rows < 0 || cols < 0 || ld_dev < (rows > 0 ? rows : 1) || ld_host < (rows > 0 ? rows : 1)) {
    set_error("upload_async: bad shape %lld x %lld", (long long)rows, (long long)cols);
    return DS_EDIM;
  }
  if (!ctx->copy) DS_CUDA(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
  const size_t es = dtype_size(dtype);
  if (rows > 0 && cols > 0)
    DS_CUDA(cudaMemcpy2DAsync(dst, ld_dev * es, src, ld_host * es, rows * es, cols, cudaMemcpyHostToDevice,
                              ctx->copy));
  cudaEvent_t ev;
  DS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  DS_CUDA(cudaEventRecord(ev, ctx->copy));
  *event_out = (void*)ev;
  return DS_OK;
}

int ds_wait_event(ds_ctx* ctx, void* event) {
  DS_ENTER(ctx);
  if (event) DS_CUDA(cudaStreamWaitEvent(ctx->stream, (cudaEvent_t)event, 0));
  return DS_OK;
}

int ds_event_destroy(void* event) {
  if (event) cudaEventDestroy((cudaEvent_t)event);
  return DS_OK;
}

int ds_upload_matrix(ds_ctx* ctx, int dtype, const void* src, int64_t rows, int64_t cols,
                     int64_t ld_host, int order, void* dst, int64_t ld_dev) {
  DS_ENTER(ctx);
  if (rows < 0 || cols < 0 || ld_dev < (rows > 0 ? rows : 1)) {
    set_error("upload: bad shape %lld x %lld ld_dev %lld", (long long)rows, (long long)cols,
              (long long)ld_dev);
    return DS_EDIM;
  }
  if (rows == 0 || cols == 0) return DS_OK;
  size_t es = dtype_size(dtype);
  if (order == 0) {
    DS_CUDA(cudaMemcpy2DAsync(dst, ld_dev * es, src, ld_host * es, rows * es, cols,
                              cudaMemcpyHostToDevice, ctx->stream));
  } else {
    // stage the C-order rows contiguously, then transpose on the device
    void* tmp = nullptr;
    DS_TRY(ctx_workspace(ctx, (size_t)rows * cols * es, &tmp));
    DS_CUDA(cudaMemcpy2DAsync(tmp, cols * es, src, ld_host * es, cols * es, rows,
                              cudaMemcpyHostToDevice, ctx->stream));
    dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
    DS_DISPATCH(dtype, T,
                transpose_kernel<T><<<grid, dim3(32, 8), 0, ctx->stream>>>(
                    (const T*)tmp, rows, cols, cols, (T*)dst, ld_dev));
    count_launch(ctx);
    DS_CHECK_LAUNCH();
  }
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

int ds_download_matrix(ds_ctx* ctx, int dtype, const void* src, int64_t rows, int64_t cols,
                       int64_t ld_dev, void* dst, int64_t ld_host) {
  DS_ENTER(ctx);
  if (rows == 0 || cols == 0) return DS_OK;
  size_t es = dtype_size(dtype);
  DS_CUDA(cudaMemcpy2DAsync(dst, ld_host * es, src, ld_dev * es, rows * es, cols,
                            cudaMemcpyDeviceToHost, ctx->stream));
  DS_CUDA(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

}  // extern "C"
