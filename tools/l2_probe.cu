// L2 persistence probe: time repeated streaming reads of an N-byte buffer with and
// without an access-policy window (hitRatio = set-aside / N).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_probe tools/l2_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__global__ void read_kernel(const double2* __restrict__ p, size_t n2, double* out) {
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = __ldg(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? atoll(argv[1]) : 134;
  const size_t bytes = mb << 20;
  int persist = 0, window = 0;
  cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaDeviceGetAttribute(&window, cudaDevAttrMaxAccessPolicyWindowSize, 0);
  double2* p;
  double* out;
  cudaMalloc(&p, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(p, 0, bytes);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t n2 = bytes / 16;
  for (int mode = 0; mode < 3; ++mode) {
    if (mode >= 1) {
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist);
      cudaStreamAttrValue v = {};
      v.accessPolicyWindow.base_ptr = p;
      v.accessPolicyWindow.num_bytes = bytes < (size_t)window ? bytes : (size_t)window;
      double hr = (double)persist / v.accessPolicyWindow.num_bytes;
      if (mode == 2) hr *= 0.9;
      v.accessPolicyWindow.hitRatio = hr > 1 ? 1.f : (float)hr;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
    }
    for (int w = 0; w < 5; ++w) read_kernel<<<148 * 8, 512, 0, s>>>(p, n2, out);
    cudaEventRecord(e0, s);
    for (int it = 0; it < 50; ++it) read_kernel<<<148 * 8, 512, 0, s>>>(p, n2, out);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%zu MiB mode=%d (0 none, 1 window, 2 window 0.9x): %.2f us/pass = %.0f GB/s (persist max %d, window max %d) %s\n",
           mb, mode, ms * 1e3 / 50, bytes / (ms * 1e-3 / 50) / 1e9, persist, window,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
