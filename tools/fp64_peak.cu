// Microbenchmark: FP64 DMMA (mma.sync f64) and DFMA peak throughput on this B200,
// plus a plain streaming-read bandwidth probe. Used to set the LU roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NACC][2];
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
template<int NACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-4;
  double c[NACC][4];
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(a[4]),"d"(a[5]),"d"(a[6]),"d"(a[7]),
                     "d"(b[0]),"d"(b[1]),"d"(b[2]),"d"(b[3]));
  }
  double s = 0; for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}
template<int NACC>
__global__ void dfma_k(double* out, int iters) {
  double c[NACC]; double a = threadIdx.x * 1e-7, b = 1.0000001;
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0; for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}
__global__ void read_bw(const double4* __restrict__ p, size_t n, double* out) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2* q = reinterpret_cast<const double2*>(p + i); double2 v = __ldcs(q), w = __ldcs(q + 1); acc += v.x + v.y + w.x + w.y;
  }
  if (acc == 12345.0) out[0] = acc;
}

template<typename K>
float timeit(K k, dim3 g, dim3 b, double* out, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<g, b>>>(out, iters); cudaDeviceSynchronize();
  cudaEventRecord(e0); k<<<g, b>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  printf("device %s SMs %d L2 %d MB smemPerBlockOptin %zu KB clock %d MHz\n", pr.name, pr.multiProcessorCount,
         pr.l2CacheSize >> 20, pr.sharedMemPerBlockOptin >> 10, pr.clockRate / 1000);
  double* out; CK(cudaMalloc(&out, 8));
  int sms = pr.multiProcessorCount;
  for (int wpb : {4, 8, 16}) {
    int iters = 20000;
    float ms = timeit(dmma_m8n8k4<8>, dim3(sms * 2), dim3(32 * wpb), out, iters);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (sms * 2) * wpb;
    printf("DMMA m8n8k4  warps/blk %2d: %.2f TFLOP/s\n", wpb, flops / ms / 1e9);
    ms = timeit(dmma_m16n8k16<4>, dim3(sms * 2), dim3(32 * wpb), out, iters / 4);
    flops = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * (sms * 2) * wpb;
    printf("DMMA m16n8k16 warps/blk %2d: %.2f TFLOP/s\n", wpb, flops / ms / 1e9);
    ms = timeit(dfma_k<16>, dim3(sms * 2), dim3(32 * wpb), out, iters);
    flops = 2.0 * 16 * iters * 32.0 * (sms * 2) * wpb;
    printf("DFMA          warps/blk %2d: %.2f TFLOP/s\n", wpb, flops / ms / 1e9);
  }
  size_t bytes = (size_t)8 << 30; double4* p; CK(cudaMalloc(&p, bytes)); cudaMemset(p, 0, bytes);
  size_t n4 = bytes / 32;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    for (int gm : {4, 8, 16}) {
      read_bw<<<sms * gm, 256>>>(p, n4, out); cudaDeviceSynchronize();
      cudaEventRecord(e0); read_bw<<<sms * gm, 256>>>(p, n4, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("read-only stream 8GiB grid %d x256: %.0f GB/s\n", sms * gm, bytes / ms / 1e6);
    }
  }
  return 0;
}
