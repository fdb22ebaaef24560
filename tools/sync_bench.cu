// Microbenchmark of grid-wide exchange patterns for the LU panel kernel (148 CTAs x 128 threads):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/sync_bench.cu -o tools/sync_bench
// Prints microseconds per round for each pattern.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t w) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;\n" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t w;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(w) : "l"(p) : "memory");
  return w;
}

// 0: fence + atomicAdd + acquire poll (current grid_sync)
// 1: red.release + acquire poll
// 2: mode 0 + one dependent L2 round trip of candidate loads + one of a row load
// 3: LL all-to-all: every thread polls 2 headers (3 words each) every iteration
// 4: LL all-to-all, one warp polls (5 headers per lane), then smem broadcast
// 5: LL with headers padded to 128 B lines, 128 threads polling
__global__ void bench(int mode, int rounds, unsigned* bar, double* cand, uint64_t* hdr, long long* out) {
  __shared__ int s_ok;
  const unsigned G = gridDim.x;
  unsigned epoch = 0;
  double acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    if (mode <= 2) {
      __syncthreads();
      epoch += 1;
      if (threadIdx.x == 0) {
        if (mode == 1) {
          red_release_add(bar, 1u);
        } else {
          __threadfence();
          atomicAdd(bar, 1u);
        }
        while (ld_acquire_u32(bar) < epoch * G) {
        }
      }
      __syncthreads();
      if (mode == 2) {
        double v = 0;
        for (unsigned b = threadIdx.x; b < G; b += blockDim.x) v += __ldcg(cand + b + (r & 1) * 1024);
        acc += v;
        __syncthreads();
        acc += __ldcg(cand + 4096 + threadIdx.x + (int)(acc > 1e300));
        __syncthreads();
        if (threadIdx.x == 0) cand[blockIdx.x + ((r + 1) & 1) * 1024] = acc;
      }
    } else {
      const uint32_t ep = (uint32_t)r + 1;
      const int stride = mode >= 5 ? 16 : 4;
      uint64_t* mine = hdr + ((size_t)(r & 1) * G + blockIdx.x) * stride;
      if (threadIdx.x == 0) {
        st_relaxed(mine, ((uint64_t)ep << 32) | 1u);
        st_relaxed(mine + 1, ((uint64_t)ep << 32) | 2u);
        st_relaxed(mine + 2, ((uint64_t)ep << 32) | 3u);
      }
      if (mode == 3 || mode == 5) {
        for (unsigned b0 = threadIdx.x; b0 < G; b0 += 2 * blockDim.x) {
          const unsigned b1 = b0 + blockDim.x < G ? b0 + blockDim.x : b0;
          const uint64_t* h0 = hdr + ((size_t)(r & 1) * G + b0) * stride;
          const uint64_t* h1 = hdr + ((size_t)(r & 1) * G + b1) * stride;
          while (true) {
            uint64_t a0 = ld_relaxed(h0), a1 = ld_relaxed(h0 + 1), a2 = ld_relaxed(h0 + 2);
            uint64_t c0 = ld_relaxed(h1), c1 = ld_relaxed(h1 + 1), c2 = ld_relaxed(h1 + 2);
            if ((a0 >> 32) == ep && (a1 >> 32) == ep && (a2 >> 32) == ep && (c0 >> 32) == ep &&
                (c1 >> 32) == ep && (c2 >> 32) == ep) {
              acc += (double)(a0 & 7) + (double)(c2 & 7);
              break;
            }
          }
        }
        __syncthreads();
      } else if (mode == 6 || mode == 7) {
        // the LU poller pattern: one warp, 128-B padded headers, pending mask (mode 7: 1 word per header)
        if (threadIdx.x < 32) {
          const int lane = threadIdx.x;
          uint64_t x[5][3];
          unsigned pending = 0;
          for (int q = 0; q < 5; ++q)
            if (lane + 32 * q < (int)G) pending |= 1u << q;
          while (pending) {
#pragma unroll
            for (int q = 0; q < 5; ++q)
              if (pending >> q & 1u) {
                const uint64_t* h = hdr + ((size_t)(r & 1) * G + lane + 32 * q) * 16;
                x[q][0] = ld_relaxed(h);
                if (mode == 6) {
                  x[q][1] = ld_relaxed(h + 1);
                  x[q][2] = ld_relaxed(h + 2);
                } else {
                  x[q][1] = x[q][2] = x[q][0];
                }
              }
#pragma unroll
            for (int q = 0; q < 5; ++q)
              if ((pending >> q & 1u) && (x[q][0] >> 32) == ep && (x[q][1] >> 32) == ep && (x[q][2] >> 32) == ep)
                pending &= ~(1u << q);
          }
          acc += (double)(x[0][0] & 7);
        }
        __syncthreads();
      } else {
        if (threadIdx.x < 32) {
          for (unsigned b0 = threadIdx.x; b0 < G; b0 += 32 * 5) {
            uint64_t w[5][3];
            while (true) {
              bool ok = true;
#pragma unroll
              for (int q = 0; q < 5; ++q) {
                const unsigned b = b0 + 32 * q < G ? b0 + 32 * q : b0;
                const uint64_t* h = hdr + ((size_t)(r & 1) * G + b) * stride;
                w[q][0] = ld_relaxed(h);
                w[q][1] = ld_relaxed(h + 1);
                w[q][2] = ld_relaxed(h + 2);
                ok = ok && (w[q][0] >> 32) == ep && (w[q][1] >> 32) == ep && (w[q][2] >> 32) == ep;
              }
              if (ok) break;
            }
            acc += (double)(w[0][0] & 7);
          }
          if (threadIdx.x == 0) s_ok = 1;
        }
        __syncthreads();
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345.678) out[1] = 1;
}

// cluster exchange: every CTA writes its candidate into every CTA's shared memory
// (DSMEM), then one cluster barrier; rounds of (write, barrier, reduce)
__global__ void bench_cluster(int rounds, long long* out) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double slots[2][16];
  const unsigned me = cl.block_rank(), G = cl.num_blocks();
  double acc = 0;
  cl.sync();
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const int par = r & 1;
    if (threadIdx.x < G) {
      double* dst = cl.map_shared_rank(&slots[par][0], threadIdx.x);
      dst[me] = (double)(r + me);
    }
    cl.sync();
    if (threadIdx.x < 32) {
      double v = threadIdx.x < G ? slots[par][threadIdx.x] : 0.0;
      for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      acc += v;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345.678) out[1] = 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned* bar;
  double* cand;
  uint64_t* hdr;
  long long* out;
  cudaMalloc(&bar, 256);
  cudaMalloc(&cand, 8 * 8192);
  cudaMalloc(&hdr, 8 * 16 * 2 * 1024);
  cudaMalloc(&out, 64);
  cudaMemset(cand, 0, 8 * 8192);
  const char* names[] = {"fence+atomic barrier", "red.release barrier", "barrier + 2 dependent L2 loads",
                         "LL all threads poll", "LL one warp polls", "LL padded lines, all threads",
                         "LL padded, one warp, pending mask", "LL padded, one warp, 1 word"};
  for (int G : {2, 4, 8, 16}) {
    cudaFuncSetAttribute(bench_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(128);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int rounds = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, bench_cluster, rounds, out);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cluster G=%2d DSMEM write + cluster.sync     %7.3f us/round (%s)\n", G, 1e3 * ms / rounds,
           cudaGetErrorString(err));
  }
  for (int G : {148, 74, 37, 16, 10}) {
    for (int mode = 0; mode < 8; ++mode) {
      const int rounds = 2000;
      cudaMemset(bar, 0, 256);
      cudaMemset(hdr, 0, 8 * 16 * 2 * 1024);
      void* args[] = {&mode, (void*)&rounds, &bar, &cand, &hdr, &out};
      int rr = rounds;
      args[1] = &rr;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)bench, dim3(G), dim3(128), args, 0, 0);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("G=%3d %-32s %7.3f us/round (%s)\n", G, names[mode], 1e3 * ms / rounds, cudaGetErrorString(err));
    }
  }
  return 0;
}
