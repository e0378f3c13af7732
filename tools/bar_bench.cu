// Micro-benchmark: grid-barrier variants and contended global atomics before a barrier,
// 1 CTA x 1024 threads per SM (the fused planner's launch shape).  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned *p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int V>
__device__ __forceinline__ void gbar(unsigned *ctr, unsigned *flags, unsigned &k, unsigned n) {
  __syncthreads();
  ++k;
  if (V == 0) {  // counter, thread 0: fence + atomicAdd, acquire poll + nanosleep(40), fence
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr, 1u);
      while (ld_acq(ctr) < k * n) __nanosleep(40);
      __threadfence();
    }
  } else if (V == 1) {  // counter, red.release, relaxed poll without sleep, fence
    if (threadIdx.x == 0) {
      red_rel(ctr, 1u);
      while (ld_rlx(ctr) < k * n) {
      }
      __threadfence();
    }
  } else if (V == 2) {  // counter, red.release, acquire poll, no fence after
    if (threadIdx.x == 0) {
      red_rel(ctr, 1u);
      while (ld_acq(ctr) < k * n) {
      }
    }
  } else if (V == 3) {  // flags, warp 0 acquire poll + nanosleep(20)
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) {
        __threadfence();
        *(volatile unsigned *)(flags + blockIdx.x) = k;
      }
      while (true) {
        bool ok = true;
        for (unsigned q = threadIdx.x; q < n; q += 32) ok &= (int)(ld_acq(flags + q) - k) >= 0;
        if (__all_sync(0xFFFFFFFFu, ok)) break;
        __nanosleep(20);
      }
      if (threadIdx.x == 0) __threadfence();
    }
  } else if (V == 4) {  // flags, relaxed poll, no sleep, fence after
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) {
        __threadfence();
        *(volatile unsigned *)(flags + blockIdx.x) = k;
      }
      while (true) {
        bool ok = true;
        for (unsigned q = threadIdx.x; q < n; q += 32) ok &= (int)(ld_rlx(flags + q) - k) >= 0;
        if (__all_sync(0xFFFFFFFFu, ok)) break;
      }
      __threadfence();
    }
  }
  __syncthreads();
}

// MODE 0: barriers only; 1: 60 contended buckets x 4 arrays of u32 REDs per CTA (packed
// arrays), then barrier, then every CTA reads the 4 x 1024 arrays; 2: same with a stride of
// 32 words per bucket
template <int V, int MODE>
__global__ void __launch_bounds__(1024, 1) k(unsigned *ctr, unsigned *flags, unsigned *arr, int iters, unsigned *sink) {
  unsigned kk = 0, acc = 0;
  const unsigned n = gridDim.x;
  for (int it = 0; it < iters; ++it) {
    if (MODE > 0) {
      const int stride = MODE == 2 ? 32 : 1;
      if (threadIdx.x < 240) {
        const int a = threadIdx.x / 60, b = threadIdx.x % 60;
        unsigned *p = arr + a * 1024 * stride + (b * 7 % 1024) * stride;
        if (a < 2) atomicAdd(p, 1u);
        else atomicMin(p, threadIdx.x + it);
      }
    }
    gbar<V>(ctr, flags, kk, n);
    if (MODE > 0) {
      const int stride = MODE == 2 ? 32 : 1;
      for (int q = 0; q < 4; ++q) acc += arr[q * 1024 * stride + threadIdx.x * stride];
      gbar<V>(ctr, flags, kk, n);
    }
  }
  if (acc == 0xFFFFFFFFu) sink[0] = acc;
}

template <int V, int MODE>
void run(const char *name, int sms) {
  unsigned *ctr, *flags, *arr, *sink;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&flags, 4 * 256);
  cudaMalloc(&arr, 4 * 4 * 1024 * 32);
  cudaMalloc(&sink, 4);
  cudaMemset(arr, 0, 4 * 4 * 1024 * 32);
  cudaFuncSetAttribute(k<V, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 150000);
  float best = 1e9;
  const int iters = 2000;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(ctr, 0, 4);
    cudaMemset(flags, 0, 4 * 256);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<V, MODE><<<sms, 1024, 150000>>>(ctr, flags, arr, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const int nb = MODE == 0 ? iters : 2 * iters;
  printf("%-44s %8.3f us per barrier (%s)\n", name, best * 1000.0f / nb, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  run<0, 0>("V0 counter+fence, acquire poll, sleep40", sms);
  run<1, 0>("V1 counter red.release, relaxed poll, fence", sms);
  run<2, 0>("V2 counter red.release, acquire poll", sms);
  run<3, 0>("V3 flags, warp acquire poll, sleep20", sms);
  run<4, 0>("V4 flags, warp relaxed poll, fence", sms);
  run<0, 1>("V0 + contended REDs packed (per 2 barriers)", sms);
  run<1, 1>("V1 + contended REDs packed", sms);
  run<4, 1>("V4 + contended REDs packed", sms);
  run<0, 2>("V0 + contended REDs stride 128B", sms);
  run<1, 2>("V1 + contended REDs stride 128B", sms);
  run<4, 2>("V4 + contended REDs stride 128B", sms);
  return 0;
}
