// Micro-benchmark: latency / throughput of warp primitives on sm_100a (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t ballot_match(uint32_t v, int bits) {
  uint32_t m = 0xFFFFFFFFu;
  for (int b = 0; b < bits; ++b) {
    const uint32_t x = __ballot_sync(0xFFFFFFFFu, (v >> b) & 1u);
    m &= ((v >> b) & 1u) ? x : ~x;
  }
  return m;
}

template <int OP>
__global__ void k(uint32_t *out, int iters, int warps_active) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= warps_active) return;
  uint32_t v = (lane * 7 + warp) & 15u, acc = 0;
  __shared__ uint32_t sh[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) acc += __match_any_sync(0xFFFFFFFFu, v + acc % 3);
    else if (OP == 1) acc += __reduce_add_sync(0xFFFFFFFFu, v + acc);
    else if (OP == 2) {
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, v);
      acc += __reduce_add_sync(peers, v + acc);
    } else if (OP == 3) acc += ballot_match(v + acc % 3, 4);
    else if (OP == 4) acc += ballot_match(v + acc % 3, 11);
    else if (OP == 5) acc += __ballot_sync(0xFFFFFFFFu, (v + acc) & 1u);
    else if (OP == 6) acc += atomicAdd(&sh[(v + acc) & 15u], 1u);        // 16 addresses, 2-way per addr
    else if (OP == 7) acc += atomicAdd(&sh[0], 1u + (acc & 1));          // all lanes one address
    else if (OP == 8) {                                                  // shfl-up scan step x5
      uint32_t x = v + acc;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += t;
      }
      acc += x;
    } else if (OP == 9) {
      __syncthreads();
      acc += 1;
    } else if (OP == 10) {  // spread addresses, all lanes, u32 add (no return)
      atomicAdd(&sh[(threadIdx.x * 33 + i * 97) & 4095], 1u);
    } else if (OP == 11) {  // spread addresses, all lanes, u64 add
      atomicAdd(reinterpret_cast<unsigned long long *>(sh) + ((threadIdx.x * 33 + i * 97) & 2047), 1ull);
    } else if (OP == 12) {  // spread, u32 min
      atomicMin(&sh[(threadIdx.x * 33 + i * 97) & 4095], (uint32_t)i);
    } else if (OP == 13) {  // spread, 8 of 32 lanes
      if ((lane & 3) == 0) atomicAdd(&sh[(threadIdx.x * 33 + i * 97) & 4095], 1u);
    } else if (OP == 14) {  // plain STS, all lanes
      sh[(threadIdx.x * 33 + i * 97) & 4095] = i;
    }
  }
  const long long t1 = clock64();
  if (lane == 0 && warp == 0) out[0] = (uint32_t)((t1 - t0) / iters);
  if (acc == 0x12345678u) out[1] = acc;
}

template <int OP>
void run(const char *name) {
  uint32_t *d;
  cudaMalloc(&d, 8);
  for (int w : {1, 32}) {
    k<OP><<<1, 1024>>>(d, 2000, w);
    uint32_t h = 0;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("%-40s warps=%2d  %5u cycles/iter  (%s)\n", name, w, h, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  run<0>("match_any");
  run<1>("reduce_add full mask");
  run<2>("match_any + reduce_add(peers)");
  run<3>("ballot match 4 bits");
  run<4>("ballot match 11 bits");
  run<5>("ballot");
  run<6>("smem atomicAdd 16 addrs");
  run<7>("smem atomicAdd 1 addr");
  run<8>("shfl_up scan (5 steps)");
  run<9>("__syncthreads (1024 thr)");
  run<10>("smem atomicAdd u32 spread, 32 lanes");
  run<11>("smem atomicAdd u64 spread, 32 lanes");
  run<12>("smem atomicMin u32 spread, 32 lanes");
  run<13>("smem atomicAdd u32 spread, 8 lanes");
  run<14>("smem store spread, 32 lanes");
  return 0;
}
