// common.cuh — device helpers shared by kernels.cu (multi-kernel path) and fused.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace ss {

#define FULL 0xFFFFFFFFu

// ------------------------------------------------------------------------------------
// small helpers

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan (blockDim.x == NT).  *total (shared memory) receives the sum;
// it is valid after the call.
template <typename T, int BT = NT>
__device__ __forceinline__ T block_excl_scan(T v, T *total) {
  __shared__ T sh[BT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T incl = warp_incl_scan(v);
  if (lane == 31) sh[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const T w = lane < BT / 32 ? sh[lane] : T(0);
    const T wi = warp_incl_scan(w);
    if (lane < BT / 32) sh[lane] = wi - w;
    if (lane == BT / 32 - 1) *total = wi;
  }
  __syncthreads();
  const T r = sh[warp] + incl - v;
  __syncthreads();
  return r;
}

// Block-wide sum; the result is valid in every thread.
template <typename T, int BT = NT>
__device__ __forceinline__ T block_sum(T v) {
  __shared__ T sh[BT / 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    T t = lane < BT / 32 ? sh[lane] : T(0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
    if (lane == 0) sh[BT / 32] = t;
  }
  __syncthreads();
  const T r = sh[BT / 32];
  __syncthreads();
  return r;
}

// Block-wide sums of N values per thread at once (one pair of barriers); results in v[].
template <typename T, int N, int BT = NT>
__device__ __forceinline__ void block_sum_v(T (&v)[N]) {
  __shared__ T sh[N][BT / 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(FULL, v[i], o);
    if (lane == 0) sh[i][warp] = v[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      T t = lane < BT / 32 ? sh[i][lane] : T(0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
      if (lane == 0) sh[i][BT / 32] = t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = sh[i][BT / 32];
  __syncthreads();
}

// Block-wide exclusive scans of N values per thread at once; v[] becomes the exclusive
// prefixes, tot[] (any memory) receives the totals in every thread.
template <typename T, int N, int BT = NT>
__device__ __forceinline__ void block_excl_scan_v(T (&v)[N], T (&tot)[N]) {
  __shared__ T sh[N][BT / 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T incl[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    incl[i] = warp_incl_scan(v[i]);
    if (lane == 31) sh[i][warp] = incl[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const T w = lane < BT / 32 ? sh[i][lane] : T(0);
      const T wi = warp_incl_scan(w);
      if (lane < BT / 32) sh[i][lane] = wi - w;
      if (lane == BT / 32 - 1) sh[i][BT / 32] = wi;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    v[i] = sh[i][warp] + incl[i] - v[i];
    tot[i] = sh[i][BT / 32];
  }
  __syncthreads();
}

// 64-bit sum over the lanes in `mask` of a 32-bit value (exact: split in 16-bit halves).
__device__ __forceinline__ unsigned long long warp_sum_u32_exact(uint32_t v) {
  uint32_t lo = __reduce_add_sync(FULL, v & 0xFFFFu);
  uint32_t hi = __reduce_add_sync(FULL, v >> 16);
  return ((unsigned long long)hi << 16) + lo;
}

__device__ __forceinline__ uint32_t phase_of(uint4 r) { return r.z & 3u; }
__device__ __forceinline__ uint32_t class_of(uint4 r) { return (r.z >> 2) & 3u; }

// Warp-aggregated byte-weighted histogram update: lanes with the same bucket form a group
// (match.any); each group reduces its bytes (exact, 16-bit halves), min and max key, and its
// lowest lane issues one shared-memory atomic per field.
__device__ __forceinline__ void hist_add(unsigned long long *h, uint32_t *mn, uint32_t *nmx, bool on,
                                         uint32_t bucket, uint32_t bits, uint32_t bytes) {
  const uint32_t grp = __match_any_sync(FULL, on ? bucket : 0xFFFFFFFFu);
  if (on) {
    const uint32_t lo = __reduce_add_sync(grp, bytes & 0xFFFFu);
    const uint32_t hi = __reduce_add_sync(grp, bytes >> 16);
    const uint32_t kmin = __reduce_min_sync(grp, bits);
    const uint32_t knmx = __reduce_min_sync(grp, ~bits);
    if ((threadIdx.x & 31) == (uint32_t)(__ffs(grp) - 1)) {
      atomicAdd(&h[bucket], ((unsigned long long)hi << 16) + lo);
      atomicMin(&mn[bucket], kmin);
      atomicMin(&nmx[bucket], knmx);
    }
  }
}

// ------------------------------------------------------------------------------------
// a1: invocation distance of one agent (readings R5, R8, R9)

__device__ __forceinline__ float distance_of(uint4 r, int64_t now, float hop_scale, const float *dint,
                                             uint64_t n_kin, uint32_t &st) {
  const uint32_t ph = phase_of(r), cl = class_of(r);
  float d;
  if (cl == 3u) st |= ST_BAD_RECORD;
  if (ph == 1u || ph == 2u) {
    d = 0.0f;                                  // WAITING / GENERATING
  } else if (ph == 3u) {
    d = __int_as_float(0x7F800000);            // IDLE: +inf
  } else if (cl == 0u || cl == 1u) {
    const int64_t remain = (int64_t)r.x - now; // D_action
    const float d_action = remain <= 0 ? 0.0f : __ll2float_rn(remain);
    d = d_action;
    if (cl == 1u) {                            // Eq. 1: D = min(D_action, D_interaction)
      float d_int = __int_as_float(0x7F800000);
      if (r.w < n_kin) d_int = dint[r.w];
      else st |= ST_BAD_RECORD;
      if (d_int < d_action) d = d_int;
    }
  } else if (cl == 2u) {                       // hop count x hop_scale (R5)
    d = (r.x == 0xFFFFFFFFu) ? __int_as_float(0x7F800000) : __fmul_rn(__uint2float_rn(r.x), hop_scale);
  } else {
    d = __int_as_float(0x7F800000);
  }
  if (d == 0.0f) d = 0.0f;  // canonical +0 (R8)
  return d;
}

// Order-preserving integer key of a finite float (signed-integer order = float order).
__device__ __forceinline__ int32_t fkey(float f) {
  const int32_t i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float fkey_inv(int32_t k) { return __int_as_float(k >= 0 ? k : k ^ 0x7FFFFFFF); }

// Explicit distance (SCALESIM_F_EXPLICIT_DIST, reading R19): word 0 holds the f32 bits;
// NaN or negative -> BAD_RECORD and +inf; -0 -> +0.
__device__ __forceinline__ float explicit_distance_of(uint4 r, uint32_t &st) {
  float d = __uint_as_float(r.x);
  if (!(d >= 0.0f)) {  // NaN or < 0 (-0 compares equal to 0 and passes)
    st |= ST_BAD_RECORD;
    d = __int_as_float(0x7F800000);
  }
  if (d == 0.0f) d = 0.0f;
  return d;
}

__device__ __forceinline__ float theta_of(const Params &p, uint32_t cl) {
  return cl == 0u ? p.theta[0] : cl == 1u ? p.theta[1] : cl == 2u ? p.theta[2] : 0.0f;
}


}  // namespace ss
