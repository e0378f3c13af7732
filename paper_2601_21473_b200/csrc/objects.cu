// objects.cu — fine-grained distance assignment for shared memory objects (
// reading R19): the distance of a memory object is the minimum distance of the agents that
// reference it.  The objects are then planned by a context with SCALESIM_F_EXPLICIT_DIST.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/scalesim.h"
#include "internal.h"

namespace ss {

constexpr int OG = 8;     // lanes per object (objects referenced by few agents waste few lanes)
constexpr int OBT = 256;  // threads per block

// Distance bits of non-negative floats (and +inf) order like the values, so the minimum is an
// unsigned minimum of the bit patterns.  NaN / negative values are out of contract: flagged and
// read as +inf; -0 reads as +0.
__device__ __forceinline__ uint32_t dist_key(uint32_t x, uint32_t &bad) {
  if (x == 0x80000000u) return 0u;
  if (x > 0x7F800000u) {
    bad = 1u;
    return 0x7F800000u;
  }
  return x;
}

__global__ void __launch_bounds__(OBT) k_object_min(const uint32_t *__restrict__ dist_bits, uint64_t n_agents,
                                                   const unsigned long long *__restrict__ ref_ptr,
                                                   const uint32_t *__restrict__ ref_agent, uint64_t n_obj,
                                                   const uint32_t *__restrict__ obj_bytes,
                                                   const uint32_t *__restrict__ obj_flags, uint4 *__restrict__ rec_out,
                                                   float *__restrict__ dist_out, uint32_t *status_out) {
  const uint32_t lane = threadIdx.x & 31, sub = lane & (OG - 1), grp = lane / OG;
  const uint64_t warp_g = (blockIdx.x * (uint64_t)OBT + threadIdx.x) / 32;
  const uint64_t n_warps = (uint64_t)gridDim.x * OBT / 32;
  uint32_t bad = 0;
  // warp-uniform loop: 32 / OG objects per warp per iteration
  for (uint64_t ob = warp_g * (32 / OG); ob < n_obj; ob += n_warps * (32 / OG)) {
    const uint64_t o = ob + grp;
    uint32_t m = 0x7F800000u;  // +inf: no referrer
    if (o < n_obj) {
      const uint64_t b = ref_ptr[o], e = ref_ptr[o + 1];
      for (uint64_t k = b + sub; k < e; k += OG) {
        const uint32_t a = ref_agent[k];
        if (a < n_agents) m = min(m, dist_key(dist_bits[a], bad));
        else bad = 1u;
      }
    }
#pragma unroll
    for (int off = OG / 2; off > 0; off >>= 1) m = min(m, __shfl_xor_sync(0xFFFFFFFFu, m, off));
    if (o < n_obj && sub == 0) {
      rec_out[o] = make_uint4(m, obj_bytes[o], obj_flags ? obj_flags[o] : 0u, 0u);
      if (dist_out) dist_out[o] = __uint_as_float(m);
    }
  }
  if (bad && status_out) atomicOr(status_out, ST_BAD_RECORD);
}

}  // namespace ss

extern "C" scalesim_status scalesim_object_min(const float *agent_dist, uint64_t n_agents, const uint64_t *ref_ptr,
                                               const uint32_t *ref_agent, uint64_t n_objects,
                                               const uint32_t *obj_bytes, const uint32_t *obj_flags,
                                               void *obj_rec_out, float *obj_dist_out, uint32_t *status_out,
                                               void *stream) {
  using namespace ss;
  if (n_objects == 0) return SCALESIM_OK;
  if (!ref_ptr || !ref_agent || !obj_bytes || !obj_rec_out || (n_agents > 0 && !agent_dist)) return SCALESIM_E_INVALID;
  if (reinterpret_cast<uintptr_t>(obj_rec_out) % 16 != 0 || reinterpret_cast<uintptr_t>(ref_ptr) % 8 != 0)
    return SCALESIM_E_INVALID;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return SCALESIM_E_CUDA;
  const uint64_t per_block = OBT / OG;
  uint64_t blocks = (n_objects + per_block - 1) / per_block;
  const uint64_t cap = (uint64_t)sms * 8;  // 8 blocks of 256 threads per SM, grid-stride beyond
  if (blocks > cap) blocks = cap;
  k_object_min<<<(unsigned)blocks, OBT, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint32_t *>(agent_dist), n_agents, reinterpret_cast<const unsigned long long *>(ref_ptr),
      ref_agent, n_objects, obj_bytes, obj_flags, static_cast<uint4 *>(obj_rec_out), obj_dist_out, status_out);
  return cudaGetLastError() == cudaSuccess ? SCALESIM_OK : SCALESIM_E_CUDA;
}
