// objects.cu — fine-grained distance assignment for shared memory objects (
// reading R19): the distance of a memory object is the minimum distance of the agents that
// reference it.  The objects are then planned by a context with SCALESIM_F_EXPLICIT_DIST.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/scalesim.h"
#include "internal.h"

namespace ss {

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

// Records of every object with distance +inf (no referrer yet); the reference pass lowers
// word 0 (and dist_out) with unsigned minima.
__global__ void __launch_bounds__(OBT) k_object_init(uint64_t n_obj, const uint32_t *__restrict__ obj_bytes,
                                                    const uint32_t *__restrict__ obj_flags, uint4 *__restrict__ rec_out,
                                                    uint32_t *__restrict__ dist_out) {
  for (uint64_t o = blockIdx.x * (uint64_t)OBT + threadIdx.x; o < n_obj; o += (uint64_t)gridDim.x * OBT) {
    rec_out[o] = make_uint4(0x7F800000u, obj_bytes[o], obj_flags ? obj_flags[o] : 0u, 0u);
    if (dist_out) dist_out[o] = 0x7F800000u;
  }
}

// last object o with ref_ptr[o] <= k (the object holding reference k; empty objects before
// it are skipped), searched in [lo, hi)
__device__ __forceinline__ uint64_t object_of(const unsigned long long *ref_ptr, uint64_t lo, uint64_t hi, uint64_t k) {
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) / 2;
    if (ref_ptr[mid] <= k) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Load-balanced segmented minimum over the references: warp w owns references
// [w * 32 * LR, (w + 1) * 32 * LR), loaded coalesced and keyed through shared memory; lane l
// walks the contiguous range [l * LR, (l + 1) * LR) of it.  Objects inside a lane's range are
// that lane's alone (plain stores); an object crossing lanes is combined across the warp by a
// segmented shuffle reduction (object ids are non-decreasing in lane order) and lowered with
// one atomicMin per warp, so a prompt shared by every agent costs refs / (32 LR) atomics.
constexpr int LR = 16;
__global__ void __launch_bounds__(OBT) k_object_refs(const uint32_t *__restrict__ dist_bits, uint64_t n_agents,
                                                    const unsigned long long *__restrict__ ref_ptr,
                                                    const uint32_t *__restrict__ ref_agent, uint64_t n_obj,
                                                    uint4 *__restrict__ rec_out,
                                                    uint32_t *__restrict__ dist_out, uint32_t *status_out) {
  __shared__ uint32_t sk[OBT / 32][32 * LR];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t warp_g = (blockIdx.x * (uint64_t)OBT + threadIdx.x) / 32;
  const uint64_t n_warps = (uint64_t)gridDim.x * OBT / 32;
  const uint64_t n_refs = ref_ptr[n_obj];
  uint32_t bad = 0;
  for (uint64_t k0 = warp_g * 32 * LR; k0 < n_refs; k0 += n_warps * 32 * LR) {
    const uint64_t cnt = n_refs - k0 < 32 * LR ? n_refs - k0 : 32 * LR;
#pragma unroll
    for (int j = 0; j < LR; ++j) {  // coalesced: all loads in flight, then the distance gathers
      const uint64_t x = j * 32 + lane;
      sk[wib][x] = x < cnt ? ref_agent[k0 + x] : 0u;
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < LR; ++j) {
      const uint64_t x = j * 32 + lane;
      if (x < cnt) {
        const uint32_t a = sk[wib][x];
        uint32_t key = 0x7F800000u;
        if (a < n_agents) key = dist_key(dist_bits[a], bad);
        else bad = 1u;
        sk[wib][x] = key;
      }
    }
    __syncwarp();
    // objects of the warp's first and last reference (lanes 0 / 1 search, the others search
    // between them)
    uint64_t o_lo = 0, o_hi = 0;
    if (lane < 2) {
      const uint64_t kk = lane == 0 ? k0 : k0 + cnt - 1;
      const uint64_t o = object_of(ref_ptr, 0, n_obj, kk);
      if (lane == 0) o_lo = o;
      else o_hi = o;
    }
    o_lo = __shfl_sync(0xFFFFFFFFu, o_lo, 0);
    o_hi = __shfl_sync(0xFFFFFFFFu, o_hi, 1);
    const uint64_t kb = k0 + (uint64_t)lane * LR, ke = (kb + LR < k0 + cnt) ? kb + LR : k0 + cnt;
    const bool act = kb < ke;
    uint64_t o_first = o_hi + 1, o_last = o_hi + 1;  // (inactive lanes: beyond every real object)
    uint32_t m_first = 0x7F800000u, m_last = 0x7F800000u;
    if (act) {
      uint64_t o = object_of(ref_ptr, o_lo, o_hi + 1, kb);
      uint64_t end = ref_ptr[o + 1];
      o_first = o;
      uint32_t m = 0x7F800000u;
      bool first = true;
      for (uint64_t k = kb; k < ke; ++k) {
        if (k >= end) {  // object o ends inside this lane's range
          if (first) m_first = m;
          else {  // interior object: only this lane touches it
            rec_out[o].x = m;
            if (dist_out) dist_out[o] = m;
          }
          first = false;
          do {  // skip objects without references
            ++o;
            end = ref_ptr[o + 1];
          } while (k >= end);
          m = 0x7F800000u;
        }
        m = min(m, sk[wib][k - k0]);
      }
      if (first) m_first = m;
      else {
        o_last = o;
        m_last = m;
      }
    }
    // combine the partials of each object across the warp: "first" partials, then "last"
    // partials (each sequence is sorted by object); leaders lower the object atomically
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      const uint64_t oo = pass == 0 ? o_first : o_last;
      uint32_t mm = pass == 0 ? m_first : m_last;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t m2 = __shfl_down_sync(0xFFFFFFFFu, mm, off);
        const uint64_t o2 = __shfl_down_sync(0xFFFFFFFFu, oo, off);
        if (lane + off < 32 && o2 == oo) mm = min(mm, m2);
      }
      const uint64_t prev = __shfl_up_sync(0xFFFFFFFFu, oo, 1);
      if ((lane == 0 || prev != oo) && oo <= o_hi && mm != 0x7F800000u) {
        atomicMin(&rec_out[oo].x, mm);
        if (dist_out) atomicMin(&dist_out[oo], mm);
      }
    }
    __syncwarp();
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
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t blocks = (n_objects + OBT - 1) / OBT;
  if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
  k_object_init<<<(unsigned)blocks, OBT, 0, st>>>(n_objects, obj_bytes, obj_flags, static_cast<uint4 *>(obj_rec_out),
                                                  reinterpret_cast<uint32_t *>(obj_dist_out));
  // the reference count (ref_ptr[n_objects]) is read on the device: no host round trip, so
  // the call stays graph-capturable; the grid strides over the references
  k_object_refs<<<(unsigned)(sms * 8), OBT, 0, st>>>(reinterpret_cast<const uint32_t *>(agent_dist), n_agents,
                                                     reinterpret_cast<const unsigned long long *>(ref_ptr), ref_agent,
                                                     n_objects, static_cast<uint4 *>(obj_rec_out),
                                                     reinterpret_cast<uint32_t *>(obj_dist_out), status_out);
  return cudaGetLastError() == cudaSuccess ? SCALESIM_OK : SCALESIM_E_CUDA;
}
