// baselines.cu — the reactive LRU baseline of the paper's evaluation (SGLang-style
// on-demand loading with least-recently-used eviction), expressed as
// explicit distances for the same planner (NEXT #3, reading R20): a requesting agent
// (WAITING / GENERATING) has distance 0 and refreshes its last use; any other agent has
// distance now - last use (+inf if never used).  Planned with theta = 0 (no prefetch), the
// kept set is the requesting agents plus the most recently used ones that fit, and evictions
// go least recently used first — LRU.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/scalesim.h"
#include "common.cuh"
#include "internal.h"

namespace ss {

__global__ void __launch_bounds__(NT) k_lru_records(const uint4 *__restrict__ rec, uint64_t n, int64_t now,
                                                   uint32_t *__restrict__ last_use, uint4 *__restrict__ out) {
  const uint32_t now32 = (uint32_t)now;
  for (uint64_t i = blockIdx.x * (uint64_t)NT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * NT) {
    const uint4 r = ld_stream(rec + i);
    const uint32_t ph = phase_of(r);
    uint32_t lu = last_use[i];
    float d;
    if (ph == 1u || ph == 2u) {  // in an LLM call: its memory is in use now
      lu = now32;
      last_use[i] = lu;
      d = 0.0f;
    } else if (lu == 0xFFFFFFFFu) {
      d = __int_as_float(0x7F800000);  // never used
    } else {
      d = __uint2float_rn(now32 - lu);  // steps since the last use
    }
    out[i] = make_uint4(__float_as_uint(d), r.y, r.z & 0x10u, 0u);  // footprint, dirty bit
  }
}

}  // namespace ss

extern "C" scalesim_status scalesim_lru_records(const uint32_t *agent_rec, uint64_t n_agents, int64_t now_tick,
                                                uint32_t *last_use, void *rec_out, void *stream) {
  using namespace ss;
  if (n_agents == 0) return SCALESIM_OK;
  if (!agent_rec || !last_use || !rec_out || reinterpret_cast<uintptr_t>(agent_rec) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(rec_out) % 16 != 0)
    return SCALESIM_E_INVALID;
  if (now_tick < 0 || now_tick >= 0xFFFFFFFFll) return SCALESIM_E_INVALID;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return SCALESIM_E_CUDA;
  uint64_t blocks = (n_agents + NT - 1) / NT;
  if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
  k_lru_records<<<(unsigned)blocks, NT, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint4 *>(agent_rec), n_agents, now_tick, last_use, static_cast<uint4 *>(rec_out));
  return cudaGetLastError() == cudaSuccess ? SCALESIM_OK : SCALESIM_E_CUDA;
}
