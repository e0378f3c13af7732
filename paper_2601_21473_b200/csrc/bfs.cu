// bfs.cu — hop counts of the diffusion class ("hop count from the information source",
// R9; NEXT #4: computed on the GPU at initialisation): level-synchronous frontier BFS over a
// CSR graph from a source set.  Each level one kernel expands the frontier, claiming a vertex
// with atomicCAS on its hop count (the BFS level of a vertex is unique, so the result does not
// depend on which parent claims it) and appending it to the next frontier.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/scalesim.h"
#include "internal.h"

namespace ss {

constexpr int BT = 256;

__global__ void __launch_bounds__(BT) k_bfs_init(uint32_t *hops, uint64_t n, const uint32_t *src, uint64_t n_src,
                                                uint32_t *front, uint32_t *cnt) {
  for (uint64_t v = blockIdx.x * (uint64_t)BT + threadIdx.x; v < n; v += (uint64_t)gridDim.x * BT)
    hops[v] = 0xFFFFFFFFu;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    cnt[0] = 0;
    cnt[1] = 0;
  }
}

__global__ void __launch_bounds__(BT) k_bfs_sources(uint32_t *hops, uint64_t n, const uint32_t *src, uint64_t n_src,
                                                   uint32_t *front, uint32_t *cnt) {
  for (uint64_t k = blockIdx.x * (uint64_t)BT + threadIdx.x; k < n_src; k += (uint64_t)gridDim.x * BT) {
    const uint32_t s = src[k];
    if (s < n && atomicCAS(&hops[s], 0xFFFFFFFFu, 0u) == 0xFFFFFFFFu) front[atomicAdd(&cnt[0], 1u)] = s;
  }
}

// one warp per frontier vertex: its neighbours in coalesced chunks of 32
__global__ void __launch_bounds__(BT) k_bfs_expand(const unsigned long long *__restrict__ row_ptr,
                                                  const uint32_t *__restrict__ col, uint64_t n, uint32_t *hops,
                                                  const uint32_t *front, const uint32_t *n_front, uint32_t *next,
                                                  uint32_t *n_next, uint32_t level) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp_g = (blockIdx.x * (uint64_t)BT + threadIdx.x) / 32, n_warps = (uint64_t)gridDim.x * BT / 32;
  const uint32_t nf = *n_front;
  for (uint64_t f = warp_g; f < nf; f += n_warps) {
    const uint32_t u = front[f];
    const uint64_t b = row_ptr[u], e = row_ptr[u + 1];
    for (uint64_t k = b + lane; k < e; k += 32) {
      const uint32_t w = col[k];
      if (w < n && hops[w] == 0xFFFFFFFFu && atomicCAS(&hops[w], 0xFFFFFFFFu, level + 1) == 0xFFFFFFFFu)
        next[atomicAdd(n_next, 1u)] = w;
    }
  }
}

}  // namespace ss

extern "C" uint64_t scalesim_bfs_scratch_bytes(uint64_t n_vertices) { return 8 * (n_vertices + 1) + 64; }

extern "C" scalesim_status scalesim_bfs_hops(const uint64_t *row_ptr, const uint32_t *col, uint64_t n_vertices,
                                             const uint32_t *sources, uint64_t n_sources, uint32_t *hops_out,
                                             void *scratch, uint64_t scratch_bytes, void *stream) {
  using namespace ss;
  if (n_vertices == 0) return SCALESIM_OK;
  if (!row_ptr || !col || !hops_out || !scratch || (n_sources > 0 && !sources) ||
      scratch_bytes < scalesim_bfs_scratch_bytes(n_vertices) || reinterpret_cast<uintptr_t>(scratch) % 16 != 0)
    return SCALESIM_E_INVALID;
  if (n_vertices >= 0xFFFFFFFFull) return SCALESIM_E_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t *cnt = static_cast<uint32_t *>(scratch);  // [0], [1]: frontier sizes (ping-pong)
  uint32_t *q[2] = {cnt + 16, cnt + 16 + (n_vertices + 1)};
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return SCALESIM_E_CUDA;
  const unsigned g = (unsigned)(sms * 8);
  const unsigned long long *rp = reinterpret_cast<const unsigned long long *>(row_ptr);
  k_bfs_init<<<g, BT, 0, st>>>(hops_out, n_vertices, sources, n_sources, q[0], cnt);
  if (n_sources > 0) k_bfs_sources<<<g, BT, 0, st>>>(hops_out, n_vertices, sources, n_sources, q[0], cnt);
  // level loop: the host reads each frontier's size (initialisation-time call: synchronous)
  for (uint32_t level = 0;; ++level) {
    const int cur = level & 1;
    uint32_t nf = 0;
    if (cudaMemcpyAsync(&nf, cnt + cur, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return SCALESIM_E_CUDA;
    if (nf == 0) break;
    if (cudaMemsetAsync(cnt + (cur ^ 1), 0, 4, st) != cudaSuccess) return SCALESIM_E_CUDA;
    uint64_t blocks = ((uint64_t)nf * 32 + BT - 1) / BT;
    if (blocks > g) blocks = g;
    k_bfs_expand<<<(unsigned)blocks, BT, 0, st>>>(rp, col, n_vertices, hops_out, q[cur], cnt + cur, q[cur ^ 1],
                                                  cnt + (cur ^ 1), level);
    if (cudaGetLastError() != cudaSuccess) return SCALESIM_E_CUDA;
  }
  return SCALESIM_OK;
}
