// sched.cu — NEXT #2: the preemptive priority load scheduler on the device (App. A
// "Load task scheduler" / "Preemption support"; SPEC.md S:291-293, S:324-327,
// S:348-356; readings R21-R23).
//
// One persistent launch runs the whole schedule: SCHED_CTAS CTAs, CTA 0 thread 0 keeps the
// task table and decides at every chunk boundary (admit the boundary's submissions and
// distance refreshes, then run the most urgent waiting task, preempting the executing one
// when a waiting task is strictly more urgent); then every CTA copies its share of the chosen
// chunk from the pinned host arena to the device arena; a grid barrier closes the slot.  The
// decision costs microseconds against a 16 MB chunk's ~300 us on the host link, so preemption
// at every boundary is free.  One channel: one chunk in flight at a time.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/scalesim.h"
#include "common.cuh"
#include "internal.h"

namespace ss {

constexpr int SCHED_CTAS = 8, SCHED_NT = 512;
constexpr uint32_t T_QUEUED = 0, T_EXECUTING = 1, T_PREEMPTED = 2, T_DONE = 3, T_CANCELLED = 4;
constexpr uint32_t NO_TASK = 0xFFFFFFFFu;

struct SchedSlot {  // the decision of one slot, read by every CTA after the first barrier
  unsigned long long src_off, dst_off, bytes;
  uint32_t task, stop;
};

__device__ __forceinline__ void sched_barrier(unsigned int *bar, unsigned int &k) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++k;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < k * gridDim.x);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(SCHED_NT) k_sched(const scalesim_load_event *ev, uint32_t n_ev, uint32_t n_agents,
                                                   float threshold, unsigned long long chunk, const uint8_t *host,
                                                   uint8_t *dev, uint32_t max_slots, scalesim_load_slot *trace,
                                                   scalesim_load_task *tasks, unsigned long long *task_src,
                                                   unsigned long long *task_dst, unsigned long long *task_bytes,
                                                   uint32_t *agent_task, uint32_t *counts, SchedSlot *slot_desc,
                                                   unsigned int *bar) {
  unsigned int k = 0;
  // CTA 0 thread 0 state (the scheduler); the table lives in global memory (tasks)
  uint32_t n_tasks = 0, exec = NO_TASK, e = 0;
  for (uint32_t slot = 0;; ++slot) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      SchedSlot sd = {0, 0, 0, NO_TASK, 0};
      // (1) this boundary's events, in order
      for (; e < n_ev && ev[e].slot <= slot; ++e) {
        const scalesim_load_event x = ev[e];
        if (x.agent >= n_agents) continue;  // (ignored: documented precondition)
        const uint32_t t = agent_task[x.agent];
        if (x.kind == SCALESIM_LOAD_SUBMIT) {
          if (t != NO_TASK) {  // coalesced: the more urgent of the two
            if (x.priority < tasks[t].priority) tasks[t].priority = x.priority;
          } else {
            scalesim_load_task nt;
            nt.agent = x.agent;
            nt.chunks = (uint32_t)(x.bytes > 0 ? (x.bytes + chunk - 1) / chunk : 1);
            nt.done = 0;
            nt.state = T_QUEUED;
            nt.priority = x.priority;
            nt.preemptions = 0;
            nt.finish_slot = NO_TASK;
            nt.pad = 0;
            tasks[n_tasks] = nt;
            task_src[n_tasks] = x.host_off;
            task_dst[n_tasks] = x.dev_off;
            task_bytes[n_tasks] = x.bytes;
            agent_task[x.agent] = n_tasks++;
          }
        } else if (t != NO_TASK && tasks[t].state != T_EXECUTING && x.priority >= threshold) {
          tasks[t].state = T_CANCELLED;  // a waiting task no longer eligible
          agent_task[x.agent] = NO_TASK;
        }
      }
      // (2) the most urgent waiting task, ties by task id
      uint32_t best = NO_TASK;
      float bp = 0.0f;
      for (uint32_t i = 0; i < n_tasks; ++i) {
        const uint32_t st = tasks[i].state;
        if (st != T_QUEUED && st != T_PREEMPTED) continue;
        const float pr = tasks[i].priority;
        if (best == NO_TASK || pr < bp) {
          best = i;
          bp = pr;
        }
      }
      if (exec == NO_TASK) {
        if (best != NO_TASK) {
          exec = best;
          tasks[best].state = T_EXECUTING;
        }
      } else if (best != NO_TASK && bp < tasks[exec].priority) {  // strictly more urgent: preempt
        tasks[exec].state = T_PREEMPTED;
        tasks[exec].preemptions++;
        exec = best;
        tasks[best].state = T_EXECUTING;
      }
      if (slot >= max_slots || (exec == NO_TASK && e >= n_ev)) {
        sd.stop = 1;
        counts[0] = slot;
        counts[1] = n_tasks;
      } else if (exec == NO_TASK) {
        trace[slot].task = NO_TASK;  // idle channel
        trace[slot].chunk = 0;
      } else {  // (3) the next chunk of the executing task (completed chunks are kept)
        const uint32_t dn = tasks[exec].done;
        const unsigned long long off = (unsigned long long)dn * chunk, b = task_bytes[exec];
        trace[slot].task = exec;
        trace[slot].chunk = dn;
        sd.task = exec;
        sd.src_off = task_src[exec] + off;
        sd.dst_off = task_dst[exec] + off;
        sd.bytes = b > off ? (b - off < chunk ? b - off : chunk) : 0ull;
        tasks[exec].done = dn + 1;
        if (dn + 1 == tasks[exec].chunks) {
          tasks[exec].state = T_DONE;
          tasks[exec].finish_slot = slot;
          agent_task[tasks[exec].agent] = NO_TASK;
          exec = NO_TASK;
        }
      }
      *slot_desc = sd;
    }
    sched_barrier(bar, k);
    const volatile SchedSlot *vs = slot_desc;  // (written by CTA 0 before the barrier)
    SchedSlot sd;
    sd.src_off = vs->src_off;
    sd.dst_off = vs->dst_off;
    sd.bytes = vs->bytes;
    sd.task = vs->task;
    sd.stop = vs->stop;
    if (sd.stop) break;
    if (sd.task != NO_TASK && sd.bytes) {
      // this CTA's share of the chunk: 16-byte vectors (offsets are 16-byte aligned), 4 in
      // flight per thread, then the byte tail
      const unsigned long long nv = sd.bytes / 16;
      const uint4 *src = reinterpret_cast<const uint4 *>(host + sd.src_off);
      uint4 *dst = reinterpret_cast<uint4 *>(dev + sd.dst_off);
      const unsigned long long stride = (unsigned long long)gridDim.x * SCHED_NT;
      unsigned long long v = (unsigned long long)blockIdx.x * SCHED_NT + threadIdx.x;
      for (; v + 3 * stride < nv; v += 4 * stride) {
        uint4 r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) r[u] = ld_stream(src + v + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) dst[v + u * stride] = r[u];
      }
      for (; v < nv; v += stride) dst[v] = ld_stream(src + v);
      if (blockIdx.x == 0 && threadIdx.x < (sd.bytes & 15ull))
        dev[sd.dst_off + nv * 16 + threadIdx.x] = host[sd.src_off + nv * 16 + threadIdx.x];
    }
    sched_barrier(bar, k);  // one chunk on the channel at a time
  }
}

__global__ void k_sched_init(uint32_t *agent_task, uint32_t n_agents, unsigned int *bar) {
  for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < n_agents; a += gridDim.x * blockDim.x)
    agent_task[a] = NO_TASK;
  if (blockIdx.x == 0 && threadIdx.x == 0) *bar = 0;
}

}  // namespace ss

using namespace ss;

static uint64_t al256(uint64_t x) { return (x + 255) / 256 * 256; }

extern "C" uint64_t scalesim_sched_scratch_bytes(uint32_t n_events, uint32_t n_agents) {
  const uint64_t n = n_events ? n_events : 1;
  return al256(24 * n) + al256(4ull * (n_agents ? n_agents : 1)) + al256(sizeof(SchedSlot)) + 256;
}

extern "C" scalesim_status scalesim_sched_run(const scalesim_load_event *events, uint32_t n_events, uint32_t n_agents,
                                              float threshold, uint64_t chunk_bytes, const void *host_arena,
                                              void *dev_arena, uint32_t max_slots, scalesim_load_slot *trace,
                                              scalesim_load_task *tasks, uint32_t *counts, void *scratch,
                                              uint64_t scratch_bytes, void *stream) {
  if ((n_events && !events) || !trace || !tasks || !counts || !scratch || chunk_bytes == 0 || chunk_bytes % 16)
    return SCALESIM_E_INVALID;
  if (scratch_bytes < scalesim_sched_scratch_bytes(n_events, n_agents) || (reinterpret_cast<uintptr_t>(scratch) & 255))
    return SCALESIM_E_INVALID;
  if (!(threshold >= 0.0f)) return SCALESIM_E_INVALID;
  if ((reinterpret_cast<uintptr_t>(host_arena) | reinterpret_cast<uintptr_t>(dev_arena)) & 15) return SCALESIM_E_INVALID;
  const uint64_t n = n_events ? n_events : 1;
  uint8_t *b = static_cast<uint8_t *>(scratch);
  unsigned long long *src = reinterpret_cast<unsigned long long *>(b);
  unsigned long long *dst = src + n, *bytes = dst + n;
  b += al256(24 * n);
  uint32_t *agent_task = reinterpret_cast<uint32_t *>(b);
  b += al256(4ull * (n_agents ? n_agents : 1));
  SchedSlot *sd = reinterpret_cast<SchedSlot *>(b);
  b += al256(sizeof(SchedSlot));
  unsigned int *bar = reinterpret_cast<unsigned int *>(b);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_sched_init<<<64, 256, 0, s>>>(agent_task, n_agents, bar);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(SCHED_CTAS);
  cfg.blockDim = dim3(SCHED_NT);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // the slot barrier needs every CTA resident
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k_sched, events, n_events, n_agents, threshold, (unsigned long long)chunk_bytes,
                         static_cast<const uint8_t *>(host_arena), static_cast<uint8_t *>(dev_arena), max_slots, trace,
                         tasks, src, dst, bytes, agent_task, counts, sd, bar) != cudaSuccess)
    return SCALESIM_E_CUDA;
  return cudaGetLastError() == cudaSuccess ? SCALESIM_OK : SCALESIM_E_CUDA;
}
