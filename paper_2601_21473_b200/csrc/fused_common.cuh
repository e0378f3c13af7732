// fused_common.cuh — device building blocks of the single-kernel plans (fused.cu: the
// shared-memory tile kernel; fused_big.cu: the streaming kernel of large contexts).  Included
// by those two translation units only.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace ss {

constexpr int FT = 1024;  // threads per CTA
constexpr int FWARPS = FT / 32;
constexpr int NB1 = 4096;  // level-1 buckets: distance bits [30:19]
constexpr int NBL = 1024;  // list-sort buckets: distance bits [30:21]
#ifndef LOAD_BATCH_V
#define LOAD_BATCH_V 2
#endif
constexpr int LOAD_BATCH = LOAD_BATCH_V;  // records in flight per thread in P1

// Integer-distance contexts (int_mode: every distance is an integer number of ticks or +inf)
// bucket level 1 by value: d < 2048 is its own bucket (single-valued), larger finite
// distances keep the float-bit buckets (bits >> 19, multi-valued) shifted down to
// [2048, 3920), and +inf is bucket 3920.  Monotone in d, so the byte-weighted select is
// unchanged; with the boundary and every list member in a single-valued bucket, list
// positions follow from per-CTA counts alone (the fast list placement below).
constexpr uint32_t IB_EXACT = 2048;  // first multi-valued bucket
constexpr uint32_t IB_INF = 3920;    // the +inf bucket
__device__ __forceinline__ uint32_t ibucket(uint32_t bits) {
  return bits < 0x45000000u ? (uint32_t)__uint_as_float(bits) : (bits >> 19) - 160u;  // 2048.0f = 0x45000000
}
__device__ __forceinline__ bool ib_multi(uint32_t b) { return b >= IB_EXACT && b < IB_INF; }

__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// epoch-tagged 48-bit payload: two 24-bit fields (ep in bits [63:48])
__device__ __forceinline__ unsigned long long pack_ep(uint32_t ep, uint32_t a, uint32_t b) {
  return ((unsigned long long)ep << 48) | ((unsigned long long)(a & 0xFFFFFFu) << 24) | (b & 0xFFFFFFu);
}
// wait until *p carries this launch's epoch (published by another CTA of the grid, which is
// co-resident); bounded: a sync failure is flagged in the status instead of hanging
__device__ __forceinline__ unsigned long long poll_ep(const unsigned long long *p, uint32_t ep,
                                                      unsigned long long *hdr) {
  unsigned long long v = ld_relaxed_u64(p);
  for (uint32_t spin = 0; (uint32_t)(v >> 48) != ep; ++spin) {
    if (spin > (1u << 22)) {
      atomicOr(reinterpret_cast<unsigned int *>(&hdr[H_STATUS]), ST_SYNC);
      break;
    }
    v = ld_relaxed_u64(p);
  }
  return v;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// %globaltimer phase stamps into the workspace (tools/timing_probe.py): compiled only into
// probe builds (-DFUSED_PROBE); each stamp is ~10 instructions and the kernel's executed code
// does not fit the 32 KB instruction cache as it is (profiles/r02_*: no_instruction stalls)
#ifdef FUSED_PROBE
#define PROBE(...) __VA_ARGS__
#else
#define PROBE(...)
#endif
#define STAMP_MAX(i) PROBE(if (threadIdx.x == 0) atomicMax(&prof[i], gtimer());)
#define STAMP0(i) PROBE(if (c == 0 && threadIdx.x == 0) prof[i] = gtimer();)

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release(unsigned int *p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid barrier for a grid of co-resident CTAs (arrive: release reduction on a counter; wait:
// acquire polling; the CTA barriers order the other threads' accesses).  bar counts arrivals
// within one launch; the k-th barrier waits for k * n arrivals (n = CTAs of the instance).
// Launch L uses bar[L & 1]; launch L-1 reset it (same stream, so every CTA of launch L-2 had
// finished).  Measured on B200 (tools/bar_bench.cu, 148 CTAs x 1024 threads): 1.22 us per
// barrier; per-CTA flags polled by a warp: 2.4 us.
struct GridBar {
  unsigned int *bar;
  unsigned int k;
  unsigned int n;  // CTAs of this instance
  __device__ __forceinline__ void sync() {
    __syncthreads();
    // a single-CTA group: the CTA barrier orders its threads' global accesses (its atomics
    // happen before the loads after it in causality order, PTX memory model)
    if (n == 1) return;
    if (threadIdx.x == 0) {
      ++k;
      red_release(bar, 1u);
      const unsigned int target = k * n;
      while (ld_acquire(bar) < target) {
      }
    }
    __syncthreads();
  }
};

// Kernel arguments: a batch of independent planner instances (one per context; C5's
// replicas x budgets), each planned by its own group of B.gsize CTAs.  A single context is
// a batch of one whose group spans every SM.
// MAXB = 1 for a single context keeps the kernel parameter block small (48 B of instance
// data instead of 7.7 KB): graph replays of the single-context step pay per launch for it.
template <int MAXB>
struct FusedArgs {
  uint32_t n_inst, gsize, fastok;
  uint32_t wsize;  // ranks per world (consecutive instances); 1: independent instances
  FusedInst inst[MAXB];
};

struct InstArgs {
  int64_t now;
  int parity;
  unsigned int epoch;  // launch number of the instance (>= 1)
  uint32_t tile;       // agents per CTA, multiple of 32
  uint32_t tw;         // tile / 32
  uint32_t fastok;     // shared memory holds the bucket-owner staging (fast list placement)
};

// dynamic shared memory carve-up
struct FSmem {
  uint32_t *keys;  // [tile] distance bits
  uint32_t *fp;    // [tile] footprint bytes; P5: in-CTA ranks
  uint32_t *memb;  // [tile] scratch: word prefixes (u64), member lists, sort buffers
  uint32_t *old_w, *elig_w, *dirty_w, *pf_w, *ev_w;  // [tw]
  uint32_t *h;     // [4 * NB1]: histogram lo/hi/min/nmax, later list counters and starts
  uint32_t *col;   // bucket-owner staging: [G][RB] CTA counts, then [4][RB] totals / offsets
};

__device__ __forceinline__ FSmem carve(uint8_t *base, uint32_t tile, uint32_t tw) {
  FSmem s;
  uint32_t *w = reinterpret_cast<uint32_t *>(base);
  s.keys = w;
  w += tile;
  s.fp = w;
  w += tile;
  s.memb = w;
  w += tile;
  s.old_w = w;
  w += tw;
  s.elig_w = w;
  w += tw;
  s.dirty_w = w;
  w += tw;
  s.pf_w = w;
  w += tw;
  s.ev_w = w;
  w += tw;
  w += (4 - ((uintptr_t)w / 4) % 4) % 4;  // 16-byte aligned: s.h is also read as u64
  s.h = w;
  s.col = w + 4 * NB1;
  return s;
}


__device__ __forceinline__ void clear_hist(uint32_t *h, int nb) {
#pragma unroll 1
  for (int b = threadIdx.x; b < nb; b += FT) {
    h[b] = 0;
    h[nb + b] = 0;
    h[2 * nb + b] = 0xFFFFFFFFu;
    h[3 * nb + b] = 0xFFFFFFFFu;
  }
}

// Level-1 histogram slot of bucket b: the bucket's low two bits go to the top, so buckets
// that differ by multiples of 4 (consecutive small integer distances: bits [22:21] fixed)
// fall in different shared-memory banks.
__device__ __forceinline__ uint32_t slot1(uint32_t b) { return (b >> 2) | ((b & 3u) << 10); }

// one lane's contribution to the byte-weighted histogram (native 32-bit shared atomics)
__device__ __forceinline__ void hist_lane(uint32_t *h, int nb, uint32_t b, uint32_t bits, uint32_t bytes) {
  atomicAdd(&h[b], bytes & 0xFFFFu);
  atomicAdd(&h[nb + b], bytes >> 16);
  atomicMin(&h[2 * nb + b], bits);
  atomicMin(&h[3 * nb + b], ~bits);
}

// this CTA's histogram: dense row (row[b] = bytes) and added to the global one (nonzero
// buckets only)
// g_coarse (level 1 only): sums over 64 consecutive buckets, one warp-reduced atomic per warp
// and bucket group that holds bytes
__device__ __forceinline__ void publish_hist(const uint32_t *h, int nb, unsigned long long *g_hist, uint32_t *g_mm,
                                             unsigned long long *row, unsigned long long *g_coarse = nullptr,
                                             bool perm = true) {
#pragma unroll 1
  for (int b = threadIdx.x; b < nb; b += FT) {
    const uint32_t q = (nb == NB1 && perm) ? slot1(b) : (uint32_t)b;
    const unsigned long long v = ((unsigned long long)h[nb + q] << 16) + h[q];
    row[b] = v;
    if (v != 0) {
      atomicAdd(&g_hist[b], v);
      if (g_mm) {
        atomicMin(&g_mm[b], h[2 * nb + q]);
        atomicMin(&g_mm[nb + b], h[3 * nb + q]);
      }
    }
    if (g_coarse && __ballot_sync(0xFFFFFFFFu, v != 0)) {  // warp-uniform (FT is a multiple of 32)
      unsigned long long t = v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
      if ((threadIdx.x & 31) == 0) atomicAdd(&g_coarse[b >> 6], t);
    }
  }
}

// Exact CTA-wide sum of a 64-bit value without a block reduction: each warp reduces the
// value's four 16-bit chunks with REDUX (a warp sums < 2^21 per chunk) and lane 0 adds them to
// four shared 32-bit counters (a CTA sums < 2^26 per chunk); after the next barrier the CTA
// total is parts_u64(acc4).  Block-wide shuffle reductions cost ~1.5 us on 1024 threads.
__device__ __forceinline__ void warp_add_u64(unsigned long long v, uint32_t *acc4) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t part = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)(v >> (16 * k)) & 0xFFFFu);
    if ((threadIdx.x & 31) == 0 && part) atomicAdd(&acc4[k], part);
  }
}
// Same for a value < 2^44 in two 22-bit chunks (a warp sums < 2^27 per chunk, a CTA of 32
// warps < 2^32): half the REDUX of warp_add_u64.  Total: parts_u44(acc2).
__device__ __forceinline__ void warp_add_u44(unsigned long long v, uint32_t *acc2) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint32_t part = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)(v >> (22 * k)) & 0x3FFFFFu);
    if ((threadIdx.x & 31) == 0 && part) atomicAdd(&acc2[k], part);
  }
}
__device__ __forceinline__ unsigned long long parts_u44(const uint32_t *acc2) {
  return (unsigned long long)acc2[0] + ((unsigned long long)acc2[1] << 22);
}
__device__ __forceinline__ unsigned long long parts_u64(const uint32_t *acc4) {
  return (unsigned long long)acc4[0] + ((unsigned long long)acc4[1] << 16) + ((unsigned long long)acc4[2] << 32) +
         ((unsigned long long)acc4[3] << 48);
}

// One out-of-line copy of the CTA-wide exclusive scan of one u64 per thread (called from several
// phases: the kernel's executed code has to stay small, see PROBE).
static __device__ __noinline__ void cta_scan1(unsigned long long (&v)[1], unsigned long long (&tot)[1]) {
  block_excl_scan_v<unsigned long long, 1, FT>(v, tot);
}
static __device__ __noinline__ void cta_scan2(unsigned long long (&v)[2], unsigned long long (&tot)[2]) {
  block_excl_scan_v<unsigned long long, 2, FT>(v, tot);
}

// The ranks of one world planned in one launch (scalesim_step_group, SCALESIM_F_LOOPBACK): each
// rank's published arrays.  The select sums the ranks' histograms after the world barrier, the
// tie prefix adds the lower ranks' bytes at D*, and the world-wide header fields are summed into
// every rank's header.  nw == 1: the context's own arrays only.
struct WorldPtrs {
  uint32_t nw, rank;
  const unsigned long long *h1[FUSED_MAX_WORLD], *h2[FUSED_MAX_WORLD], *h3[FUSED_MAX_WORLD];
  const uint32_t *m1[FUSED_MAX_WORLD], *m2[FUSED_MAX_WORLD];
  unsigned long long *acc[FUSED_MAX_WORLD], *hdr[FUSED_MAX_WORLD];
};

struct Sel {
  uint32_t prefix;
  unsigned long long below, rem;
  uint32_t dstar, all_fit, done, level_res, b_res;  // bucket (and level) holding the agents at D*
};

// Level 1 of the select by one warp and two dependent loads: the 64 coarse sums (buckets
// b >> 6), then the 64 buckets of the coarse bucket where the running byte sum crosses the
// budget.  Same result as select_level(level 1); no block-wide scan.
static __device__ void select_level1_warp(const WorldPtrs &W, int par, unsigned long long budget, Sel &sel, bool imode,
                                   unsigned long long *prof) {
  __shared__ unsigned long long s1_prev, s1_tot;
  __shared__ uint32_t s1_b, s1_min, s1_nmax;
  const bool mm = !imode;  // min / max keys kept (non-integer distances)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    ulonglong2 cc = make_ulonglong2(0, 0);
    for (uint32_t r = 0; r < W.nw; ++r) {  // coarse sums of the world
      const ulonglong2 t = reinterpret_cast<const ulonglong2 *>(W.h1[r] + 2 * NB1 + 64 * par)[lane];
      cc.x += t.x;
      cc.y += t.y;
    }
    const unsigned long long incl = warp_incl_scan(cc.x + cc.y), ex = incl - cc.x - cc.y;
    PROBE(if (blockIdx.x == 0 && lane == 0) prof[33] = gtimer();)  // coarse sums loaded and scanned
    const uint32_t m1 = __ballot_sync(0xFFFFFFFFu, incl > budget);
    const uint32_t m0 = __ballot_sync(0xFFFFFFFFu, ex + cc.x > budget);
    if (m1 == 0) {  // every eligible agent fits
      if (lane == 31) {
        s1_b = 0xFFFFFFFFu;
        s1_tot = incl;
      }
    } else {
      const int L = __ffs(m1) - 1;
      const bool even = (m0 >> L) & 1u;
      const uint32_t C = 2 * L + (even ? 0 : 1);
      const unsigned long long below = __shfl_sync(0xFFFFFFFFu, even ? ex : ex + cc.x, L);
      ulonglong2 f = make_ulonglong2(0, 0);
      uint32_t mn0 = 0xFFFFFFFFu, mn1 = 0xFFFFFFFFu, nx0 = 0xFFFFFFFFu, nx1 = 0xFFFFFFFFu;
      for (uint32_t r = 0; r < W.nw; ++r) {
        const ulonglong2 t = reinterpret_cast<const ulonglong2 *>(W.h1[r] + NB1 * par + 64 * C)[lane];
        f.x += t.x;
        f.y += t.y;
        if (mm) {
          const uint32_t *g_mm = W.m1[r] + 2 * NB1 * par;
          const uint2 mn = reinterpret_cast<const uint2 *>(g_mm + 64 * C)[lane];
          const uint2 nx = reinterpret_cast<const uint2 *>(g_mm + NB1 + 64 * C)[lane];
          mn0 = min(mn0, mn.x);
          mn1 = min(mn1, mn.y);
          nx0 = min(nx0, nx.x);
          nx1 = min(nx1, nx.y);
        }
      }
      const unsigned long long fi = below + warp_incl_scan(f.x + f.y), fe = fi - f.x - f.y;
      PROBE(if (blockIdx.x == 0 && lane == 0) prof[34] = gtimer();)  // fine buckets loaded and scanned
      const uint32_t n1 = __ballot_sync(0xFFFFFFFFu, fi > budget);  // nonzero: the coarse bucket crosses
      const uint32_t n0 = __ballot_sync(0xFFFFFFFFu, fe + f.x > budget);
      const int Lf = __ffs(n1) - 1;
      if (lane == Lf) {
        const bool ev = (n0 >> Lf) & 1u;
        s1_b = 64 * C + 2 * Lf + (ev ? 0 : 1);
        s1_prev = ev ? fe : fe + f.x;
        s1_min = ev ? mn0 : mn1;
        s1_nmax = ev ? nx0 : nx1;
      }
    }
  }
  __syncthreads();
  PROBE(if (blockIdx.x == 0 && threadIdx.x == 0) prof[35] = gtimer();)  // select barrier passed
  const uint32_t b = s1_b;
  if (b == 0xFFFFFFFFu) {
    sel.all_fit = 1;
    sel.done = 1;
    sel.dstar = 0xFFFFFFFFu;
    sel.rem = budget - s1_tot;
  } else {
    sel.below = s1_prev;
    // integer mode: value buckets below IB_EXACT and the +inf bucket hold one distance each;
    // a multi-valued bucket refines on the float bits (bits >> 19 == b + 160)
    sel.prefix |= (imode ? b + 160u : b) << 19;
    const bool int_single = imode && (b < IB_EXACT || b == IB_INF);
    const bool single = int_single || (mm && s1_min == ~s1_nmax);
    if (single) {
      sel.dstar = int_single ? (b == IB_INF ? 0x7F800000u : __float_as_uint((float)b)) : s1_min;
      sel.rem = budget - sel.below;
      sel.done = 1;
      sel.level_res = 1;
      sel.b_res = b;
    }
  }
  __syncthreads();
}

// Boundary bucket of histogram level `level` (every CTA computes the same result).
static __device__ void select_level(const WorldPtrs &W, int par, int level, unsigned long long budget, Sel &sel,
                             bool imode = false) {
  const int nb = level == 1 ? NB1 : (level == 2 ? 1024 : 512);
  const int shift = level == 1 ? 19 : (level == 2 ? 9 : 0);
  const int per = nb / FT;  // 4, 1 or 0 (level 3: threads < 512)
  __shared__ unsigned long long sh_tot, sh_prev;
  __shared__ uint32_t sh_b, sh_min, sh_nmax;
  if (threadIdx.x == 0) sh_b = 0xFFFFFFFFu;
  unsigned long long hv[4] = {0, 0, 0, 0};
  uint32_t mnv[4] = {0, 0, 0, 0}, nmxv[4] = {0, 0, 0, 0};
  unsigned long long loc = 0;
  const int mine = per > 0 ? per : ((int)threadIdx.x < nb ? 1 : 0);
  const int b0 = per > 0 ? threadIdx.x * per : threadIdx.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) {  // all loads at once (min / max with the bytes: no second round trip)
    if (k < mine) {
      mnv[k] = nmxv[k] = 0xFFFFFFFFu;
      for (uint32_t r = 0; r < W.nw; ++r) {  // the world's sums
        hv[k] += (level == 2 ? W.h2[r] : W.h3[r])[1024 * par + b0 + k];
        if (level == 2) {
          mnv[k] = min(mnv[k], W.m2[r][2048 * par + b0 + k]);
          nmxv[k] = min(nmxv[k], W.m2[r][2048 * par + nb + b0 + k]);
        }
      }
    }
  }
  const bool g_mm = level == 2;
#pragma unroll
  for (int k = 0; k < 4; ++k) loc += hv[k];
  const unsigned long long ex = block_excl_scan<unsigned long long, FT>(loc, &sh_tot);
  __syncthreads();
  unsigned long long run = sel.below + ex;
  for (int k = 0; k < mine; ++k) {
    const unsigned long long prev = run;
    run += hv[k];
    if (run > budget && prev <= budget) {  // exactly one bucket crosses (sums are monotone)
      sh_b = b0 + k;
      sh_prev = prev;
      sh_min = mnv[k];
      sh_nmax = nmxv[k];
    }
  }
  __syncthreads();
  const uint32_t b = sh_b;
  if (b == 0xFFFFFFFFu) {  // level 1 only: every eligible agent fits
    sel.all_fit = 1;
    sel.done = 1;
    sel.dstar = 0xFFFFFFFFu;
    sel.rem = budget - (sel.below + sh_tot);
  } else {
    sel.below = sh_prev;
    sel.prefix |= b << shift;
    // integer distances (level 1, no min / max kept): a bucket of exponent <= 4 (d < 32),
    // the zero bucket and the +inf bucket each hold one value, bits = b << 19
    const bool int_single = imode && level == 1 && ((b >> 4) <= 131u || b == 0xFF0u);
    const bool single = int_single || (g_mm && sh_min == ~sh_nmax);
    if (level == 3 || single) {
      sel.dstar = (level == 3) ? sel.prefix : (int_single ? (b << 19) : sh_min);
      sel.rem = budget - sel.below;
      sel.done = 1;
      sel.level_res = level;
      sel.b_res = b;
    }
  }
  __syncthreads();
}

// Stable sort of a segment of n (key, id) pairs by key, ascending, for one CTA: LSD radix
// sort with 8-bit digits over the varying bits only.  Warp w < SW owns the contiguous range
// [w*L, (w+1)*L) of the input, so (digit, warp, position) order is stable.  cnt: 256 * SW
// words of shared memory.  Buffers may be shared or global memory.  Result in (ka, ia).
constexpr int SW = 16;
static __device__ void cta_sort_pairs(uint32_t *ka, uint32_t *ia, uint32_t *kb, uint32_t *ib, uint32_t n, uint32_t *cnt) {
  if (n <= 1) return;
  __shared__ uint32_t sh_or, sh_and, sh_tot;
  if (threadIdx.x == 0) {
    sh_or = 0;
    sh_and = 0xFFFFFFFFu;
  }
  __syncthreads();
  uint32_t o = 0, a = 0xFFFFFFFFu;
  for (uint32_t e = threadIdx.x; e < n; e += FT) {
    o |= ka[e];
    a &= ka[e];
  }
  o = __reduce_or_sync(0xFFFFFFFFu, o);
  a = __reduce_and_sync(0xFFFFFFFFu, a);
  if ((threadIdx.x & 31) == 0) {
    atomicOr(&sh_or, o);
    atomicAnd(&sh_and, a);
  }
  __syncthreads();
  const uint32_t varying = sh_or ^ sh_and;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t L = (n + SW - 1) / SW;
  const uint32_t lo = warp < SW ? min(n, warp * L) : n, hi = warp < SW ? min(n, lo + L) : n;
  for (int shift = 0; shift < 32; shift += 8) {
    if (((varying >> shift) & 0xFFu) == 0) continue;
    // cnt[d * SW + w]: members of digit d in warp w's range
    for (int b = threadIdx.x; b < 256 * SW; b += FT) cnt[b] = 0;
    __syncthreads();
    for (uint32_t e = lo + lane; e < hi; e += 32) atomicAdd(&cnt[((ka[e] >> shift) & 0xFFu) * SW + warp], 1u);
    __syncthreads();
    {  // exclusive scan in (digit, warp) order: 4 consecutive entries per thread
      uint32_t v[4], sum = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[j] = cnt[threadIdx.x * 4 + j];
        sum += v[j];
      }
      uint32_t ex = block_excl_scan<uint32_t, FT>(sum, &sh_tot);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        cnt[threadIdx.x * 4 + j] = ex;
        ex += v[j];
      }
    }
    __syncthreads();
    for (uint32_t e0 = lo; e0 < hi; e0 += 32) {
      const uint32_t e = e0 + lane;
      const bool valid = e < hi;
      const uint32_t k = valid ? ka[e] : 0u, id = valid ? ia[e] : 0u;
      const uint32_t dg = valid ? ((k >> shift) & 0xFFu) : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, dg);
      if (valid) {
        const uint32_t pos = cnt[dg * SW + warp] + __popc(peers & lanemask_lt());
        kb[pos] = k;
        ib[pos] = id;
      }
      __syncwarp();
      if (valid && (peers & lanemask_lt()) == 0) cnt[dg * SW + warp] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < n; e += FT) {  // back into (ka, ia)
      ka[e] = kb[e];
      ia[e] = ib[e];
    }
    __syncthreads();
  }
}


// Stable sort of n 32-bit entries by their bits [20, 32) (the list bucket of a streaming-kernel
// candidate), ascending, for one CTA: LSD radix sort with 6-bit digits over the varying digits
// only.  Warp w owns the contiguous range [w*L, (w+1)*L), so (digit, warp, position) order is
// stable; a lane's rank among the lower lanes of its digit comes from six ballots.  cnt:
// SB_CNT words of shared memory, warp-major with a 65-word stride (a warp's lanes with different
// digits hit different banks).  Buffers may be shared or global memory.  Result in a.
constexpr uint32_t SB_STRIDE = 65, SB_CNT = FWARPS * SB_STRIDE;
static __device__ void cta_sort_buckets(uint32_t *a, uint32_t *b, uint32_t n, uint32_t *cnt) {
  if (n <= 1) return;
  __shared__ uint32_t sh_or2, sh_and2, sh_tot2;
  if (threadIdx.x == 0) {
    sh_or2 = 0;
    sh_and2 = 0xFFFFFFFFu;
  }
  __syncthreads();
  uint32_t o = 0, an = 0xFFFFFFFFu;
  for (uint32_t e = threadIdx.x; e < n; e += FT) {
    o |= a[e];
    an &= a[e];
  }
  o = __reduce_or_sync(0xFFFFFFFFu, o);
  an = __reduce_and_sync(0xFFFFFFFFu, an);
  if ((threadIdx.x & 31) == 0) {
    atomicOr(&sh_or2, o);
    atomicAnd(&sh_and2, an);
  }
  __syncthreads();
  const uint32_t varying = sh_or2 ^ sh_and2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t L = (n + FWARPS - 1) / FWARPS;
  const uint32_t lo = min(n, warp * L), hi = min(n, lo + L);
  uint32_t *src = a, *dst = b;
  for (int shift = 20; shift < 32; shift += 6) {
    if (((varying >> shift) & 0x3Fu) == 0) continue;
    // cnt[w * SB_STRIDE + d]: entries of digit d in warp w's range
    for (int x = threadIdx.x; x < (int)SB_CNT; x += FT) cnt[x] = 0;
    __syncthreads();
    for (uint32_t e = lo + lane; e < hi; e += 32) atomicAdd(&cnt[warp * SB_STRIDE + ((src[e] >> shift) & 0x3Fu)], 1u);
    __syncthreads();
    {  // exclusive scan in (digit, warp) order: entries 2t and 2t + 1 of that order per thread
      const uint32_t e0 = threadIdx.x * 2, e1 = e0 + 1;
      const uint32_t a0 = (e0 % FWARPS) * SB_STRIDE + e0 / FWARPS, a1 = (e1 % FWARPS) * SB_STRIDE + e1 / FWARPS;
      const uint32_t v0 = cnt[a0], v1 = cnt[a1];
      const uint32_t ex = block_excl_scan<uint32_t, FT>(v0 + v1, &sh_tot2);
      cnt[a0] = ex;
      cnt[a1] = ex + v0;
    }
    __syncthreads();
    for (uint32_t e0 = lo; e0 < hi; e0 += 32) {
      const uint32_t e = e0 + lane;
      const bool valid = e < hi;
      const uint32_t x = valid ? src[e] : 0u, dg = (x >> shift) & 0x3Fu;
      uint32_t peers = __ballot_sync(0xFFFFFFFFu, valid);
#pragma unroll
      for (int bb = 0; bb < 6; ++bb) {
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (dg >> bb) & 1u);
        peers &= ((dg >> bb) & 1u) ? bal : ~bal;
      }
      const uint32_t below = __popc(peers & lanemask_lt());
      const uint32_t c0 = valid ? cnt[warp * SB_STRIDE + dg] : 0u;
      __syncwarp();
      if (valid) {
        dst[c0 + below] = x;
        if (below == 0) cnt[warp * SB_STRIDE + dg] = c0 + __popc(peers);
      }
      __syncwarp();
    }
    __syncthreads();
    uint32_t *t = src;
    src = dst;
    dst = t;
  }
  if (src != a) {
    for (uint32_t e = threadIdx.x; e < n; e += FT) a[e] = src[e];
    __syncthreads();
  }
}


}  // namespace ss
