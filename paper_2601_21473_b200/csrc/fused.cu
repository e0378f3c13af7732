// fused.cu — one persistent kernel per planning step (world == 1).
//
// One CTA per SM (1024 threads, co-residency checked at init); CTA c owns the contiguous
// agent tile [c*T, (c+1)*T), so CTA order is id order.  Phases:
//   P1  score the tile (a1, a2): batched 128-bit record loads, distance, eligibility; keys,
//       footprints and residency/eligibility/dirty bits stay in shared memory; byte-weighted
//       histogram of distance bits [30:19] (4096 buckets) with per-bucket min/max key, added
//       to the global histogram with atomics
//   --- grid barrier
//   P2  every CTA resolves the boundary distance D* from the global histogram (a3); levels
//       2 ([18:9]) and 3 ([8:0]) run, each behind a barrier, only when the boundary bucket
//       holds several distances
//   P3  tie group: each CTA publishes its bytes at d == D*, then sums the preceding CTAs'
//       values (per-CTA flags tagged with the launch epoch: no barrier)
//   P4  emit (a4, a5): kept bits, new residency words, byte totals; per-CTA member counts of
//       the two lists per 1024-bucket of distance bits [30:21] (dense rows) + global totals
//   --- grid barrier
//   P5  stable bucket sort of the lists: slot = bucket start + members of that bucket in the
//       preceding CTAs (prefetch: ascending id) or following CTAs (evict: descending id) +
//       in-CTA rank
//   --- grid barrier (only when the members of a list bucket hold several distances)
//   P6  such segments are re-sorted by (distance, id): ranks by counting, the comparisons
//       spread evenly over all CTAs (short segments), or a radix sort by one CTA (long ones)
// Decisions follow DESIGN.md §3 exactly as the multi-kernel path (kernels.cu) does; both give
// bit-identical plans (tests/test_gpu_parity.py runs both).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace ss {

constexpr int FT = 1024;  // threads per CTA
constexpr int FWARPS = FT / 32;
constexpr int NB1 = 4096;  // level-1 buckets: distance bits [30:19]
constexpr int NBL = 1024;  // list-sort buckets: distance bits [30:21]
constexpr int LOAD_BATCH = 4;  // records in flight per thread in P1

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

// Grid barrier for a grid of co-resident CTAs.  bar counts arrivals within one launch; the
// k-th barrier waits for k * n arrivals (n = CTAs of the instance).  Launch L uses bar[L & 1]; launch L-1 reset it
// (same stream, so every CTA of launch L-2 had finished).
struct GridBar {
  unsigned int *bar;
  unsigned int k;
  unsigned int n;  // CTAs of this instance
  __device__ __forceinline__ void sync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++k;
      __threadfence();
      atomicAdd(bar, 1u);
      const unsigned int target = k * n;
      while (ld_acquire(bar) < target) __nanosleep(40);  // back off: 148 CTAs poll one line
      __threadfence();
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
  uint32_t n_inst, gsize;
  FusedInst inst[MAXB];
};

struct InstArgs {
  int64_t now;
  int parity;
  unsigned int epoch;  // launch number of the instance (>= 1), tags the per-CTA tie flags
  uint32_t tile;       // agents per CTA, multiple of 32
  uint32_t tw;         // tile / 32
};

// dynamic shared memory carve-up
struct FSmem {
  uint32_t *keys;  // [tile] distance bits
  uint32_t *fp;    // [tile] footprint bytes; P5: in-CTA ranks
  uint32_t *memb;  // [tile] scratch: word prefixes (u64), member lists, sort buffers
  uint32_t *old_w, *elig_w, *dirty_w, *pf_w, *ev_w;  // [tw]
  uint32_t *h;     // [4 * NB1]: histogram lo/hi/min/nmax, later list counters and starts
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
  return s;
}

size_t fused_smem_bytes(uint32_t tile) {
  const uint32_t tw = tile / 32;
  return (size_t)4 * (3 * tile + 5 * tw + 4 * NB1) + 16;
}

__device__ __forceinline__ void clear_hist(uint32_t *h, int nb) {
  for (int b = threadIdx.x; b < nb; b += FT) {
    h[b] = 0;
    h[nb + b] = 0;
    h[2 * nb + b] = 0xFFFFFFFFu;
    h[3 * nb + b] = 0xFFFFFFFFu;
  }
}

// one lane's contribution to the byte-weighted histogram (native 32-bit shared atomics)
__device__ __forceinline__ void hist_lane(uint32_t *h, int nb, uint32_t b, uint32_t bits, uint32_t bytes) {
  atomicAdd(&h[b], bytes & 0xFFFFu);
  atomicAdd(&h[nb + b], bytes >> 16);
  atomicMin(&h[2 * nb + b], bits);
  atomicMin(&h[3 * nb + b], ~bits);
}

// this CTA's histogram: dense row (row[b] = bytes) and added to the global one (nonzero
// buckets only)
__device__ __forceinline__ void publish_hist(const uint32_t *h, int nb, unsigned long long *g_hist, uint32_t *g_mm,
                                             unsigned long long *row) {
  for (int b = threadIdx.x; b < nb; b += FT) {
    const unsigned long long v = ((unsigned long long)h[nb + b] << 16) + h[b];
    row[b] = v;
    if (v != 0) {
      atomicAdd(&g_hist[b], v);
      if (g_mm) {
        atomicMin(&g_mm[b], h[2 * nb + b]);
        atomicMin(&g_mm[nb + b], h[3 * nb + b]);
      }
    }
  }
}

struct Sel {
  uint32_t prefix;
  unsigned long long below, rem;
  uint32_t dstar, all_fit, done, level_res, b_res;  // bucket (and level) holding the agents at D*
};

// Boundary bucket of histogram level `level` (every CTA computes the same result).
__device__ void select_level(const unsigned long long *g_hist, const uint32_t *g_mm, int level,
                             unsigned long long budget, Sel &sel) {
  const int nb = level == 1 ? NB1 : (level == 2 ? 1024 : 512);
  const int shift = level == 1 ? 19 : (level == 2 ? 9 : 0);
  const int per = nb / FT;  // 4, 1 or 0 (level 3: threads < 512)
  __shared__ unsigned long long sh_tot, sh_prev;
  __shared__ uint32_t sh_b;
  if (threadIdx.x == 0) sh_b = 0xFFFFFFFFu;
  unsigned long long hv[4] = {0, 0, 0, 0};
  unsigned long long loc = 0;
  const int mine = per > 0 ? per : ((int)threadIdx.x < nb ? 1 : 0);
  const int b0 = per > 0 ? threadIdx.x * per : threadIdx.x;
  for (int k = 0; k < mine; ++k) {
    hv[k] = g_hist[b0 + k];
    loc += hv[k];
  }
  const unsigned long long ex = block_excl_scan<unsigned long long, FT>(loc, &sh_tot);
  __syncthreads();
  unsigned long long run = sel.below + ex;
  for (int k = 0; k < mine; ++k) {
    const unsigned long long prev = run;
    run += hv[k];
    if (run > budget && prev <= budget) {  // exactly one bucket crosses (sums are monotone)
      sh_b = b0 + k;
      sh_prev = prev;
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
    const bool single = g_mm != nullptr && g_mm[b] == ~g_mm[nb + b];
    if (level == 3 || single) {
      sel.dstar = (level == 3) ? sel.prefix : g_mm[b];
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
__device__ void cta_sort_pairs(uint32_t *ka, uint32_t *ia, uint32_t *kb, uint32_t *ib, uint32_t n, uint32_t *cnt) {
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

template <int MAXB>
__global__ void __launch_bounds__(FT, 1) k_fused_plan(const __grid_constant__ FusedArgs<MAXB> B) {
  const uint32_t gi = blockIdx.x / B.gsize;
  const uint32_t c = blockIdx.x % B.gsize, G = B.gsize;
  const FusedInst &I = B.inst[gi];
  __shared__ __align__(16) Params sp;  // the instance's parameters (device copy + per-launch fields)
  {
    const uint32_t *src = reinterpret_cast<const uint32_t *>(I.params);
    uint32_t *dst = reinterpret_cast<uint32_t *>(&sp);
    for (uint32_t q = threadIdx.x; q < sizeof(Params) / 4; q += FT) dst[q] = src[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    sp.rec = I.rec;
    sp.kin = I.kin;
    sp.cur = (int)I.cur;
  }
  __syncthreads();
  const Params &p = sp;
  const InstArgs A = {I.now, (int)I.parity, I.epoch, I.tile, I.tile / 32};
  const Dev &d = p.d;
  GridBar grid{d.f_bar + A.parity, 0u, G};
  unsigned long long *prof = d.f_prof;
  if (threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    atomicMin(&prof[0], t);
    if (c == 0) prof[2] = t;
  }
  if (c == 0 && threadIdx.x == 0) d.f_bar[A.parity ^ 1] = 0u;  // for launch L+1
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const FSmem s = carve(smem_raw, A.tile, A.tw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = (uint64_t)c * A.tile;
  const uint32_t n_here =
      base >= p.n_local ? 0u : (uint32_t)((p.n_local - base) < A.tile ? (p.n_local - base) : A.tile);
  const uint32_t tw_here = (n_here + 31) / 32;
  const int par = A.parity;
  // accumulators of this launch: [0] zero-distance bytes [1] h2d [2] d2h [3] tie kept
  // [4] eligible agents [5] status
  unsigned long long *acc = d.f_acc + 8 * par;
  const uint32_t *bm_old = d.bm[p.cur];
  uint32_t *bm_new = d.bm[p.cur ^ 1];

  // ---------------- P1: score + level-1 histogram
  // per-thread copies of the parameters used per agent (Params lives in shared memory)
  const float hop_scale = p.hop_scale, th0 = p.theta[0], th1 = p.theta[1], th2 = p.theta[2];
  const uint64_t n_kin = p.n_kin;
  const float *dint = d.dint;
  const uint4 *rec = p.rec + base;
  uint32_t *gkeys = p.keep_dist ? d.keys + base : nullptr;
  const int64_t now = A.now;
  clear_hist(s.h, NB1);
  for (uint32_t w = threadIdx.x; w < A.tw; w += FT) s.old_w[w] = w < tw_here ? bm_old[base / 32 + w] : 0u;
  __syncthreads();
  uint32_t st = 0;
  unsigned long long zero_b = 0;
  for (uint32_t k0 = 0; k0 < A.tw * 32; k0 += LOAD_BATCH * FT) {
    uint4 r[LOAD_BATCH];
#pragma unroll
    for (int j = 0; j < LOAD_BATCH; ++j) {  // all loads in flight before any use
      const uint32_t k = k0 + j * FT + threadIdx.x;
      r[j] = k < n_here ? ld_stream(rec + k) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < LOAD_BATCH; ++j) {
      const uint32_t k = k0 + j * FT + threadIdx.x;
      if (k >= A.tw * 32) continue;  // warp-uniform (tw * 32 is a multiple of 32)
      const bool valid = k < n_here;
      const bool res = (s.old_w[k >> 5] >> (k & 31)) & 1u;
      const uint32_t ph = r[j].z & 3u, cl = (r[j].z >> 2) & 3u;
      float dist, th;
      if (__ballot_sync(0xFFFFFFFFu, valid && cl != 0u)) {
        // the warp holds interaction / diffusion / malformed records: general definition
        dist = valid ? distance_of(r[j], now, hop_scale, dint, n_kin, st) : 0.0f;
        th = (cl & 2u) ? ((cl & 1u) ? 0.0f : th2) : ((cl & 1u) ? th1 : th0);
      } else {
        // independent agents only: remaining action ticks, 0 while in an LLM
        // phase, +inf when idle — the same values distance_of gives for class 0
        const int64_t remain = (int64_t)r[j].x - now;
        const float d_action = remain <= 0 ? 0.0f : __ll2float_rn(remain);
        dist = (ph == 1u || ph == 2u) ? 0.0f : (ph == 3u ? __int_as_float(0x7F800000) : d_action);
        th = th0;
      }
      const uint32_t bits = __float_as_uint(dist);
      const bool elig = valid && (res || dist == 0.0f || dist < th);
      s.keys[k] = bits;
      s.fp[k] = r[j].y;
      if (gkeys && valid) gkeys[k] = bits;
      const uint32_t eb = __ballot_sync(0xFFFFFFFFu, elig);
      const uint32_t db = __ballot_sync(0xFFFFFFFFu, valid && ((r[j].z >> 4) & 1u));
      if (lane == 0) {
        s.elig_w[k >> 5] = eb;
        s.dirty_w[k >> 5] = db;
      }
      if (elig) hist_lane(s.h, NB1, bits >> 19, bits, r[j].y);
      if (valid && dist == 0.0f) zero_b += r[j].y;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&prof[25], gtimer());  // P1 loop done
  // this CTA's level-1 bytes: dense row (its column entry gives the tie prefix in P3) and
  // the global sum
  publish_hist(s.h, NB1, d.f_hist1 + NB1 * par, d.f_mm1 + 2 * NB1 * par, d.f_rows1 + (uint64_t)c * NB1);
  if (threadIdx.x == 0) atomicMax(&prof[26], gtimer());  // published
  zero_b = block_sum<unsigned long long, FT>(zero_b);
  st = __reduce_or_sync(0xFFFFFFFFu, st);
  if (lane == 0 && st) atomicOr(reinterpret_cast<unsigned int *>(&acc[5]), st);
  if (threadIdx.x == 0 && zero_b) atomicAdd(&acc[0], zero_b);
  if (threadIdx.x == 0) atomicMax(&prof[11], gtimer());
  if (c == 0 && threadIdx.x == 0) prof[3] = gtimer();
  grid.sync();
  if (c == 0 && threadIdx.x == 0) prof[4] = gtimer();

  // ---------------- P2: select
  {  // clear the other parity's accumulators for the next launch, spread over the CTAs
    const int q = par ^ 1;
    const uint32_t gt = c * FT + threadIdx.x, gs = G * FT;
    for (uint32_t b = gt; b < NB1; b += gs) {
      d.f_hist1[NB1 * q + b] = 0;
      d.f_mm1[2 * NB1 * q + b] = 0xFFFFFFFFu;
      d.f_mm1[2 * NB1 * q + NB1 + b] = 0xFFFFFFFFu;
    }
    for (uint32_t b = gt; b < 2 * NBL; b += gs) d.f_tot[2 * NBL * q + b] = 0;
    for (uint32_t b = gt; b < 4 * NBL; b += gs) d.f_lmm[4 * NBL * q + b] = 0xFFFFFFFFu;
    for (uint32_t b = gt; b < 1024; b += gs) {
      d.f_hist2[1024 * q + b] = 0;
      d.f_hist3[1024 * q + b] = 0;
      d.f_mm2[2048 * q + b] = 0xFFFFFFFFu;
      d.f_mm2[2048 * q + 1024 + b] = 0xFFFFFFFFu;
    }
    if (gt < 8) d.f_acc[8 * q + gt] = 0;
  }
  const uint32_t *mm1 = d.f_mm1 + 2 * NB1 * par;
  Sel sel = {0, 0, 0, 0xFFFFFFFFu, 0, 0, 1, 0};
  select_level(d.f_hist1 + NB1 * par, mm1, 1, p.budget, sel);
  for (int level = 2; level <= 3 && !sel.done; ++level) {
    const int hi_shift = level == 2 ? 19 : 9, shift = level == 2 ? 9 : 0;
    const int nb = level == 2 ? 1024 : 512;
    const uint32_t want = sel.prefix >> hi_shift;
    clear_hist(s.h, nb);
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < n_here; k += FT) {
      const uint32_t bits = s.keys[k];
      if (((s.elig_w[k >> 5] >> (k & 31)) & 1u) && (bits >> hi_shift) == want)
        hist_lane(s.h, nb, (bits >> shift) & (nb - 1), bits, s.fp[k]);
    }
    __syncthreads();
    unsigned long long *gh = level == 2 ? d.f_hist2 + 1024 * par : d.f_hist3 + 1024 * par;
    uint32_t *gm = level == 2 ? d.f_mm2 + 2048 * par : nullptr;
    publish_hist(s.h, nb, gh, gm, (level == 2 ? d.f_rows2 : d.f_rows3) + (uint64_t)c * 1024);
    grid.sync();
    select_level(gh, gm, level, p.budget, sel);
  }
  const bool all_fit = sel.all_fit;
  const uint32_t dstar = sel.dstar;
  if (c == 0 && threadIdx.x == 0) prof[9] = gtimer();

  // ---------------- P3: tie group: id-order prefix of the bytes at d == D*
  unsigned long long *word_tie = reinterpret_cast<unsigned long long *>(s.memb);  // [tw]
  for (uint32_t w = warp; w < A.tw; w += FWARPS) {
    const uint32_t k = w * 32 + lane;
    const bool tie = !all_fit && ((s.elig_w[w] >> lane) & 1u) && s.keys[k] == dstar;
    unsigned long long v = 0;
    if (__ballot_sync(0xFFFFFFFFu, tie)) v = warp_sum_u32_exact(tie ? s.fp[k] : 0u);  // most words: no tie
    if (lane == 0) word_tie[w] = v;
  }
  __syncthreads();
  __shared__ unsigned long long sh_tie_excl, sh_chunk;
  {  // exclusive scan over the tile's words (tw <= FUSED_MAX_TILE / 32 <= FT: one word per thread)
    const uint32_t w = threadIdx.x;
    const unsigned long long v = w < A.tw ? word_tie[w] : 0ull;
    const unsigned long long ex = block_excl_scan<unsigned long long, FT>(v, &sh_chunk);
    if (w < A.tw) word_tie[w] = ex;
    __syncthreads();
  }
  {  // preceding CTAs: their bytes in the resolving bucket (published rows; one load each)
    unsigned long long t = 0;
    if (!all_fit && threadIdx.x < c) {
      const unsigned long long *rows = sel.level_res == 1 ? d.f_rows1 : (sel.level_res == 2 ? d.f_rows2 : d.f_rows3);
      const uint32_t stride = sel.level_res == 1 ? NB1 : 1024;
      t = rows[(uint64_t)threadIdx.x * stride + sel.b_res];
    }
    t = block_sum<unsigned long long, FT>(t);
    if (threadIdx.x == 0) sh_tie_excl = t;
  }
  __syncthreads();
  if (c == 0 && threadIdx.x == 0) prof[10] = gtimer();
  if (threadIdx.x == 0) atomicMax(&prof[14], gtimer());

  // ---------------- P4: emit
  uint32_t *cnt_pf = s.h, *cnt_ev = s.h + NBL;  // per-CTA list members per list bucket
  uint32_t *mm_l = s.h + 10 * NBL;  // [4][NBL]: prefetch min, prefetch ~max, evict min, evict ~max
  for (int b = threadIdx.x; b < 2 * NBL; b += FT) s.h[b] = 0;
  for (int b = threadIdx.x; b < 4 * NBL; b += FT) mm_l[b] = 0xFFFFFFFFu;
  __syncthreads();
  unsigned long long h2d = 0, d2h = 0, tie_kept = 0;
  uint32_t n_el = 0;
  constexpr uint32_t WB_CAP = 5 * NBL;
  uint32_t *wb_list = s.h + 2 * NBL;  // evicted dirty agents of this tile (s.h[2NBL, 7NBL) is free here)
  __shared__ uint32_t sh_nwb;
  if (threadIdx.x == 0) sh_nwb = 0;
  __syncthreads();
  for (uint32_t w = warp; w < A.tw; w += FWARPS) {
    const uint32_t k = w * 32 + lane;
    const bool el = (s.elig_w[w] >> lane) & 1u;  // 0 beyond n_here
    const uint32_t key = s.keys[k];
    const bool tie = el && !all_fit && key == dstar;
    const uint32_t fp = s.fp[k];
    bool tie_ok = false;
    if (__ballot_sync(0xFFFFFFFFu, tie)) {  // id-order inclusive prefix of the tie bytes
      unsigned long long incl = tie ? fp : 0u;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
      }
      incl += sh_tie_excl + word_tie[w];
      tie_ok = tie && incl <= sel.rem;
    }
    const bool kept = el && (all_fit || key < dstar || tie_ok);
    if (tie && kept) tie_kept += fp;
    const uint32_t kw = __ballot_sync(0xFFFFFFFFu, kept);
    const uint32_t old = s.old_w[w];
    const uint32_t pfw = kw & ~old, evw = old & ~kw;
    if (lane == 0) {
      if (w < tw_here) bm_new[base / 32 + w] = kw;
      s.pf_w[w] = pfw;
      s.ev_w[w] = evw;
      n_el += __popc(s.elig_w[w]);
    }
    if ((pfw >> lane) & 1u) {
      h2d += fp;
      atomicAdd(&cnt_pf[key >> 21], 1u);
      atomicMin(&mm_l[key >> 21], key);
      atomicMin(&mm_l[NBL + (key >> 21)], ~key);
    }
    if ((evw >> lane) & 1u) {
      if ((s.dirty_w[w] >> lane) & 1u) {  // R13: write-back bytes, loaded after the loop
        const uint32_t slot = atomicAdd(&sh_nwb, 1u);
        if (slot < WB_CAP) wb_list[slot] = k;
        else d2h += d.wb_bytes[base + k];
      }
      atomicAdd(&cnt_ev[key >> 21], 1u);
      atomicMin(&mm_l[2 * NBL + (key >> 21)], key);
      atomicMin(&mm_l[3 * NBL + (key >> 21)], ~key);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&prof[27], gtimer());  // P4 word loop done
  for (uint32_t q = threadIdx.x; q < min(sh_nwb, WB_CAP); q += FT) d2h += d.wb_bytes[base + wb_list[q]];
  uint32_t *cpf = d.f_cta_cpf + (uint64_t)c * NBL, *cev = d.f_cta_cev + (uint64_t)c * NBL;
  uint32_t *tot_pf = d.f_tot + 2 * NBL * par, *tot_ev = d.f_tot + 2 * NBL * par + NBL;
  {
    const int b = threadIdx.x;  // NBL == FT
    const uint32_t a = cnt_pf[b], e = cnt_ev[b];
    cpf[b] = a;
    cev[b] = e;
    if (a) {
      atomicAdd(&tot_pf[b], a);
      atomicMin(&d.f_lmm[4 * NBL * par + b], mm_l[b]);
      atomicMin(&d.f_lmm[4 * NBL * par + NBL + b], mm_l[NBL + b]);
    }
    if (e) {
      atomicAdd(&tot_ev[b], e);
      atomicMin(&d.f_lmm[4 * NBL * par + 2 * NBL + b], mm_l[2 * NBL + b]);
      atomicMin(&d.f_lmm[4 * NBL * par + 3 * NBL + b], mm_l[3 * NBL + b]);
    }
  }
  if (threadIdx.x == 0) atomicMax(&prof[28], gtimer());  // rows published
  {
    unsigned long long sums[4] = {h2d, d2h, tie_kept, (unsigned long long)n_el};
    block_sum_v<unsigned long long, 4, FT>(sums);
    if (threadIdx.x < 4 && sums[threadIdx.x]) atomicAdd(&acc[1 + threadIdx.x], sums[threadIdx.x]);
  }
  if (threadIdx.x == 0) atomicMax(&prof[12], gtimer());
  if (c == 0 && threadIdx.x == 0) prof[5] = gtimer();
  grid.sync();
  if (c == 0 && threadIdx.x == 0) prof[6] = gtimer();

  // ---------------- P5: stable bucket sort of the lists
  uint32_t *g_pf = s.h + 2 * NBL, *g_ev = s.h + 3 * NBL;  // first slot of this CTA's members per bucket
  uint32_t *tpf = s.h + 8 * NBL, *tev = s.h + 9 * NBL;    // list bucket totals (shared copy)
  // list bucket b needs the re-sort by full distance iff its members hold several distances
  uint32_t *lmulti = s.h + 7 * NBL;  // bit 0: prefetch list, bit 1: evict list
  {
    const uint32_t b = threadIdx.x;
    const uint32_t *lmm = d.f_lmm + 4 * NBL * par;
    const uint32_t mp = lmm[b], xp = ~lmm[NBL + b], me = lmm[2 * NBL + b], xe = ~lmm[3 * NBL + b];
    lmulti[b] = ((mp != 0xFFFFFFFFu && mp != xp) ? 1u : 0u) | ((me != 0xFFFFFFFFu && me != xe) ? 2u : 0u);
  }
  __shared__ uint32_t sh_npf, sh_nev, sh_mpf, sh_mev, sh_need;
  {
    const uint32_t b = threadIdx.x, rb = NBL - 1 - b;  // NBL == FT; evict: descending buckets
    uint32_t v[2] = {tot_pf[b], tot_ev[rb]}, tt[2];
    tpf[b] = v[0];
    tev[rb] = v[1];
    block_excl_scan_v<uint32_t, 2, FT>(v, tt);
    g_pf[b] = v[0];
    g_ev[rb] = v[1];
    if (threadIdx.x == 0) {
      sh_npf = tt[0];
      sh_nev = tt[1];
    }
  }
  // members in list order (prefetch ascending id, evict descending id; tile-local indices)
  // into memb; one word per thread (tw <= FT)
  {
    const uint32_t w = threadIdx.x;
    const uint32_t pw = w < A.tw ? s.pf_w[w] : 0u, ew = w < A.tw ? s.ev_w[w] : 0u;
    uint32_t v[2] = {(uint32_t)__popc(pw), (uint32_t)__popc(ew)}, tt[2];
    block_excl_scan_v<uint32_t, 2, FT>(v, tt);
    const uint32_t need = __syncthreads_or(lmulti[threadIdx.x] != 0u);
    if (threadIdx.x == 0) {
      sh_mpf = tt[0];
      sh_mev = tt[1];
      sh_need = need;
    }
    uint32_t m = pw, o = v[0];
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      s.memb[o++] = w * 32 + bit;
    }
    m = ew;
    o = tt[0] + tt[1] - 1 - v[1];
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      s.memb[o--] = w * 32 + bit;
    }
  }
  __syncthreads();
  const uint32_t m_pf = sh_mpf, m_ev = sh_mev;
  uint32_t *mem_pf = s.memb, *mem_ev = s.memb + m_pf;
  // own nonzero list buckets (for the column prefix)
  uint32_t *own_b = s.h + 6 * NBL;
  __shared__ uint32_t sh_nown;
  if (threadIdx.x == 0) sh_nown = 0;
  __syncthreads();
  if (cnt_pf[threadIdx.x] || cnt_ev[threadIdx.x]) own_b[atomicAdd(&sh_nown, 1u)] = threadIdx.x;
  __syncthreads();
  // (a) warps 0/1: in-CTA rank of every member within its bucket (list order), into fp[]
  // (b) other warps: members of the same bucket in the preceding (prefetch) / following
  //     (evict) CTAs, added to the bucket starts
  if (warp < 2) {
    const uint32_t *mem = warp == 0 ? mem_pf : mem_ev;
    const uint32_t m = warp == 0 ? m_pf : m_ev;
    uint32_t *run = warp == 0 ? s.h + 4 * NBL : s.h + 5 * NBL;
    for (uint32_t b = lane; b < NBL; b += 32) run[b] = 0;
    __syncwarp();
    for (uint32_t e0 = 0; e0 < m; e0 += 32) {
      const uint32_t e = e0 + lane;
      const bool on = e < m;
      const uint32_t bk = on ? (s.keys[mem[e]] >> 21) : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, bk);
      uint32_t r = 0;
      if (on) r = run[bk] + __popc(peers & lanemask_lt());
      __syncwarp();
      if (on && (peers & lanemask_lt()) == 0) run[bk] += __popc(peers);
      __syncwarp();
      if (on) s.fp[(warp == 0 ? 0 : m_pf) + e] = r;
    }
  } else {
    const uint32_t nown = sh_nown;
    for (uint32_t j = warp - 2; j < nown; j += FWARPS - 2) {
      const uint32_t b = own_b[j];
      const bool has_pf = cnt_pf[b] != 0, has_ev = cnt_ev[b] != 0;
      uint32_t ppf = 0, pev = 0;
      for (uint32_t q = lane; q < G; q += 32) {
        if (has_pf && q < c) ppf += d.f_cta_cpf[(uint64_t)q * NBL + b];
        if (has_ev && q > c) pev += d.f_cta_cev[(uint64_t)q * NBL + b];
      }
      ppf = __reduce_add_sync(0xFFFFFFFFu, ppf);
      pev = __reduce_add_sync(0xFFFFFFFFu, pev);
      if (lane == 0) {
        g_pf[b] += ppf;
        g_ev[b] += pev;
      }
    }
  }
  __syncthreads();
  // members of buckets holding several distances are also staged (key, id) by slot for P6
  for (uint32_t e = threadIdx.x; e < m_pf + m_ev; e += FT) {
    const uint32_t k = s.memb[e];
    const uint32_t key = s.keys[k];
    const uint32_t bk = key >> 21;
    const uint32_t id = (uint32_t)(p.shard_begin + base + k);
    if (e < m_pf) {
      const uint32_t slot = g_pf[bk] + s.fp[e];
      d.pf_ids[slot] = id;
      if (lmulti[bk] & 1u) {
        d.sort_ka[slot] = key;
        d.sort_va[slot] = id;
      }
    } else {
      const uint32_t slot = g_ev[bk] + s.fp[e];
      d.ev_ids[slot] = id;
      if (lmulti[bk] & 2u) {
        d.f_sk2[slot] = ~key;  // evict: descending (distance, id) = ascending complement
        d.f_sv2[slot] = id;
      }
    }
  }
  // header (CTA 0): all accumulators are complete after the last barrier
  if (c == 0 && threadIdx.x == 0) {
    unsigned long long *H = d.header;
    H[H_N_PF] = sh_npf;
    H[H_N_EV] = sh_nev;
    H[H_H2D] = acc[1];
    H[H_D2H] = acc[2];
    H[H_CUT_BITS] = all_fit ? 0xFFFFFFFFull : dstar;
    H[H_CUT_REM] = sel.rem;
    H[H_KEPT] = (p.budget - sel.rem) + (all_fit ? 0ull : acc[3]);
    H[H_N_ELIG] = acc[4];
    uint32_t status = (uint32_t)acc[5] | d.state->status;  // + BAD_KIN/BAD_RECORD of k_int_compact
    if (acc[0] > p.budget) status |= ST_INSUFFICIENT;
    H[H_STATUS] = status;
    H[H_SEQ] += 1;
  }
  if (threadIdx.x == 0) atomicMax(&prof[13], gtimer());
  if (c == 0 && threadIdx.x == 0) prof[7] = gtimer();
  if (!sh_need) {  // uniform: every CTA computed it from the same global totals
    if (threadIdx.x == 0) atomicMax(&prof[1], gtimer());
    return;
  }
  grid.sync();
  if (c == 0 && threadIdx.x == 0) prof[8] = gtimer();

  // ---------------- P6: order the segments of list buckets whose members hold several
  // distances by (distance, id).  Segment table in list order (prefetch list first).  Short
  // segments: every element's rank is counted against its segment's keys, the comparison
  // work spread evenly over all CTAs; long ones are radix-sorted in global memory by one CTA.
  uint32_t *seg_start = s.h + 10 * NBL, *seg_len = s.h + 12 * NBL;  // [2 * NBL] each
  __shared__ uint32_t sh_nsmall, sh_nbig, sh_tmp, sh_gp, sh_nds;
  uint32_t *dense_gp = s.h + 14 * NBL;  // [2 * NBL]: nonempty short segments in list order
  uint32_t big_mask = 0, big_x = 0;  // this thread's long segments (bits for gp 2t, 2t+1) and their index
  {
    // thread t owns the (list, bucket) positions 2t, 2t+1 of the 2048 in list order
    // (prefetch buckets ascending, then evict buckets descending)
    uint32_t len[2], small[2], big[2];
    for (int q = 0; q < 2; ++q) {
      const uint32_t gp = 2 * threadIdx.x + q;
      const int list = gp < NBL ? 0 : 1;
      const uint32_t b = list == 0 ? gp : (2 * NBL - 1 - gp);
      len[q] = list == 0 ? tpf[b] : tev[b];
      const bool mv = (lmulti[b] >> list) & 1u;
      small[q] = (mv && 4 * len[q] <= 3 * A.tile) ? 1u : 0u;  // sortable in shared memory
      big[q] = (mv && 4 * len[q] > 3 * A.tile) ? 1u : 0u;
    }
    // segment start within its list (the evict list starts at position NBL)
    uint32_t v[4] = {len[0] + len[1], small[0] * len[0] + small[1] * len[1], big[0] + big[1], small[0] + small[1]};
    uint32_t tt[4];
    block_excl_scan_v<uint32_t, 4, FT>(v, tt);
    const uint32_t lx = v[0], dx = v[3];
    big_x = v[2];
    if (threadIdx.x == 0) {
      sh_nsmall = tt[1];
      sh_nbig = tt[2];
      sh_nds = tt[3];
    }
    const uint32_t start0 = (2 * threadIdx.x < NBL) ? lx : lx - sh_npf;
    const uint32_t start1 = (2 * threadIdx.x + 1 < NBL) ? lx + len[0] : lx + len[0] - sh_npf;
    if (small[0]) dense_gp[dx] = 2 * threadIdx.x;
    if (small[1]) dense_gp[dx + small[0]] = 2 * threadIdx.x + 1;
    big_mask = big[0] | (big[1] << 1);
    seg_start[2 * threadIdx.x] = start0;
    seg_start[2 * threadIdx.x + 1] = start1;
    seg_len[2 * threadIdx.x] = small[0] ? len[0] : 0u;
    seg_len[2 * threadIdx.x + 1] = small[1] ? len[1] : 0u;
  }
  __syncthreads();
  const uint32_t small_total = sh_nsmall, nbig = sh_nbig;
  if (c == 0 && threadIdx.x == 0) {
    prof[16] = small_total;
    prof[17] = nbig;
  }
  {
    const uint32_t m = max(seg_len[2 * threadIdx.x], seg_len[2 * threadIdx.x + 1]);
    if (m) atomicMax(&prof[18], (unsigned long long)m);
  }
  if (threadIdx.x == 0) atomicMax(&prof[19], gtimer());
  // long segments (rare): the j-th is radix-sorted in global memory by CTA j % G
  for (uint32_t j = c; j < nbig; j += G) {
    if ((big_mask & 1u) && big_x == j) sh_gp = 2 * threadIdx.x;
    if ((big_mask & 2u) && big_x + (big_mask & 1u) == j) sh_gp = 2 * threadIdx.x + 1;
    __syncthreads();
    const uint32_t gp = sh_gp;
    const int list = gp < NBL ? 0 : 1;
    const uint32_t b = list == 0 ? gp : (2 * NBL - 1 - gp);
    const uint32_t t = list == 0 ? tpf[b] : tev[b];
    const uint32_t start = seg_start[gp];
    uint32_t *ids = list == 0 ? d.pf_ids : d.ev_ids;
    uint32_t *ka = (list == 0 ? d.sort_ka : d.f_sk2) + start;
    uint32_t *ia = (list == 0 ? d.sort_va : d.f_sv2) + start;
    uint32_t *kb = (list == 0 ? d.sort_kb : d.f_sk3) + start;
    uint32_t *ib = (list == 0 ? d.sort_vb : d.f_sv3) + start;
    cta_sort_pairs(ka, ia, kb, ib, t, s.h);  // counters in s.h[0, 4096): not needed any more
    for (uint32_t e = threadIdx.x; e < t; e += FT) ids[start + e] = ia[e];
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(&prof[20], gtimer());
  // short segments (fit in shared memory, 4 words per element): segment i (dense order) is
  // sorted by CTA i % G.  Keys are first mapped to order-preserving small codes
  // (key - min) >> g, g = common trailing zeros of the differences (integer-tick distances in
  // one list bucket give a handful of codes), so the stable radix sort needs one 8-bit pass.
  {
    const uint32_t nds = sh_nds;
    const unsigned long long t_r0 = gtimer();
    __shared__ uint32_t sh_min, sh_or;
    for (uint32_t i = c; i < nds; i += G) {
      const uint32_t gp = dense_gp[i];
      const int list = gp < NBL ? 0 : 1;
      const uint32_t t = seg_len[gp], start = seg_start[gp];
      const uint32_t *sk = (list == 0 ? d.sort_ka : d.f_sk2) + start;
      const uint32_t *si = (list == 0 ? d.sort_va : d.f_sv2) + start;
      uint32_t *ka = s.keys, *ia = s.keys + t, *kb = s.keys + 2 * t, *ib = s.keys + 3 * t;  // 4t <= 3 * tile
      uint32_t mn = 0xFFFFFFFFu;
      for (uint32_t j = threadIdx.x; j < t; j += FT) {
        const uint32_t k = sk[j];
        ka[j] = k;
        ia[j] = si[j];
        mn = min(mn, k);
      }
      mn = __reduce_min_sync(0xFFFFFFFFu, mn);
      if (threadIdx.x == 0) {
        sh_min = 0xFFFFFFFFu;
        sh_or = 0;
      }
      __syncthreads();
      if (lane == 0) atomicMin(&sh_min, mn);
      __syncthreads();
      mn = sh_min;
      uint32_t o = 0;
      for (uint32_t j = threadIdx.x; j < t; j += FT) o |= ka[j] - mn;
      o = __reduce_or_sync(0xFFFFFFFFu, o);
      if (lane == 0 && o) atomicOr(&sh_or, o);
      __syncthreads();
      const uint32_t g = sh_or ? (uint32_t)(__ffs(sh_or) - 1) : 0u;
      for (uint32_t j = threadIdx.x; j < t; j += FT) ka[j] = (ka[j] - mn) >> g;  // order-preserving code
      __syncthreads();
      cta_sort_pairs(ka, ia, kb, ib, t, s.h);  // counters in s.h[0, 4096)
      uint32_t *out = (list == 0 ? d.pf_ids : d.ev_ids) + start;
      for (uint32_t j = threadIdx.x; j < t; j += FT) out[j] = ia[j];
      __syncthreads();
    }
    if (threadIdx.x == 0) atomicMax(&prof[21], gtimer() - t_r0);
  }
  if (threadIdx.x == 0) atomicMax(&prof[1], gtimer());
}

// host side
bool fused_supported(const Params &p, int grid, uint32_t *tile_out) {
  if (p.world != 1 || grid <= 0 || grid > FUSED_MAX_CTAS) return false;
  uint64_t tile = (p.n_local + grid - 1) / grid;  // grid = CTAs of the instance
  tile = (tile + 31) / 32 * 32;
  if (tile == 0) tile = 32;
  if (tile > FUSED_MAX_TILE) return false;
  *tile_out = (uint32_t)tile;
  return true;
}

// 1 CTA of FT threads per SM must be resident for the whole grid (grid barrier).
template <int MAXB>
static bool prepare_one(uint32_t tile) {
  if (cudaFuncSetAttribute(k_fused_plan<MAXB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)fused_smem_bytes(FUSED_MAX_TILE)) != cudaSuccess)
    return false;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused_plan<MAXB>, FT, fused_smem_bytes(tile)) !=
      cudaSuccess)
    return false;
  return per_sm >= 1;
}

bool fused_prepare(int grid, uint32_t tile) {
  return grid >= 1 && prepare_one<1>(tile) && prepare_one<FUSED_MAX_BATCH>(tile);
}

template <int MAXB>
static void launch_t(const FusedInst *insts, uint32_t n, uint32_t gsize, cudaStream_t s) {
  FusedArgs<MAXB> B;
  B.n_inst = n;
  B.gsize = gsize;
  uint32_t tile = 32;
  for (uint32_t i = 0; i < n; ++i) {
    B.inst[i] = insts[i];
    tile = insts[i].tile > tile ? insts[i].tile : tile;
  }
  k_fused_plan<MAXB><<<n * gsize, FT, fused_smem_bytes(tile), s>>>(B);
}

int launch_fused_batch(const FusedInst *insts, uint32_t n, uint32_t gsize, cudaStream_t s) {
  if (n == 1) launch_t<1>(insts, n, gsize, s);
  else launch_t<FUSED_MAX_BATCH>(insts, n, gsize, s);
  return 1;
}

}  // namespace ss
