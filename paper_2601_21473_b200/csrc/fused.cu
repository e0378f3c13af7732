// fused.cu — one persistent cooperative kernel per planning step (world == 1).
//
// One CTA per SM (1024 threads); CTA c owns the contiguous agent tile [c*T, (c+1)*T), so
// CTA order is id order.  Phases, separated by grid barriers (cooperative launch):
//   P1  score the tile (a1, a2): 128-bit record loads, distance, eligibility; keys stay in
//       shared memory; byte-weighted level-1 histogram of the distance bits [30:20] with
//       per-bucket min/max key -> published per CTA (dense) and summed globally (atomics)
//   --- barrier
//   P2  every CTA resolves the boundary distance D* redundantly from the global histogram
//       (a3; levels 2/3 of the radix select, each behind a barrier, only when the boundary
//       bucket holds several distances)
//   P3  exclusive prefix of the tie-group bytes over the preceding CTAs, read from the
//       published per-CTA histograms (no extra barrier)
//   P4  emit (a4, a5): kept bits, new residency, byte totals; per-CTA counts of the
//       prefetch / evict members per level-1 bucket, published (dense) + global totals
//   --- barrier
//   P5  bucket (counting) sort of the lists: position = bucket start + members of the same
//       bucket in preceding CTAs + in-CTA id-order rank -> lists sorted by (bucket, id)
//   --- barrier (only when a list has members in a bucket holding several distances)
//   P6  each such segment is stably re-sorted by the full distance key by one CTA
//
// Every decision uses the same definitions as the multi-kernel path (kernels.cu), DESIGN.md
// §3; the two paths give bit-identical plans (tests/test_gpu_parity.py runs both).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace ss {

constexpr int FT = 1024;  // threads per CTA
constexpr int FWARPS = FT / 32;

// Grid barrier for a grid of co-resident CTAs (one per SM, checked with the occupancy API
// at init).  bar counts arrivals monotonically within one launch; the k-th barrier waits for
// k * gridDim.x arrivals.  Launch L uses bar[L & 1]; launch L-1 reset it (same stream, so
// every CTA of launch L-2 had finished).
struct GridBar {
  unsigned int *bar;
  unsigned int k;
  __device__ __forceinline__ void sync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++k;
      __threadfence();
      atomicAdd(bar, 1u);
      const unsigned int target = k * gridDim.x;
      unsigned int v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        if (v >= target) break;
        __nanosleep(20);
      }
      __threadfence();
    }
    __syncthreads();
  }
};

struct FusedArgs {
  Params p;
  int64_t now;
  int parity;
  unsigned int *bar;  // [2] barrier counters
  uint32_t tile;   // agents per CTA, multiple of 32
  uint32_t tw;     // tile / 32
};

// dynamic shared memory carve-up
struct FSmem {
  uint32_t *keys;    // [tile] distance bits of the tile's agents
  uint32_t *memb;    // [tile] member list scratch (ids local to the tile) / sort scratch
  uint32_t *old_w, *elig_w, *pf_w, *ev_w;  // [tw]
  uint32_t *h_lo, *h_hi, *h_min, *h_nmax;  // [2048] histogram (16-bit halves of bytes)
  unsigned long long *scratch;             // [64]
};

__device__ __forceinline__ FSmem carve(uint8_t *base, uint32_t tile, uint32_t tw) {
  FSmem s;
  uint32_t *w = reinterpret_cast<uint32_t *>(base);
  s.keys = w;
  w += tile;
  s.memb = w;
  w += tile;
  s.old_w = w;
  w += tw;
  s.elig_w = w;
  w += tw;
  s.pf_w = w;
  w += tw;
  s.ev_w = w;
  w += tw;
  s.h_lo = w;
  w += 2048;
  s.h_hi = w;
  w += 2048;
  s.h_min = w;
  w += 2048;
  s.h_nmax = w;
  w += 2048;
  uintptr_t a = (reinterpret_cast<uintptr_t>(w) + 15) & ~uintptr_t(15);
  s.scratch = reinterpret_cast<unsigned long long *>(a);
  return s;
}

size_t fused_smem_bytes(uint32_t tile) {
  const uint32_t tw = tile / 32;
  return (size_t)4 * (2 * tile + 4 * tw + 4 * 2048) + 16 + 64 * 8;
}

__device__ __forceinline__ void clear_hist(const FSmem &s, int nb) {
  for (int b = threadIdx.x; b < nb; b += FT) {
    s.h_lo[b] = 0;
    s.h_hi[b] = 0;
    s.h_min[b] = 0xFFFFFFFFu;
    s.h_nmax[b] = 0xFFFFFFFFu;
  }
}

// one lane's contribution to the byte-weighted histogram (native 32-bit shared atomics)
__device__ __forceinline__ void hist_lane(const FSmem &s, uint32_t b, uint32_t bits, uint32_t bytes) {
  atomicAdd(&s.h_lo[b], bytes & 0xFFFFu);
  atomicAdd(&s.h_hi[b], bytes >> 16);
  atomicMin(&s.h_min[b], bits);
  atomicMin(&s.h_nmax[b], ~bits);
}

// publish this CTA's histogram (dense, for the tie prefix) and add it to the global one
__device__ __forceinline__ void publish_hist(const FSmem &s, int nb, unsigned long long *cta_row,
                                             unsigned long long *g_hist, uint32_t *g_mm) {
  for (int b = threadIdx.x; b < nb; b += FT) {
    const unsigned long long v = ((unsigned long long)s.h_hi[b] << 16) + s.h_lo[b];
    cta_row[b] = v;
    if (v != 0) {
      atomicAdd(&g_hist[b], v);
      if (g_mm) {
        atomicMin(&g_mm[b], s.h_min[b]);
        atomicMin(&g_mm[nb + b], s.h_nmax[b]);
      }
    }
  }
}

struct Sel {
  uint32_t prefix;
  unsigned long long below, rem;
  uint32_t dstar, all_fit, done, level_res, b_res;
};

// Find the boundary bucket of histogram level `level` (every CTA computes the same result).
__device__ void select_level(const FSmem &s, const unsigned long long *g_hist, const uint32_t *g_mm, int level,
                             unsigned long long budget, Sel &sel) {
  const int nb = level == 1 ? 2048 : 1024;
  const int shift = level == 1 ? 20 : (level == 2 ? 10 : 0);
  const int per = nb / FT;  // 2 or 1
  unsigned long long *sh = s.scratch;
  __shared__ unsigned long long sh_tot, sh_prev;
  __shared__ uint32_t sh_b;
  if (threadIdx.x == 0) sh_b = 0xFFFFFFFFu;
  unsigned long long loc = 0;
  unsigned long long hv[2];
  for (int k = 0; k < per; ++k) {
    hv[k] = g_hist[threadIdx.x * per + k];
    loc += hv[k];
  }
  const unsigned long long ex = block_excl_scan<unsigned long long, FT>(loc, &sh_tot);
  __syncthreads();
  unsigned long long run = sel.below + ex;
  for (int k = 0; k < per; ++k) {
    const unsigned long long prev = run;
    run += hv[k];
    if (run > budget && prev <= budget) {
      sh_b = threadIdx.x * per + k;
      sh_prev = prev;
    }
  }
  __syncthreads();
  const uint32_t b = sh_b;
  (void)sh;
  if (b == 0xFFFFFFFFu) {  // level 1 only: every eligible agent fits
    sel.all_fit = 1;
    sel.done = 1;
    sel.dstar = 0xFFFFFFFFu;
    sel.rem = budget - (sel.below + sh_tot);
    sel.level_res = level;
    sel.b_res = 0;
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

// Stable LSD radix sort of n (key, id) pairs by key (ascending) for one CTA.  Buffers may
// be shared or global memory (generic pointers).  Digits [0,11) [11,22) [22,32); constant
// digits are skipped.  Result in (ka, ia).
__device__ void cta_sort_pairs(uint32_t *ka, uint32_t *ia, uint32_t *kb, uint32_t *ib, uint32_t n, uint32_t *cnt) {
  __shared__ uint32_t sh_or, sh_and;
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
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = pass == 0 ? 0 : (pass == 1 ? 11 : 22);
    const uint32_t mask = pass == 2 ? 0x3FFu : 0x7FFu;
    if (((varying >> shift) & mask) == 0) continue;
    for (int b = threadIdx.x; b < 2048; b += FT) cnt[b] = 0;
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < n; e += FT) atomicAdd(&cnt[(ka[e] >> shift) & mask], 1u);
    __syncthreads();
    {  // exclusive scan of the 2048 counters, 2 per thread
      __shared__ uint32_t tot;
      const uint32_t c0 = cnt[2 * threadIdx.x], c1 = cnt[2 * threadIdx.x + 1];
      const uint32_t ex = block_excl_scan<uint32_t, FT>(c0 + c1, &tot);
      __syncthreads();
      cnt[2 * threadIdx.x] = ex;
      cnt[2 * threadIdx.x + 1] = ex + c0;
      __syncthreads();
    }
    for (uint32_t c0 = 0; c0 < n; c0 += FT) {
      const uint32_t e = c0 + threadIdx.x;
      const bool valid = e < n;
      const uint32_t k = valid ? ka[e] : 0u, id = valid ? ia[e] : 0u;
      const uint32_t dg = valid ? ((k >> shift) & mask) : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, dg);
      const uint32_t rank = __popc(peers & lanemask_lt());
      const bool leader = (peers & lanemask_lt()) == 0;
      const uint32_t nw = (min(n - c0, (uint32_t)FT) + 31) / 32;
      for (uint32_t w = 0; w < nw; ++w) {
        if ((uint32_t)warp == w && valid) {
          const uint32_t pos = cnt[dg] + rank;
          kb[pos] = k;
          ib[pos] = id;
        }
        __syncwarp();
        if ((uint32_t)warp == w && valid && leader) cnt[dg] += __popc(peers);
        __syncthreads();
      }
    }
    __syncthreads();
    uint32_t *t;
    t = ka; ka = kb; kb = t;
    t = ia; ia = ib; ib = t;
    // keep the caller's view: results must end in the original (ka, ia) buffers
    for (uint32_t e = threadIdx.x; e < n; e += FT) {
      kb[e] = ka[e];
      ib[e] = ia[e];
    }
    __syncthreads();
    t = ka; ka = kb; kb = t;
    t = ia; ia = ib; ib = t;
  }
  (void)lane;
}

__global__ void __launch_bounds__(FT, 1) k_fused_plan(FusedArgs A) {
  GridBar grid{A.bar + A.parity, 0u};
  if (blockIdx.x == 0 && threadIdx.x == 0) A.bar[A.parity ^ 1] = 0u;  // for launch L+1
  const Params &p = A.p;
  const Dev &d = p.d;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const FSmem s = carve(smem_raw, A.tile, A.tw);
  const uint32_t c = blockIdx.x, G = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = (uint64_t)c * A.tile;
  const uint32_t n_here = base >= p.n_local ? 0u : (uint32_t)((p.n_local - base) < A.tile ? (p.n_local - base) : A.tile);
  const uint32_t tw_here = (n_here + 31) / 32;
  const int par = A.parity;
  unsigned long long *acc = d.f_acc + 8 * par;  // [0] zero bytes [1] h2d [2] d2h [3] tie kept [4] n_elig [5] status
  const uint32_t *bm_old = d.bm[p.cur];
  uint32_t *bm_new = d.bm[p.cur ^ 1];

  // ---------------- P1: score + level-1 histogram
  clear_hist(s, 2048);
  for (uint32_t w = threadIdx.x; w < A.tw; w += FT) s.old_w[w] = w < tw_here ? bm_old[base / 32 + w] : 0u;
  __syncthreads();
  uint32_t st = 0;
  unsigned long long zero_b = 0;
  for (uint32_t k = threadIdx.x; k < A.tw * 32; k += FT) {
    const bool valid = k < n_here;
    const uint64_t i = base + k;
    uint4 r = make_uint4(0, 0, 0, 0);
    if (valid) r = ld_stream(p.rec + i);
    const bool res = (s.old_w[k >> 5] >> (k & 31)) & 1u;
    const float dist = valid ? distance_of(r, A.now, p.hop_scale, d.dint, p.n_kin, st) : 0.0f;
    const uint32_t bits = __float_as_uint(dist);
    const bool elig = valid && (res || dist == 0.0f || dist < theta_of(p, class_of(r)));
    s.keys[k] = bits;
    if (valid) d.keys[i] = bits;
    const uint32_t eb = __ballot_sync(0xFFFFFFFFu, elig);
    if (lane == 0) s.elig_w[k >> 5] = eb;
    if (elig) hist_lane(s, bits >> 20, bits, r.y);
    if (valid && dist == 0.0f) zero_b += r.y;
  }
  __syncthreads();
  publish_hist(s, 2048, d.f_cta_h1 + (uint64_t)c * 2048, d.f_hist1 + 2048 * par, d.f_mm1 + 4096 * par);
  zero_b = block_sum<unsigned long long, FT>(zero_b);
  st = __reduce_or_sync(0xFFFFFFFFu, st);
  if (lane == 0 && st) atomicOr(reinterpret_cast<unsigned int *>(&acc[5]), st);
  if (threadIdx.x == 0 && zero_b) atomicAdd(&acc[0], zero_b);
  grid.sync();

  // ---------------- P2: select
  if (c == 0) {  // clear the other parity's accumulators for the next step
    const int q = par ^ 1;
    for (int b = threadIdx.x; b < 2048; b += FT) {
      d.f_hist1[2048 * q + b] = 0;
      d.f_mm1[4096 * q + b] = 0xFFFFFFFFu;
      d.f_mm1[4096 * q + 2048 + b] = 0xFFFFFFFFu;
      d.f_tot[4096 * q + b] = 0;
      d.f_tot[4096 * q + 2048 + b] = 0;
    }
    for (int b = threadIdx.x; b < 1024; b += FT) {
      d.f_hist2[1024 * q + b] = 0;
      d.f_hist3[1024 * q + b] = 0;
      d.f_mm2[2048 * q + b] = 0xFFFFFFFFu;
      d.f_mm2[2048 * q + 1024 + b] = 0xFFFFFFFFu;
    }
    if (threadIdx.x < 8) d.f_acc[8 * q + threadIdx.x] = 0;
  }
  Sel sel = {0, 0, 0, 0xFFFFFFFFu, 0, 0, 0, 0};
  select_level(s, d.f_hist1 + 2048 * par, d.f_mm1 + 4096 * par, 1, p.budget, sel);
  for (int level = 2; level <= 3 && !sel.done; ++level) {
    const int hi_shift = level == 2 ? 20 : 10, shift = level == 2 ? 10 : 0;
    const uint32_t want = sel.prefix >> hi_shift;
    clear_hist(s, 1024);
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < n_here; k += FT) {
      const uint32_t bits = s.keys[k];
      if (((s.elig_w[k >> 5] >> (k & 31)) & 1u) && (bits >> hi_shift) == want)
        hist_lane(s, (bits >> shift) & 1023u, bits, p.rec[base + k].y);
    }
    __syncthreads();
    unsigned long long *gh = level == 2 ? d.f_hist2 + 1024 * par : d.f_hist3 + 1024 * par;
    uint32_t *gm = level == 2 ? d.f_mm2 + 2048 * par : nullptr;
    publish_hist(s, 1024, (level == 2 ? d.f_cta_h2 : d.f_cta_h3) + (uint64_t)c * 1024, gh, gm);
    grid.sync();
    select_level(s, gh, gm, level, p.budget, sel);
  }

  // ---------------- P3: tie-group prefix over the preceding CTAs
  __shared__ unsigned long long sh_tie_excl;
  if (warp == 0) {
    unsigned long long t = 0;
    if (!sel.all_fit) {
      const unsigned long long *col = sel.level_res == 1 ? d.f_cta_h1 : (sel.level_res == 2 ? d.f_cta_h2 : d.f_cta_h3);
      const uint32_t stride = sel.level_res == 1 ? 2048 : 1024;
      for (uint32_t q = lane; q < c; q += 32) t += col[(uint64_t)q * stride + sel.b_res];
    }
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    if (lane == 0) sh_tie_excl = t;
  }
  __syncthreads();

  // ---------------- P4: emit
  // tie bytes per word (id order), then word-level exclusive scan
  const bool all_fit = sel.all_fit;
  const uint32_t dstar = sel.dstar;
  uint32_t *word_tie = s.memb;  // [tw] scratch (u32 is enough? bytes per word can exceed 2^32: use 2 words)
  unsigned long long *word_tie64 = reinterpret_cast<unsigned long long *>(s.memb);
  for (uint32_t w = warp; w < A.tw; w += FWARPS) {
    const uint32_t k = w * 32 + lane;
    const bool tie = !all_fit && ((s.elig_w[w] >> lane) & 1u) && s.keys[k] == dstar && k < n_here;
    const uint32_t fp = tie ? p.rec[base + k].y : 0u;
    unsigned long long v = fp;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (lane == 0) word_tie64[w] = v;
  }
  (void)word_tie;
  __syncthreads();
  {  // exclusive scan over the tile's words (tw <= 1024*? ; loop in chunks of FT)
    __shared__ unsigned long long tot;
    unsigned long long carry = 0;
    for (uint32_t w0 = 0; w0 < A.tw; w0 += FT) {
      const uint32_t w = w0 + threadIdx.x;
      const unsigned long long v = w < A.tw ? word_tie64[w] : 0ull;
      const unsigned long long ex = block_excl_scan<unsigned long long, FT>(v, &tot);
      __syncthreads();
      if (w < A.tw) word_tie64[w] = carry + ex;
      carry += tot;
      __syncthreads();
    }
  }
  unsigned long long h2d = 0, d2h = 0, tie_kept = 0;
  uint32_t n_el = 0;
  for (uint32_t w = warp; w < A.tw; w += FWARPS) {
    const uint32_t k = w * 32 + lane;
    const bool valid = k < n_here;
    const bool el = (s.elig_w[w] >> lane) & 1u;
    const uint32_t key = s.keys[k];
    const bool tie = valid && el && !all_fit && key == dstar;
    const uint32_t fp = tie ? p.rec[base + k].y : 0u;
    unsigned long long incl = fp;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += t;
    }
    incl += sh_tie_excl + word_tie64[w];
    const bool kept = valid && el && (all_fit || key < dstar || (tie && incl <= sel.rem));
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
    if ((pfw >> lane) & 1u) h2d += p.rec[base + k].y;
    if ((evw >> lane) & 1u) {
      const uint4 r = p.rec[base + k];
      if ((r.z >> 4) & 1u) {  // R13: KV + HIST blocks of a dirty evicted agent
        for (uint64_t b = p.blk_ptr[base + k]; b < p.blk_ptr[base + k + 1]; ++b)
          if (p.blk_kind[b] != 0) d2h += p.blk_size[b];
      }
    }
  }
  __syncthreads();
  // list members per level-1 bucket (reuse the histogram arrays as counters)
  for (int b = threadIdx.x; b < 2048; b += FT) {
    s.h_lo[b] = 0;  // prefetch count
    s.h_hi[b] = 0;  // evict count
  }
  __syncthreads();
  for (uint32_t w = warp; w < A.tw; w += FWARPS) {
    const uint32_t k = w * 32 + lane;
    if ((s.pf_w[w] >> lane) & 1u) atomicAdd(&s.h_lo[s.keys[k] >> 20], 1u);
    if ((s.ev_w[w] >> lane) & 1u) atomicAdd(&s.h_hi[s.keys[k] >> 20], 1u);
  }
  __syncthreads();
  uint32_t *cpf = d.f_cta_cpf + (uint64_t)c * 2048, *cev = d.f_cta_cev + (uint64_t)c * 2048;
  uint32_t *tot_pf = d.f_tot + 4096 * par, *tot_ev = d.f_tot + 4096 * par + 2048;
  for (int b = threadIdx.x; b < 2048; b += FT) {
    const uint32_t a = s.h_lo[b], e = s.h_hi[b];
    cpf[b] = a;
    cev[b] = e;
    if (a) atomicAdd(&tot_pf[b], a);
    if (e) atomicAdd(&tot_ev[b], e);
  }
  h2d = block_sum<unsigned long long, FT>(h2d);
  d2h = block_sum<unsigned long long, FT>(d2h);
  tie_kept = block_sum<unsigned long long, FT>(tie_kept);
  n_el = block_sum<uint32_t, FT>(n_el);
  if (threadIdx.x == 0) {
    if (h2d) atomicAdd(&acc[1], h2d);
    if (d2h) atomicAdd(&acc[2], d2h);
    if (tie_kept) atomicAdd(&acc[3], tie_kept);
    if (n_el) atomicAdd(&acc[4], (unsigned long long)n_el);
  }
  grid.sync();

  // ---------------- P5: bucket sort of the lists
  // bucket starts (prefetch ascending buckets, evict descending buckets)
  uint32_t *g_pf = s.h_min, *g_ev = s.h_nmax;  // [2048] starts
  __shared__ uint32_t sh_npf, sh_nev;
  {
    const uint32_t a0 = tot_pf[2 * threadIdx.x], a1 = tot_pf[2 * threadIdx.x + 1];
    const uint32_t ex = block_excl_scan<uint32_t, FT>(a0 + a1, &sh_npf);
    g_pf[2 * threadIdx.x] = ex;
    g_pf[2 * threadIdx.x + 1] = ex + a0;
    // evict: scan over reversed bucket order r = 2047 - b
    const uint32_t r0 = 2 * threadIdx.x, r1 = r0 + 1;
    const uint32_t e0 = tot_ev[2047 - r0], e1 = tot_ev[2047 - r1];
    const uint32_t exe = block_excl_scan<uint32_t, FT>(e0 + e1, &sh_nev);
    g_ev[2047 - r0] = exe;
    g_ev[2047 - r1] = exe + e0;
  }
  __syncthreads();
  // preceding-CTA counts of the buckets this CTA has members in
  for (int b = warp; b < 2048; b += FWARPS) {
    const uint32_t mine_pf = s.h_lo[b], mine_ev = s.h_hi[b];
    if (mine_pf == 0 && mine_ev == 0) continue;  // warp-uniform
    uint32_t ppf = 0, pev = 0;
    for (uint32_t q = lane; q < G; q += 32) {
      if (mine_pf && q < c) ppf += d.f_cta_cpf[(uint64_t)q * 2048 + b];
      if (mine_ev && q > c) pev += d.f_cta_cev[(uint64_t)q * 2048 + b];
    }
    ppf = __reduce_add_sync(0xFFFFFFFFu, ppf);
    pev = __reduce_add_sync(0xFFFFFFFFu, pev);
    if (lane == 0) {
      g_pf[b] += ppf;  // now: first output slot of this CTA's members of bucket b
      g_ev[b] += pev;
    }
  }
  __syncthreads();
  // in-CTA ranks: warp 0 walks the prefetch members in ascending id order, warp 1 the
  // evict members in descending id order
  if (warp == 0) {
    for (uint32_t w = 0; w < A.tw; ++w) {
      const uint32_t m = s.pf_w[w];
      if (m == 0) continue;
      const bool on = (m >> lane) & 1u;
      const uint32_t b = on ? (s.keys[w * 32 + lane] >> 20) : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
      if (on) {
        const uint32_t pos = g_pf[b] + __popc(peers & lanemask_lt());
        d.pf_ids[pos] = (uint32_t)(p.shard_begin + base + w * 32 + lane);
      }
      __syncwarp();
      if (on && (peers & lanemask_lt()) == 0) g_pf[b] += __popc(peers);
      __syncwarp();
    }
  } else if (warp == 1) {
    for (uint32_t w = A.tw; w-- > 0;) {
      const uint32_t m = s.ev_w[w];
      if (m == 0) continue;
      // descending id: lane j handles bit 31 - j
      const uint32_t bit = 31 - lane;
      const bool on = (m >> bit) & 1u;
      const uint32_t b = on ? (s.keys[w * 32 + bit] >> 20) : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
      if (on) {
        const uint32_t pos = g_ev[b] + __popc(peers & lanemask_lt());
        d.ev_ids[pos] = (uint32_t)(p.shard_begin + base + w * 32 + bit);
      }
      __syncwarp();
      if (on && (peers & lanemask_lt()) == 0) g_ev[b] += __popc(peers);
      __syncwarp();
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

  // ---------------- P6: re-sort list segments whose bucket holds several distances
  // (decided identically by every CTA from global data)
  const uint32_t *mm1 = d.f_mm1 + 4096 * par;
  __shared__ uint32_t sh_need;
  if (threadIdx.x == 0) sh_need = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < 2048; b += FT) {
    const bool multi = mm1[b] != ~mm1[2048 + b];
    if (multi && (tot_pf[b] > 1 || tot_ev[b] > 1)) atomicOr(&sh_need, 1u);
  }
  __syncthreads();
  if (!sh_need) return;
  grid.sync();
  // segment k (bucket order, prefetch list first) is re-sorted by CTA k mod G, in rounds
  // of up to 64 segments per CTA
  __shared__ uint32_t q_n, q_start[64], q_len[64], q_list[64];
  __shared__ uint32_t seg_base, tot_tmp, seg_tmp;
  for (uint32_t round = 0;; ++round) {
    if (threadIdx.x == 0) {
      q_n = 0;
      seg_base = 0;
    }
    __syncthreads();
    for (int list = 0; list < 2; ++list) {
      const uint32_t *tot = list == 0 ? tot_pf : tot_ev;
      uint32_t len[2], need[2];
      for (int k = 0; k < 2; ++k) {
        const uint32_t r = 2 * threadIdx.x + k;  // position in list order
        const uint32_t b = list == 0 ? r : 2047 - r;
        len[k] = tot[b];
        need[k] = (len[k] > 1 && mm1[b] != ~mm1[2048 + b]) ? 1u : 0u;
      }
      const uint32_t st_ex = block_excl_scan<uint32_t, FT>(len[0] + len[1], &tot_tmp);
      const uint32_t sg_ex = block_excl_scan<uint32_t, FT>(need[0] + need[1], &seg_tmp);
      uint32_t start = st_ex, sg = seg_base + sg_ex;
      for (int k = 0; k < 2; ++k) {
        if (need[k]) {
          const uint32_t j = sg / G;  // this segment's index among CTA (sg % G)'s segments
          if (sg % G == c && j >= round * 64 && j < (round + 1) * 64) {
            const uint32_t slot = j - round * 64;
            q_start[slot] = start;
            q_len[slot] = len[k];
            q_list[slot] = list;
            atomicAdd(&q_n, 1u);
          }
          ++sg;
        }
        start += len[k];
      }
      __syncthreads();
      if (threadIdx.x == 0) seg_base += seg_tmp;
      __syncthreads();
    }
    const uint32_t nq = q_n;  // the CTA's segments of this round occupy slots [0, nq)
    for (uint32_t qi = 0; qi < nq; ++qi) {
      const uint32_t list = q_list[qi], start = q_start[qi], t = q_len[qi];
      uint32_t *ids = list == 0 ? d.pf_ids : d.ev_ids;
      const bool fits = t <= A.tile;
      uint32_t *ka = fits ? s.keys : (list == 0 ? d.sort_ka : d.f_sk2) + start;
      uint32_t *ia = fits ? s.memb : (list == 0 ? d.sort_va : d.f_sv2) + start;
      uint32_t *kb = (list == 0 ? d.sort_kb : d.f_sk3) + start;
      uint32_t *ib = (list == 0 ? d.sort_vb : d.f_sv3) + start;
      for (uint32_t e = threadIdx.x; e < t; e += FT) {
        const uint32_t id = ids[start + e];
        const uint32_t key = d.keys[id - p.shard_begin];
        ka[e] = list == 0 ? key : ~key;
        ia[e] = id;
      }
      __syncthreads();
      cta_sort_pairs(ka, ia, kb, ib, t, s.h_lo);
      for (uint32_t e = threadIdx.x; e < t; e += FT) ids[start + e] = ia[e];
      __syncthreads();
    }
    const uint32_t total_segs = seg_base;
    __syncthreads();
    if ((round + 1) * 64 * G >= total_segs) break;  // uniform: every CTA sees the same totals
  }
}

// host side
bool fused_supported(const Params &p, int grid, uint32_t *tile_out) {
  if (p.world != 1 || grid <= 0 || grid > FUSED_MAX_CTAS) return false;
  uint64_t tile = (p.n_local + grid - 1) / grid;
  tile = (tile + 31) / 32 * 32;
  if (tile == 0) tile = 32;
  if (tile > FUSED_MAX_TILE) return false;
  *tile_out = (uint32_t)tile;
  return true;
}

// 1 CTA of FT threads per SM must be resident for the whole grid (grid barrier).
bool fused_prepare(int grid, uint32_t tile) {
  if (cudaFuncSetAttribute(k_fused_plan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)fused_smem_bytes(FUSED_MAX_TILE)) != cudaSuccess)
    return false;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused_plan, FT, fused_smem_bytes(tile)) != cudaSuccess)
    return false;
  return per_sm >= 1 && grid >= 1;
}

int launch_fused_plan(const Params &p, int64_t now, int parity, int grid, uint32_t tile, unsigned int *bar,
                      cudaStream_t s) {
  FusedArgs A;
  A.p = p;
  A.now = now;
  A.parity = parity;
  A.bar = bar;
  A.tile = tile;
  A.tw = tile / 32;
  k_fused_plan<<<grid, FT, fused_smem_bytes(tile), s>>>(A);
  return 1;
}

}  // namespace ss
