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

#include <type_traits>

#include "fused_common.cuh"

namespace ss {

size_t fused_smem_bytes(uint32_t tile) {
  const uint32_t tw = tile / 32;
  return (size_t)4 * (3 * tile + 5 * tw + 4 * NB1) + 16;
}

// A/B only (-DAB_P1_TMA): P1 staging by bulk copies (fast variant): the tile's records land in
// shared memory in chunks of P1_CH records, each with its own mbarrier, all issued at once by
// one thread.  The chunks live in memory P1 does not use: the scratch array s.memb, then from
// s.h + 3 NB1 on (the need list, the owner staging s.col and any dynamic shared memory beyond
// them).  Parity-green, but measured slower at C4 (profiles/r02_v65_ab_p1_tma.log,
// r02_v66_probe.log: P1 loop 8.1 vs 6.8 us, step 26.9 vs 24.5 us): the register-load P1 is
// issue-bound, not load-bound, so taking the loads off the warps gains nothing while the
// copies arrive later than the warps' own batches.
constexpr uint32_t P1_CH = 256, P1_MAXCH = 32;
static size_t p1_region2_off(uint32_t tile) {  // byte offset of s.h + 3 NB1 (carve)
  return ((size_t)4 * (3 * tile + 5 * (tile / 32)) + 15) / 16 * 16 + (size_t)4 * 3 * NB1;
}
// dynamic shared memory the staging needs for a full tile (0: staging impossible)
static size_t p1_staging_bytes(uint32_t tile) {
  const uint32_t ch_m = tile * 4 / (P1_CH * 16), nch = (tile + P1_CH - 1) / P1_CH;
  if (nch > P1_MAXCH) return 0;
  return p1_region2_off(tile) + (size_t)(nch > ch_m ? nch - ch_m : 0) * P1_CH * 16;
}

template <int MAXB>
__global__ void __launch_bounds__(FT, 1) k_fused_plan(const __grid_constant__ FusedArgs<MAXB> B) {
  // (single context: instance 0 at constant offsets, so its fields stay in uniform registers)
  const uint32_t gi = MAXB == 1 ? 0u : blockIdx.x / B.gsize;
  const uint32_t c = MAXB == 1 ? blockIdx.x : blockIdx.x % B.gsize, G = B.gsize;
  const FusedInst &I = B.inst[gi];
  if (threadIdx.x == 0) {  // this tile's records into L2 while the parameters are fetched
    const uint64_t b0 = (uint64_t)c * I.tile;
    if (b0 < I.n_local) {
      const uint64_t nb = 16 * (I.n_local - b0 < I.tile ? I.n_local - b0 : I.tile);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(I.rec + b0), "r"((uint32_t)nb) : "memory");
      const uint64_t wb0 = b0 / 32, nw = (nb / 16 + 31) / 32;  // residency words of the tile
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(I.bm_old + wb0 - (wb0 & 3)),
                   "r"((uint32_t)(((nw + (wb0 & 3)) * 4 + 15) / 16 * 16)) : "memory");
    }
  }
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
  // Programmatic dependent launch: everything above (parameter copy, L2 prefetch of the
  // inputs) overlaps the tail of the previous kernel on the stream; from here on this launch
  // sees all of its writes.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // ... and the next launch may be scheduled right away: its CTAs take SMs as this grid's CTAs
  // exit and wait (above) for this grid's completion before touching any state
  asm volatile("griddepcontrol.launch_dependents;");
  const Params &p = sp;
  const InstArgs A = {I.now, (int)I.parity, I.epoch, I.tile, I.tile / 32, B.fastok};
  const Dev &d = p.d;
  // the world this instance is a rank of (its peers' arrays), or itself
  __shared__ WorldPtrs sw;
  const uint32_t nw = MAXB == 1 ? 1u : B.wsize, rank = MAXB == 1 ? 0u : gi % nw;
  if (threadIdx.x < nw) {
    const Dev &q = nw == 1 ? d : B.inst[gi - rank + threadIdx.x].params->d;
    sw.h1[threadIdx.x] = q.f_hist1;
    sw.h2[threadIdx.x] = q.f_hist2;
    sw.h3[threadIdx.x] = q.f_hist3;
    sw.m1[threadIdx.x] = q.f_mm1;
    sw.m2[threadIdx.x] = q.f_mm2;
    sw.acc[threadIdx.x] = q.f_acc;
    sw.hdr[threadIdx.x] = q.header;
    if (threadIdx.x == 0) {
      sw.nw = nw;
      sw.rank = rank;
    }
  }
  __shared__ unsigned int *sw_bar;  // rank 0's world-barrier counters
  if (threadIdx.x == 32) sw_bar = (nw == 1 ? d.f_bar : B.inst[gi - rank].params->d.f_bar) + 2;
  __syncthreads();
  const WorldPtrs &W = sw;
  GridBar wgrid{sw_bar + A.parity, 0u, nw * G};              // every CTA of the world
  if (c == 0 && threadIdx.x == 0) {
    d.f_bar[A.parity ^ 1] = 0u;  // for launch L+1
    if (rank == 0) sw_bar[A.parity ^ 1] = 0u;
    // header fields summed by every CTA after B1 (fast list placement) or written after B4
    unsigned long long *H = d.header;
    H[H_N_PF] = 0ull;
    H[H_N_EV] = 0ull;
    H[H_H2D] = 0ull;
    H[H_D2H] = 0ull;
    H[H_KEPT] = 0ull;
    H[H_N_ELIG] = 0ull;
    H[H_STATUS] = 0ull;
  }
  unsigned long long *prof = d.f_prof;
  PROBE(if (threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    atomicMin(&prof[0], t);
    atomicMax(&prof[15], t);  // last CTA past the dependency wait
    if (c == 0) prof[2] = t;
  })
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const FSmem s = carve(smem_raw, A.tile, A.tw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = (uint64_t)c * A.tile;
  const uint32_t n_here =
      base >= p.n_local ? 0u : (uint32_t)((p.n_local - base) < A.tile ? (p.n_local - base) : A.tile);
  const uint32_t tw_here = (n_here + 31) / 32;
  const int par = A.parity;
  // P1 record staging (see P1_CH): CTA-uniform decision; the copies go out right away
  const bool fast = p.int_mode != 0 && p.explicit_dist == 0 && A.now >= 0 && A.now <= 0xFFFFFFFFll && !p.keep_dist;
  __shared__ __align__(8) unsigned long long s_p1bar[P1_MAXCH];
  const uint32_t p1_chm = A.tile * 4 / (P1_CH * 16), p1_nch = (n_here + P1_CH - 1) / P1_CH;
  uint4 *const p1_r1 = reinterpret_cast<uint4 *>(s.memb), *const p1_r2 = reinterpret_cast<uint4 *>(s.h + 3 * NB1);
  bool p1_tma;
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const uint32_t off2 = (uint32_t)(reinterpret_cast<uint8_t *>(p1_r2) - smem_raw);
    const uint32_t ch2 = dyn > off2 ? (dyn - off2) / (P1_CH * 16) : 0u;
#ifdef AB_P1_TMA
    p1_tma = fast && n_here > 0 && p1_nch <= P1_MAXCH && p1_nch <= p1_chm + ch2;
#else
    p1_tma = false;
#endif
  }
  if (p1_tma && threadIdx.x == 0) {
    for (uint32_t j = 0; j < p1_nch; ++j)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_p1bar[j])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (uint32_t j = 0; j < p1_nch; ++j) {
      const uint32_t nb = 16 * min(P1_CH, n_here - j * P1_CH);
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&s_p1bar[j]);
      uint4 *dst = j < p1_chm ? p1_r1 + j * P1_CH : p1_r2 + (j - p1_chm) * P1_CH;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nb) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(dst)),
                   "l"(p.rec + base + j * P1_CH), "r"(nb), "r"(b)
                   : "memory");
    }
  }
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
  const bool imode = p.int_mode != 0, xdist = p.explicit_dist != 0;
  // remaining ticks in 32-bit arithmetic when now fits (t_next is 32-bit): exact for < 2^24,
  // rounded to nearest as __ll2float_rn above
  const bool now32 = now >= 0 && now <= 0xFFFFFFFFll;
  const uint32_t nowl = (uint32_t)now;
  // The tile is streamed in batches of LOAD_BATCH records per thread, double-buffered (two
  // batches in flight).  Measured on B200 (profiles/r01_v8_ab_*.log, r01_v9_ab_dbuf.log): a
  // per-slot rolling refill and deeper single batches are slower.  Lanes past the tile's end
  // load its last record (no zero-fill) and are masked by `valid`.
  const uint32_t last = n_here ? n_here - 1 : 0u;
  uint4 r[LOAD_BATCH];
  auto load_into = [&](uint4 (&rr)[LOAD_BATCH], uint32_t k0) {
#pragma unroll
    for (int j = 0; j < LOAD_BATCH; ++j)  // all loads of a batch in flight before any use
      rr[j] = n_here ? ld_stream(rec + min(k0 + j * FT + threadIdx.x, last)) : make_uint4(0, 0, 0, 0);
  };
  const uint32_t *bm_tile = bm_old + base / 32;
  for (uint32_t w = threadIdx.x; w < A.tw; w += FT) s.old_w[w] = w < tw_here ? bm_tile[w] : 0u;
  if (p1_tma) {  // (integer mode: no min / max rows; [3 NB1, 4 NB1) holds staged records)
    for (int b = threadIdx.x; b < NB1; b += FT) {
      s.h[b] = 0;
      s.h[NB1 + b] = 0;
    }
  } else {
    clear_hist(s.h, NB1);
  }
  if (imode)  // [2 * NB1, 3 * NB1): eligible counts per bucket (non-resident | resident << 16)
    for (int b = threadIdx.x; b < NB1; b += FT) s.h[2 * NB1 + b] = 0u;  // (4 per thread)
  // this CTA's eligible agents in multi-valued integer buckets (placed by one CTA, fast path)
  constexpr uint32_t LOVF = 32;
  __shared__ uint4 s_ovf[LOVF];
  __shared__ uint32_t s_novf;
  if (threadIdx.x == 0) s_novf = 0;
  // chunk counters: [0,4) zero-distance bytes, [4,11) P4 sums, [20,24) P3 tie prefix
  __shared__ uint32_t sacc[24];
  if (threadIdx.x < 24) sacc[threadIdx.x] = 0;
  __syncthreads();
  uint32_t st = 0;
  unsigned long long zero_b = 0;  // (integer mode: bucket 0 of the histogram instead)
  // One record: distance (a1), eligibility (a2), shared-memory state, level-1 histogram.
  // Compiled four ways: CHECK (a batch that runs past the tile's end: `valid` masks) and FAST
  // (integer mode, no explicit distances, 32-bit now, no distance copy: the class-0 path with
  // nothing else live; warps holding other classes still take the general definition).
  auto record = [&](const uint4 rj, const uint32_t wd, auto check_tag, auto fast_tag) {
    constexpr bool CHECK = decltype(check_tag)::value, FAST = decltype(fast_tag)::value;
    const uint32_t k = wd * 32 + lane;
    const bool valid = CHECK ? k < n_here : true;
    const bool res = (s.old_w[wd] >> lane) & 1u;
    const uint32_t ph = rj.z & 3u, cl = (rj.z >> 2) & 3u;
    float dist, th;
    if (!FAST && xdist) {  // explicit distances (R19)
      dist = valid ? explicit_distance_of(rj, st) : 0.0f;
      th = th0;
    } else if (__ballot_sync(0xFFFFFFFFu, valid && cl != 0u)) {
      // the warp holds interaction / diffusion / malformed records: general definition
      dist = valid ? distance_of(rj, now, hop_scale, dint, n_kin, st) : 0.0f;
      th = (cl & 2u) ? ((cl & 1u) ? 0.0f : th2) : ((cl & 1u) ? th1 : th0);
    } else {
      // independent agents only: remaining action ticks, 0 while in an LLM
      // phase, +inf when idle — the same values distance_of gives for class 0
      float d_action;
      if (FAST || now32) {
        d_action = rj.x > nowl ? __uint2float_rn(rj.x - nowl) : 0.0f;
      } else {
        const int64_t remain = (int64_t)rj.x - now;
        d_action = remain <= 0 ? 0.0f : __ll2float_rn(remain);
      }
      dist = (ph == 1u || ph == 2u) ? 0.0f : (ph == 3u ? __int_as_float(0x7F800000) : d_action);
      th = th0;
    }
    const uint32_t bits = valid ? __float_as_uint(dist) : 0u;
    const bool elig = valid && (res || dist == 0.0f || dist < th);
    s.keys[k] = bits;
    s.fp[k] = valid ? rj.y : 0u;
    if (!FAST && gkeys && valid) gkeys[k] = bits;
    const uint32_t eb = __ballot_sync(0xFFFFFFFFu, elig);
    const uint32_t db = __ballot_sync(0xFFFFFFFFu, valid && ((rj.z >> 4) & 1u));
    if (lane == 0) {
      s.elig_w[wd] = eb;
      s.dirty_w[wd] = db;
    }
    if (elig) {
      const uint32_t q = (FAST || imode) ? ibucket(bits) : slot1(bits >> 19);
      atomicAdd(&s.h[q], rj.y & 0xFFFFu);
      atomicAdd(&s.h[NB1 + q], rj.y >> 16);
      if (FAST || imode) {  // eligible counts by residency (fast list placement)
        atomicAdd(&s.h[2 * NB1 + q], res ? 0x10000u : 1u);
        if (ib_multi(q)) {  // rare: a multi-valued bucket
          const uint32_t j = atomicAdd(&s_novf, 1u);
          if (j < LOVF) s_ovf[j] = make_uint4(bits, (uint32_t)(p.shard_begin + base + k), res ? 1u : 0u, 0u);
        }
      } else {  // min / max key only where a bucket can hold several distances
        atomicMin(&s.h[2 * NB1 + q], bits);
        atomicMin(&s.h[3 * NB1 + q], ~bits);
      }
    }
    if (!FAST && !imode && valid && dist == 0.0f) zero_b += rj.y;
  };
  using T_ = std::true_type;
  using F_ = std::false_type;
  // one record body per variant (always masked; a rolled loop): the kernel's executed code has
  // to stay small (instruction-fetch stalls, see PROBE)
  auto batch = [&](uint4 (&rr)[LOAD_BATCH], uint32_t k0) {
#pragma unroll
    for (int j = 0; j < LOAD_BATCH; ++j) {
      const uint32_t wd = (k0 + j * FT) / 32 + warp;  // this warp's residency word (k & 31 == lane)
      if (wd >= A.tw) continue;                        // warp-uniform
      if (fast) record(rr[j], wd, T_(), T_());
      else record(rr[j], wd, T_(), F_());
    }
  };
  // two batches in flight: the next one's loads go out before the current one is processed
  // (measured: P1 loop 6.0 vs 6.3 us with single batches, profiles/r01_v9_ab_dbuf.log)
  uint4 r2[LOAD_BATCH];
  const uint32_t BS = LOAD_BATCH * FT, nk = A.tw * 32;
  if (p1_tma) {  // records from the staged chunks, each consumed as soon as its copy lands
#pragma unroll 1
    for (uint32_t k0 = 0; k0 < nk; k0 += FT) {
      const uint32_t wd = k0 / 32 + warp;
      if (wd >= A.tw) break;  // (warp-uniform; later rounds are further out)
      const uint32_t k = k0 + threadIdx.x, j = k / P1_CH;
      uint4 rj = make_uint4(0, 0, 0, 0);
      if (k < n_here) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&s_p1bar[j]);
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0; selp.u32 %0, 1, 0, q; }"
                       : "=r"(ok)
                       : "r"(b)
                       : "memory");
        rj = (j < p1_chm ? p1_r1 + j * P1_CH : p1_r2 + (j - p1_chm) * P1_CH)[k % P1_CH];
      }
      record(rj, wd, T_(), T_());
    }
  } else {
  load_into(r, 0);
#ifdef AB_P1_UNROLL2  // A/B: the two batches of a loop iteration as separate code copies
  for (uint32_t k0 = 0; k0 < nk; k0 += 2 * BS) {
    if (k0 + BS < nk) load_into(r2, k0 + BS);
    batch(r, k0);
    if (k0 + BS >= nk) break;
    if (k0 + 2 * BS < nk) load_into(r, k0 + 2 * BS);
    batch(r2, k0 + BS);
  }
#else
#pragma unroll 1
  for (uint32_t k0 = 0; k0 < nk; k0 += BS) {
    if (k0 + BS < nk) load_into(r2, k0 + BS);
    batch(r, k0);
#pragma unroll
    for (int j = 0; j < LOAD_BATCH; ++j) r[j] = r2[j];
  }
#endif
  }
  if (!imode) warp_add_u64(zero_b, sacc);
  __syncthreads();
  STAMP_MAX(25)  // P1 loop done
  // this CTA's level-1 bytes: dense row (its column entry gives the tie prefix in P3) and
  // the global sum
  publish_hist(s.h, NB1, d.f_hist1 + NB1 * par, imode ? nullptr : d.f_mm1 + 2 * NB1 * par,
               d.f_rows1 + (uint64_t)c * NB1, d.f_hist1 + 2 * NB1 + 64 * par, !imode);
  // bucket owners (fast list placement): CTA o owns buckets [o RB, (o + 1) RB)
  const uint32_t RB = ((NB1 + G - 1) / G + 3u) & ~3u;
  const uint32_t o_lo = min((uint32_t)NB1, c * RB), o_n = min((uint32_t)NB1, o_lo + RB) - o_lo;
  const uint32_t QP = (G + 31) / 32;  // CTAs per lane in a column scan
  if (imode) {
    // this CTA's eligible counts per bucket: one dense row (16 KB, every launch)
    if (G > 1)
      reinterpret_cast<uint4 *>(d.f_crow + ((uint64_t)par * G + c) * NB1)[threadIdx.x] =
          reinterpret_cast<const uint4 *>(s.h + 2 * NB1)[threadIdx.x];  // (NB1 / 4 == FT)
    const uint32_t nov = s_novf;  // (CTA-uniform: the P1 loop ended with a barrier)
    if (nov) {
      __shared__ unsigned long long s_ovbase;
      if (threadIdx.x == 0)  // more than this CTA can stage: push the count past the cap
        s_ovbase = atomicAdd(&acc[6], nov <= LOVF ? (unsigned long long)nov : FUSED_OVF_CAP + 1ull);
      __syncthreads();
      const unsigned long long ob = s_ovbase;
      if (threadIdx.x < nov && nov <= LOVF && ob + threadIdx.x < FUSED_OVF_CAP)
        d.f_ovf[(uint64_t)par * BIG_OVF_CAP + ob + threadIdx.x] = s_ovf[threadIdx.x];
    }
  }
  STAMP_MAX(26)  // published
  st = __reduce_or_sync(0xFFFFFFFFu, st);
  if (lane == 0 && st) atomicOr(reinterpret_cast<unsigned int *>(&acc[5]), st);
  if (threadIdx.x == 0) {
    // integer mode: every distance is an integer or +inf, so level-1 bucket 0 (bits < 2^19)
    // holds exactly the d == 0 agents, all eligible (slot1(0) == 0)
    const unsigned long long zb = imode ? ((unsigned long long)s.h[NB1] << 16) + s.h[0] : parts_u64(sacc);
    if (zb) atomicAdd(&acc[0], zb);
  }
  STAMP_MAX(11)
  STAMP0(3)
  wgrid.sync();  // (the world's CTAs: every instance's own when nw == 1)
  STAMP0(4)
  // CTA 0's header inputs of the fast tail (the status bits, the plan sequence number, the
  // world's zero-distance bytes), all final now: copied into shared memory asynchronously, so
  // that the kernel does not end on a chain of dependent global loads
  // (16-byte pairs through L2 (cp.async.cg): acc[4..5], header[12..13], each rank's acc[0..1])
  __shared__ __align__(16) unsigned long long s_tail[4 + 2 * FUSED_MAX_WORLD];
  __shared__ uint32_t s_st0;
  if (c == 0 && threadIdx.x == 0) {
    cp_async16(&s_tail[0], &acc[4]);
    cp_async16(&s_tail[2], &d.header[H_SEQ - 1]);
    for (uint32_t r = 0; r < nw; ++r) cp_async16(&s_tail[4 + 2 * r], &W.acc[r][8 * par]);
    // (written by an earlier kernel: no stale L1 copy)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_st0)),
                 "l"(&d.state->status)
                 : "memory");
    cp_async_commit();
  }

  // ---------------- P2: select
  {  // clear the other parity's accumulators for the next launch, spread over the CTAs
    const int q = par ^ 1;
    const uint32_t gt = c * FT + threadIdx.x, gs = G * FT;
    for (uint32_t b = gt; b < NB1; b += gs) {
      d.f_hist1[NB1 * q + b] = 0;
      if (b < 64) d.f_hist1[2 * NB1 + 64 * q + b] = 0;  // coarse sums
      d.f_mm1[2 * NB1 * q + b] = 0xFFFFFFFFu;
      d.f_mm1[2 * NB1 * q + NB1 + b] = 0xFFFFFFFFu;
    }
    for (uint32_t b = gt; b < 2 * NBL; b += gs) d.f_tot[2 * NBL * q + b] = 0;
    for (uint32_t b = gt; b < 1024; b += gs) {
      d.f_hist2[1024 * q + b] = 0;
      d.f_hist3[1024 * q + b] = 0;
      d.f_mm2[2048 * q + b] = 0xFFFFFFFFu;
      d.f_mm2[2048 * q + 1024 + b] = 0xFFFFFFFFu;
    }
    if (gt < 8) d.f_acc[8 * q + gt] = 0;
  }
  // bucket owner: this CTA's range of every CTA's count row, staged while warp 0 selects
  const bool owners = imode && A.fastok && G > 1;
  if (owners && warp > 0) {
    const uint32_t ch = o_n / 4;  // 16-byte chunks per CTA row segment
    for (uint32_t x = threadIdx.x - 32; x < G * ch; x += FT - 32) {
      const uint32_t q = x / ch, k = x - q * ch;
      cp_async16(s.col + q * RB + 4 * k, d.f_crow + ((uint64_t)par * G + q) * NB1 + o_lo + 4 * k);
    }
    cp_async_commit();
  }
  // eligible agents in multi-valued buckets: this instance's (placed by its overflow CTA) and
  // the world's (the fast list decision must agree across the ranks)
  __shared__ unsigned long long sh_novf, sh_novf_w;
  if (threadIdx.x == 32) {  // (warp 0 runs the select)
    unsigned long long v = 0;
    if (imode)
      for (uint32_t r = 0; r < nw; ++r) v += W.acc[r][8 * par + 6];
    sh_novf_w = v;
    sh_novf = imode ? acc[6] : 0ull;
  }
  Sel sel = {0, 0, 0, 0xFFFFFFFFu, 0, 0, 1, 0};
  STAMP0(32)  // other parity cleared
  select_level1_warp(W, par, p.budget, sel, imode, prof);
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
    wgrid.sync();  // (the world's CTAs: every instance's own when nw == 1)
    select_level(W, par, level, p.budget, sel);
  }
  const bool all_fit = sel.all_fit;
  const uint32_t dstar = sel.dstar;
  STAMP0(9)

  // ---------------- fast list placement (integer distances; grid-uniform decision).  With the
  // boundary D* in a single-valued bucket b* (or everything kept), a list member's position
  // is known from counts published before B1: prefetch members (eligible non-residents kept)
  // of bucket b <= b* sit at  sum_{b' < b} NR[b'] + NR of b in the preceding CTAs + its rank
  // in this CTA (ascending id); evict members (residents not kept) of bucket b >= b* at
  // sum_{b' > b} R[b'] + R of b in the following CTAs + its rank (descending id).  At b* the
  // tie cut is an id prefix, so CTAs before the cut keep all their ties and CTAs after it keep
  // none: the same column sums hold there.  Agents in multi-valued buckets (rare, at most
  // FUSED_OVF_CAP) are ranked by one CTA.  No second grid barrier.
#ifdef AB_NO_FAST  // A/B experiments only (tools/)
  const bool fastp = false;
#else
  const bool fastp = imode && A.fastok && sh_novf_w <= FUSED_OVF_CAP &&
                     (all_fit || (sel.level_res == 1 && (sel.b_res < IB_EXACT || sel.b_res == IB_INF)));
#endif
  if (c == 0 && threadIdx.x == 0) atomicAdd(&prof[fastp ? 48 : 49], 1ull);  // launches per list path
  const uint32_t bs = all_fit ? (uint32_t)NB1 : sel.b_res;  // boundary bucket (NB1: every eligible agent kept)
  uint32_t *const lcnt = s.h + 2 * NB1;  // this CTA's eligible counts per bucket (P1)
  uint32_t *const need = s.h + 3 * NB1;  // buckets where this CTA has list members
  const uint32_t ep = A.epoch & 0xFFFFu;  // tags the owners' published offsets of this launch
  __shared__ uint32_t sh_m;
  uint32_t m_need = 0;
  // P3's load of the preceding CTAs' tie bytes goes out first (its latency hides behind the
  // owner pass)
  unsigned long long t_rows = 0;  // preceding CTAs' bytes in the resolving bucket (published rows)
  if (!all_fit && threadIdx.x < c) {
    const unsigned long long *rows = sel.level_res == 1 ? d.f_rows1 : (sel.level_res == 2 ? d.f_rows2 : d.f_rows3);
    const uint32_t stride = sel.level_res == 1 ? NB1 : 1024;
    t_rows = rows[(uint64_t)threadIdx.x * stride + sel.b_res];
  }
  // ... and the lower ranks' bytes at D* (rank r owns the r-th contiguous id range of the world)
  if (!all_fit && warp == FWARPS - 1 && lane < rank) {
    const unsigned long long *hh = sel.level_res == 1 ? W.h1[lane] + NB1 * par
                                                      : (sel.level_res == 2 ? W.h2[lane] : W.h3[lane]) + 1024 * par;
    t_rows = hh[sel.b_res];
  }
  if (owners) {
    cp_async_wait_all();
    __syncthreads();
    STAMP_MAX(40)  // owner staging landed
    if (fastp) {
      // Bucket owner pass (this CTA's range of RB buckets, every CTA's counts staged in s.col):
      // for bucket b and CTA q, the prefetch offset  W_nr(b) + sum_{q' < q} nr_q'(b)  and the
      // evict offset  W_r(b) + sum_{q' > q} r_q'(b), relative to the range start (W: the range's
      // buckets before b ascending / after b descending), published tagged with the launch
      // epoch; and the range totals.  Consumers add the range starts.
      uint32_t *tn = s.col + G * RB, *tr = tn + RB;
      for (uint32_t j = warp; j < o_n; j += FWARPS) {  // totals over the CTAs
        uint32_t a = 0, e = 0;
        for (uint32_t i = 0; i < QP; ++i) {
          const uint32_t q = lane * QP + i;
          if (q < G) {
            const uint32_t v = s.col[q * RB + j];
            a += v & 0xFFFFu;
            e += v >> 16;
          }
        }
        a = __reduce_add_sync(0xFFFFFFFFu, a);
        e = __reduce_add_sync(0xFFFFFFFFu, e);
        if (lane == 0) {
          tn[j] = a;
          tr[j] = e;
        }
      }
      __syncthreads();
      STAMP_MAX(46)  // owner pass 1
      // the range's totals (owner o's share of both lists), published; each warp of the pass below
      // sums the offsets of its bucket within the range itself (no serial scan)
      if (warp == 0) {
        uint32_t ta = 0, te = 0;
        for (uint32_t l = lane; l < o_n; l += 32) {
          ta += tn[l];
          te += tr[l];
        }
        ta = __reduce_add_sync(0xFFFFFFFFu, ta);
        te = __reduce_add_sync(0xFFFFFFFFu, te);
        if (lane == 0) st_relaxed_u64(&d.f_rt[par * FUSED_MAX_CTAS + c], pack_ep(ep, ta, te));
      }
      for (uint32_t j = warp; j < o_n; j += FWARPS) {  // per-CTA offsets: 32 consecutive CTAs per store
        uint32_t w_n = 0, w_r = 0;  // the range's buckets before j (prefetch) / after j (evict)
        for (uint32_t l0 = 0; l0 < o_n; l0 += 32) {
          const uint32_t l = l0 + lane;
          w_n += __reduce_add_sync(0xFFFFFFFFu, (l < o_n && l < j) ? tn[l] : 0u);
          w_r += __reduce_add_sync(0xFFFFFFFFu, (l < o_n && l > j) ? tr[l] : 0u);
        }
        const uint32_t t_r = tr[j];
        unsigned long long *P = d.f_pos + ((uint64_t)par * NB1 + o_lo + j) * FUSED_MAX_CTAS;
        // lane l owns CTAs [l QP, (l + 1) QP) (QP <= 5): their counts summed in registers, one
        // scan pair over the lanes, then the lane's own running sums (no chain of 32-CTA rounds)
        constexpr int QMAX = (FUSED_MAX_CTAS + 31) / 32;
        uint32_t vv[QMAX], a_l = 0, e_l = 0;
#pragma unroll
        for (int i = 0; i < QMAX; ++i) {
          const uint32_t q = lane * QP + i;
          vv[i] = ((uint32_t)i < QP && q < G) ? s.col[q * RB + j] : 0u;
          a_l += vv[i] & 0xFFFFu;
          e_l += vv[i] >> 16;
        }
        const uint32_t ia = warp_incl_scan(a_l), ie = warp_incl_scan(e_l);
        uint32_t ca = ia - a_l, ce = ie - e_l;  // the CTAs before the lane's first
        const uint32_t b = o_lo + j;
#pragma unroll
        for (int i = 0; i < QMAX; ++i) {
          const uint32_t q = lane * QP + i;
          const uint32_t v = vv[i], a = v & 0xFFFFu, e = v >> 16;
          // (only the entries a consumer reads: its list buckets, and CTA 0's / the last CTA's)
          const bool used =
#ifdef NO_OWNER_SKIP
            true;
#else
            (b < bs ? a != 0u : (b > bs ? e != 0u : v != 0u)) || q == 0 || q == G - 1;
#endif
          // prefetch: CTAs before q; evict: CTAs after q (total minus inclusive prefix)
          if ((uint32_t)i < QP && q < G && used) st_relaxed_u64(&P[q], pack_ep(ep, w_n + ca, w_r + t_r - (ce + e)));
          ca += a;
          ce += e;
        }
      }
    }
  }
  STAMP_MAX(41)  // owner pass done
  if (fastp && G > 1) {
    // the buckets where this CTA has list members (multi-valued ones go to the overflow CTA)
    if (threadIdx.x == 0) sh_m = 0;
    __syncthreads();
#pragma unroll 1
    for (uint32_t b = threadIdx.x; b < NB1; b += FT) {
      const uint32_t v = lcnt[b];
      const bool nd = !ib_multi(b) && (b < bs ? (v & 0xFFFFu) != 0u : (b > bs ? (v >> 16) != 0u : v != 0u));
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, nd);
      uint32_t j0 = 0;
      if (lane == 0 && bal) j0 = atomicAdd(&sh_m, (uint32_t)__popc(bal));
      j0 = __shfl_sync(0xFFFFFFFFu, j0, 0);
      if (nd) need[j0 + __popc(bal & lanemask_lt())] = b;
    }
    __syncthreads();
    m_need = sh_m;
  }
  STAMP_MAX(42)  // need list
  // the owners' range totals and this CTA's first list-bucket offsets: loads issued now (their
  // latency hides behind P3 / P4), the epoch tag checked where they are used
  unsigned long long rv_pre = 0, pv_pre = 0;
  // ... and the list starts CTA 0 (bucket b*) and the last CTA (the multi-valued buckets) need:
  // threads 0 / 1 of CTA 0 and 32 / 33 of the last CTA, one entry each (sp_b / sp_q: its bucket
  // and CTA column)
  unsigned long long sp_pre = 0;
  uint32_t sp_b = NB1, sp_q = 0;
  if (fastp && G > 1) {
    if (threadIdx.x < m_need)
      pv_pre = ld_relaxed_u64(d.f_pos + ((uint64_t)par * NB1 + need[threadIdx.x]) * FUSED_MAX_CTAS + c);
    if (threadIdx.x < G) rv_pre = ld_relaxed_u64(&d.f_rt[par * FUSED_MAX_CTAS + threadIdx.x]);
    if (c == 0 && threadIdx.x < 2 && bs < (uint32_t)NB1) {
      sp_b = bs;
      sp_q = threadIdx.x == 0 ? 0u : G - 1;
    }
    if (c == G - 1 && (threadIdx.x == 32 || threadIdx.x == 33)) {
      sp_b = threadIdx.x == 32 ? IB_EXACT : IB_INF - 1;
      sp_q = threadIdx.x == 32 ? 0u : G - 1;
    }
    if (sp_b < (uint32_t)NB1) sp_pre = ld_relaxed_u64(&d.f_pos[((uint64_t)par * NB1 + sp_b) * FUSED_MAX_CTAS + sp_q]);
  }

  // ---------------- fast list placement tail (integer distances, fastp: grid-uniform)
  if (fastp) {
    uint32_t *const h32 = s.h;  // [0, NB1): prefetch positions, [NB1, 2 NB1): evict positions
    __shared__ uint32_t sh_spf, sh_sev, sh_mvpf, sh_mvev;
    unsigned long long *word_tie = reinterpret_cast<unsigned long long *>(s.memb);  // [tw + 1]
    unsigned long long sh_tie_excl = 0;
    if (!all_fit) {  // (CTA-uniform)
      // P3: per word (a warp) the kept agents below D* and the tie group at D* (staged in the
      // prefetch / evict word arrays), the tie bytes; their id-order scan over the tile
#pragma unroll 1
      for (uint32_t w = warp; w < A.tw; w += FWARPS) {
        const uint32_t k = w * 32 + lane;
        const uint32_t elw = s.elig_w[w], key = s.keys[k];
        const uint32_t klt = __ballot_sync(0xFFFFFFFFu, key < dstar) & elw;
        const uint32_t tiew = __ballot_sync(0xFFFFFFFFu, key == dstar) & elw;
        unsigned long long v = 0;
        if (tiew) v = warp_sum_u32_exact(((tiew >> lane) & 1u) ? s.fp[k] : 0u);
        if (lane == 0) {
          word_tie[w] = v;
          s.pf_w[w] = klt;
          s.ev_w[w] = tiew;
        }
      }
      __syncthreads();
      if (warp * 32 < c || (warp == FWARPS - 1 && rank > 0)) warp_add_u64(t_rows, sacc + 20);  // preceding CTAs' and ranks' total
      {  // exclusive scan of the words' tie bytes on the first ceil(tw / 32) warps, one barrier
         // (which also completes the sum above)
        const uint32_t w = threadIdx.x, nsw = (A.tw + 31) / 32;
        __shared__ unsigned long long sh_wt[FWARPS];
        const unsigned long long v = w < A.tw ? word_tie[w] : 0ull;
        unsigned long long incl = 0;
        if ((uint32_t)warp < nsw) {
          incl = warp_incl_scan(v);
          if (lane == 31) sh_wt[warp] = incl;
        }
        __syncthreads();
        if ((uint32_t)warp < nsw) {
          unsigned long long pre = 0;
          for (int k = 0; k < warp; ++k) pre += sh_wt[k];
          if (w < A.tw) word_tie[w] = pre + incl - v;
          if ((uint32_t)warp == nsw - 1 && lane == 31) word_tie[A.tw] = pre + incl;  // (memb: tile / 2 >= tw + 1 u64)
        }
      }
      sh_tie_excl = parts_u64(sacc + 20);
      __syncthreads();
    }
    STAMP_MAX(14)
    // P4, one word per thread: kept word (the tie group's id-order prefix within the budget),
    // prefetch / evict words, new residency, byte sums; the write-back byte loads of the evicted
    // dirty agents go out now and are consumed at the end
    unsigned long long h2d = 0, tie_kept = 0;
    uint32_t pfw = 0, evw = 0, wbm = 0, wb0 = 0, wb1 = 0, n_el = 0;
    if (threadIdx.x < A.tw) {
      const uint32_t w = threadIdx.x;
      const uint32_t elw = s.elig_w[w];
      uint32_t kw = all_fit ? elw : s.pf_w[w];
      const uint32_t tiew = all_fit ? 0u : s.ev_w[w];
      if (tiew) {
        const unsigned long long lo = sh_tie_excl + word_tie[w], hi = sh_tie_excl + word_tie[w + 1];
        if (hi <= sel.rem) {
          kw |= tiew;
          tie_kept = hi - lo;
        } else if (lo <= sel.rem) {  // the one word of the grid that straddles the budget
          unsigned long long incl = lo;
          for (uint32_t m = tiew; m; m &= m - 1) {
            const uint32_t l = __ffs(m) - 1, fp = s.fp[w * 32 + l];
            incl += fp;
            if (incl <= sel.rem) {
              kw |= 1u << l;
              tie_kept += fp;
            }
          }
        }
      }
      const uint32_t old = s.old_w[w];
      pfw = kw & ~old;
      evw = old & ~kw;
      if (w < tw_here) bm_new[base / 32 + w] = kw;
      n_el = __popc(elw);
      for (uint32_t m = pfw; m; m &= m - 1) h2d += s.fp[w * 32 + __ffs(m) - 1];
      wbm = evw & s.dirty_w[w];
      const uint32_t *wbw = d.wb_bytes + base + 32 * w;
      if (wbm) {
        wb0 = wbw[__ffs(wbm) - 1];
        wbm &= wbm - 1;
      }
      if (wbm) {
        wb1 = wbw[__ffs(wbm) - 1];
        wbm &= wbm - 1;
      }
    }
    STAMP_MAX(27)  // P4 done
    warp_add_u44(h2d, sacc + 4);
    warp_add_u44(tie_kept, sacc + 8);
    n_el = __reduce_add_sync(0xFFFFFFFFu, n_el);
    if (lane == 0 && n_el) atomicAdd(&sacc[10], n_el);
    STAMP_MAX(50)
    // one scan for two things: [0] this tile's list members per word (prefetch | evict << 16 /
    // << 32), [1] the range starts from the owners' range totals (G > 1) or, one CTA, its own
    // counts.  G > 1: every nonzero value sits in the first max(tw, G) threads, and every sum fits
    // 32 bits (members of a tile < 2^16 per list, list lengths < 2^24), so only those warps scan,
    // in 32-bit parts, behind one barrier (measured: the generic two-level u64 scan took ~1 us)
    uint32_t vp, ve, tp, te, rs_pf = 0, rs_ev = 0, r_tot = 0, rp_tot = 0, re = 0, tv[4];
    unsigned long long s2_1 = 0, sv_1 = 0;  // (G == 1)
    if (G > 1) {
      unsigned long long rv = rv_pre;
      if (threadIdx.x < G && (uint32_t)(rv >> 48) != ep) rv = poll_ep(&d.f_rt[par * FUSED_MAX_CTAS + threadIdx.x], ep, d.header);
      re = threadIdx.x < G ? (uint32_t)rv & 0xFFFFFFu : 0u;
      const uint32_t a0 = (uint32_t)__popc(pfw) | ((uint32_t)__popc(evw) << 16);
      const uint32_t b0 = threadIdx.x < G ? (uint32_t)(rv >> 24) & 0xFFFFFFu : 0u;
      __shared__ uint32_t sh3[3][FWARPS];
      const uint32_t nsw = ((A.tw > G ? A.tw : G) + 31) / 32;  // (CTA-uniform)
      uint32_t ia = 0, ib = 0, ic = 0;
      if (warp < nsw) {
        ia = warp_incl_scan(a0);
        ib = warp_incl_scan(b0);
        ic = warp_incl_scan(re);
        if (lane == 31) {
          sh3[0][warp] = ia;
          sh3[1][warp] = ib;
          sh3[2][warp] = ic;
        }
      }
      __syncthreads();
      const uint32_t x0 = lane < nsw ? sh3[0][lane] : 0u, x2 = lane < nsw ? sh3[2][lane] : 0u;
      const uint32_t x1 = lane < nsw ? sh3[1][lane] : 0u;
      const uint32_t t0 = __reduce_add_sync(0xFFFFFFFFu, x0);
      r_tot = __reduce_add_sync(0xFFFFFFFFu, x2);
      rp_tot = __reduce_add_sync(0xFFFFFFFFu, x1);
      tp = t0 & 0xFFFFu;
      te = t0 >> 16;
      if (warp < nsw) {
        const uint32_t lt = (uint32_t)lane < (uint32_t)warp;
        const uint32_t e0 = __reduce_add_sync(0xFFFFFFFFu, lt ? x0 : 0u) + ia - a0;
        vp = e0 & 0xFFFFu;
        ve = e0 >> 16;
        rs_pf = __reduce_add_sync(0xFFFFFFFFu, lt ? x1 : 0u) + ib - b0;
        rs_ev = __reduce_add_sync(0xFFFFFFFFu, lt ? x2 : 0u) + ic - re;
      } else {
        vp = ve = 0;
      }
    } else {
      unsigned long long sv[2], s2[2];
      sv[0] = (unsigned long long)__popc(pfw) | ((unsigned long long)__popc(evw) << 32);
      unsigned long long loc = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        tv[k] = lcnt[4 * threadIdx.x + k];
        loc += (unsigned long long)(tv[k] & 0xFFFFu) | ((unsigned long long)(tv[k] >> 16) << 32);
      }
      sv[1] = loc;
      cta_scan2(sv, s2);
      vp = (uint32_t)sv[0];
      ve = (uint32_t)(sv[0] >> 32);
      tp = (uint32_t)s2[0];
      te = (uint32_t)(s2[0] >> 32);
      sv_1 = sv[1];
      s2_1 = s2[1];
      r_tot = (uint32_t)(s2_1 >> 32);
    }
    {  // this tile's members in list order (prefetch ascending id, evict descending id)
      const uint32_t w = threadIdx.x;
      uint32_t m = pfw, o = vp;
      while (m) {  // (bucket << 16 | local index: tile < 2^16)
        const uint32_t k = w * 32 + __ffs(m) - 1;
        s.memb[o++] = (ibucket(s.keys[k]) << 16) | k;
        m &= m - 1;
      }
      m = evw;
      o = tp + te - 1 - ve;
      while (m) {
        const uint32_t k = w * 32 + __ffs(m) - 1;
        s.memb[o--] = (ibucket(s.keys[k]) << 16) | k;
        m &= m - 1;
      }
    }
    if (G > 1) {
      uint32_t *rps = s.col, *rpe = s.col + G;  // range starts (the owner staging is free)
      if (threadIdx.x < G) {
        rps[threadIdx.x] = rs_pf;
        rpe[threadIdx.x] = r_tot - rs_ev - re;
      }
      __syncthreads();
      STAMP_MAX(53)
      // positions of this CTA's first member in each of its list buckets
      const unsigned long long *Pc = d.f_pos + (uint64_t)par * NB1 * FUSED_MAX_CTAS + c;
      for (uint32_t j = threadIdx.x; j < m_need; j += FT) {
        const uint32_t b = need[j];
        unsigned long long v = j == threadIdx.x ? pv_pre : ld_relaxed_u64(Pc + (uint64_t)b * FUSED_MAX_CTAS);
        if ((uint32_t)(v >> 48) != ep) v = poll_ep(Pc + (uint64_t)b * FUSED_MAX_CTAS, ep, d.header);
        h32[b] = rps[b / RB] + ((uint32_t)(v >> 24) & 0xFFFFFFu);
        h32[NB1 + b] = rpe[b / RB] + ((uint32_t)v & 0xFFFFFFu);
      }
      // the prefetched entry (sp_pre) of bucket sp_b, CTA column sp_q (0: the prefetch start,
      // sum_{b' < b} NR[b']; G - 1: the evict start, sum_{b' > b} R[b']), polled if not yet current
      auto sp_pos = [&]() {
        unsigned long long v = sp_pre;
        if ((uint32_t)(v >> 48) != ep) v = poll_ep(&d.f_pos[((uint64_t)par * NB1 + sp_b) * FUSED_MAX_CTAS + sp_q], ep, d.header);
        return sp_q == 0 ? rps[sp_b / RB] + ((uint32_t)(v >> 24) & 0xFFFFFFu) : rpe[sp_b / RB] + ((uint32_t)v & 0xFFFFFFu);
      };
      if (c == 0 && threadIdx.x < 2) {
        if (threadIdx.x == 0) sh_spf = bs < (uint32_t)NB1 ? sp_pos() : rp_tot;
        else sh_sev = bs < (uint32_t)NB1 ? sp_pos() : 0u;
      }
      if (c == G - 1 && (threadIdx.x == 32 || threadIdx.x == 33)) {
        if (threadIdx.x == 32) sh_mvpf = sp_pos();
        else sh_mvev = sp_pos();
      }
      STAMP_MAX(54)
    } else {
      // one CTA: its counts are the totals (S_pf(b) = sum_{b' < b} NR, S_ev(b) = sum_{b' > b} R)
      unsigned long long run = sv_1;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t b = 4 * threadIdx.x + k;
        run += (unsigned long long)(tv[k] & 0xFFFFu) | ((unsigned long long)(tv[k] >> 16) << 32);
        const uint32_t spf = (uint32_t)run - (tv[k] & 0xFFFFu), sev = r_tot - (uint32_t)(run >> 32);
        h32[b] = spf;
        h32[NB1 + b] = sev;
        if (b == bs) {
          sh_spf = spf;
          sh_sev = sev;
        }
        if (b == IB_EXACT) sh_mvpf = spf;
        if (b == IB_INF - 1) sh_mvev = sev;
      }
      if (bs == (uint32_t)NB1 && threadIdx.x == 0) {
        sh_spf = (uint32_t)s2_1;
        sh_sev = 0;
      }
    }
    __syncthreads();
    STAMP_MAX(38)  // positions and member lists
    const uint32_t m_pf = tp, m_ev = te;
    // positions: a member's place = its bucket's first position for this CTA + its rank among
    // the bucket's members before it in list order.  One thread per member (rank by a scan of the
    // members before it in shared memory) when both lists fit the CTA; else warp 0 the prefetch
    // members, warp 1 the evict members, 32 at a time in list order with the bucket positions as
    // cursors
    const bool par_place = m_pf + m_ev <= (uint32_t)FT;  // (CTA-uniform)
    if (par_place) {
      const uint32_t t = threadIdx.x;
      const bool pf = t < m_pf, mine = t < m_pf + m_ev;
      bool at_bs = false;
      if (mine) {
        const uint32_t i = pf ? t : t - m_pf;
        const uint32_t *mem = s.memb + (pf ? 0u : m_pf);
        const uint32_t bk = mem[i], b = bk >> 16;
        if (!ib_multi(b)) {
          uint32_t rank = 0;
          for (uint32_t j = 0; j < i; ++j) rank += (mem[j] >> 16) == b;
          (pf ? d.pf_ids : d.ev_ids)[h32[(pf ? 0u : (uint32_t)NB1) + b] + rank] = (uint32_t)(p.shard_begin + base + (bk & 0xFFFFu));
          at_bs = b == bs;
        }
      }
      const uint32_t npb = __popc(__ballot_sync(0xFFFFFFFFu, at_bs && pf)), neb = __popc(__ballot_sync(0xFFFFFFFFu, at_bs && !pf));
      if (lane == 0 && npb) atomicAdd(&d.header[H_N_PF], (unsigned long long)npb);
      if (lane == 0 && neb) atomicAdd(&d.header[H_N_EV], (unsigned long long)neb);
      PROBE(if (threadIdx.x == 0) atomicMax(&prof[43], gtimer());)
    } else if (warp < 2) {
      const uint32_t m = warp == 0 ? m_pf : m_ev;
      const uint32_t *mem = s.memb + (warp == 0 ? 0u : m_pf);
      uint32_t *cur = h32 + (warp == 0 ? 0u : (uint32_t)NB1);
      uint32_t *out = warp == 0 ? d.pf_ids : d.ev_ids;
      uint32_t nb = 0;
      for (uint32_t e0 = 0; e0 < m; e0 += 32) {
        const uint32_t e = e0 + lane;
        const uint32_t bk = e < m ? mem[e] : 0xFFFFFFFFu;
        const uint32_t k = bk & 0xFFFFu, b = e < m ? bk >> 16 : 0xFFFFFFFFu;
        const bool on = e < m && !ib_multi(b);
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, on ? b : 0xFFFFFFFFu);
        uint32_t pos = 0;
        if (on) pos = cur[b] + __popc(peers & lanemask_lt());
        __syncwarp();
        if (on && (peers & lanemask_lt()) == 0) cur[b] += __popc(peers);
        if (on) out[pos] = (uint32_t)(p.shard_begin + base + k);
        nb += __popc(__ballot_sync(0xFFFFFFFFu, on && b == bs));
        __syncwarp();
      }
      if (lane == 0 && nb) atomicAdd(&d.header[warp == 0 ? H_N_PF : H_N_EV], (unsigned long long)nb);
      PROBE(if (lane == 0) atomicMax(&prof[43 + warp], gtimer());)
    }
    if (c == G - 1 && sh_novf > 0 && warp >= 2) {
      // the agents in multi-valued buckets (all CTAs'): prefetch members (non-residents below
      // b*) after the value buckets below 2048, evict members (residents above b*) after the
      // +inf bucket; ranked by (key, id) among themselves
      __shared__ uint4 s_ov[FUSED_OVF_CAP];
      const uint32_t nov = (uint32_t)sh_novf;
      const uint32_t t = threadIdx.x - 64;  // warps 2..31 (named barrier 1)
      for (uint32_t x = t; x < nov; x += FT - 64) s_ov[x] = d.f_ovf[(uint64_t)par * BIG_OVF_CAP + x];
      asm volatile("bar.sync 1, %0;" ::"r"(FT - 64) : "memory");
      const uint32_t pf0 = sh_mvpf, ev0 = sh_mvev;
      for (uint32_t x = t; x < nov; x += FT - 64) {
        const uint4 q = s_ov[x];
        const uint32_t b = ibucket(q.x);
        const int lst = (!q.z && b < bs) ? 0 : ((q.z && b > bs) ? 1 : -1);
        if (lst < 0) continue;
        uint32_t rank = 0;
        for (uint32_t u = 0; u < nov; ++u) {
          const uint4 f = s_ov[u];
          const uint32_t fb = ibucket(f.x);
          if (lst == 0 ? (!f.z && fb < bs) : (f.z && fb > bs))
            rank += lst == 0 ? (f.x < q.x || (f.x == q.x && f.y < q.y)) : (f.x > q.x || (f.x == q.x && f.y > q.y));
        }
        if (lst == 0) d.pf_ids[pf0 + rank] = q.y;
        else d.ev_ids[ev0 + rank] = q.y;
      }
    }
    {
      unsigned long long d2h = (unsigned long long)wb0 + wb1;
      while (wbm) {  // (rare: a word with more than two dirty evicted agents)
        d2h += d.wb_bytes[base + 32 * threadIdx.x + __ffs(wbm) - 1];
        wbm &= wbm - 1;
      }
      warp_add_u44(d2h, sacc + 6);
    }
    __syncthreads();
    STAMP_MAX(39)  // placed
    if (threadIdx.x == 0) {  // this CTA's sums into the header (zeroed before B1)
      unsigned long long *H = d.header;
      const unsigned long long v_h2d = parts_u44(sacc + 4), v_tie = parts_u44(sacc + 8), v_wb = parts_u44(sacc + 6);
      if (v_h2d) atomicAdd(&H[H_H2D], v_h2d);
      for (uint32_t r = 0; r < nw; ++r) {  // world-wide fields: into every rank's header
        if (v_tie) atomicAdd(&W.hdr[r][H_KEPT], v_tie);
        if (sacc[10]) atomicAdd(&W.hdr[r][H_N_ELIG], (unsigned long long)sacc[10]);
      }
      if (v_wb) atomicAdd(&H[H_D2H], v_wb);
      if (c == 0) {
        if (sh_spf) atomicAdd(&H[H_N_PF], (unsigned long long)sh_spf);
        if (sh_sev) atomicAdd(&H[H_N_EV], (unsigned long long)sh_sev);
        atomicAdd(&H[H_KEPT], p.budget - sel.rem);
        cp_async_wait_all();  // (s_tail, s_st0: this thread's copies)
        uint32_t status = (uint32_t)s_tail[1] | s_st0;
        unsigned long long zb = 0;  // bytes of the world's distance-0 agents
        for (uint32_t r = 0; r < nw; ++r) zb += s_tail[4 + 2 * r];
        if (zb > p.budget) status |= ST_INSUFFICIENT;
        H[H_CUT_BITS] = all_fit ? 0xFFFFFFFFull : dstar;
        H[H_CUT_REM] = sel.rem;
        atomicOr(reinterpret_cast<unsigned int *>(&H[H_STATUS]), status);
        H[H_SEQ] = s_tail[3] + 1;
      }
    }
      STAMP_MAX(1)
    return;
  }
  // ---------------- P3 (general path): tie group: id-order prefix of the bytes at d == D*
  unsigned long long *word_tie = reinterpret_cast<unsigned long long *>(s.memb);  // [tw]
#pragma unroll 1
  for (uint32_t w = warp; w < A.tw; w += FWARPS) {
    const uint32_t k = w * 32 + lane;
    const bool tie = !all_fit && ((s.elig_w[w] >> lane) & 1u) && s.keys[k] == dstar;
    unsigned long long v = 0;
    if (__ballot_sync(0xFFFFFFFFu, tie)) v = warp_sum_u32_exact(tie ? s.fp[k] : 0u);  // most words: no tie
    if (lane == 0) word_tie[w] = v;
  }
  __syncthreads();
  // exclusive scan over the tile's words (tw <= FUSED_MAX_TILE / 32 <= FT: one word per
  // thread) and, in the same pass, the preceding CTAs' total
  if (warp * 32 < c || (warp == FWARPS - 1 && rank > 0)) warp_add_u64(t_rows, sacc + 20);  // preceding CTAs' and ranks' total
  {
    const uint32_t w = threadIdx.x;
    unsigned long long v[1] = {w < A.tw ? word_tie[w] : 0ull}, tt[1];
    cta_scan1(v, tt);  // (its barriers complete the sum)
    if (w < A.tw) word_tie[w] = v[0];
    if (threadIdx.x == 0) word_tie[A.tw] = tt[0];  // (memb holds tile / 2 >= tw + 1 words of 64 bits)
  }
  const unsigned long long sh_tie_excl = parts_u64(sacc + 20);
  __syncthreads();
  STAMP0(10)
  STAMP_MAX(14)

  // ---------------- P4: emit
  uint32_t *cnt_pf = s.h, *cnt_ev = s.h + NBL;  // per-CTA list members per list bucket
  uint32_t *lor_l = s.h + 6 * NBL;   // [2][NBL]: OR of the key bits below the list bucket
  uint32_t *mm_l = s.h + 10 * NBL;  // [4][NBL]: prefetch min, prefetch ~max, evict min, evict ~max
  for (int b = threadIdx.x; b < 2 * NBL; b += FT) {
    s.h[b] = 0;
    lor_l[b] = 0;
  }
  for (int b = threadIdx.x; b < 4 * NBL; b += FT) mm_l[b] = 0xFFFFFFFFu;
  __syncthreads();
  unsigned long long h2d = 0, tie_kept = 0;
  uint32_t n_el = 0;
#pragma unroll 1
  for (uint32_t w = warp; w < A.tw; w += FWARPS) {
    const uint32_t k = w * 32 + lane;
    const uint32_t elw = s.elig_w[w];  // 0 beyond n_here
    const uint32_t key = s.keys[k];
    uint32_t kw = elw;  // kept agents of the word
    if (!all_fit) {
      kw = __ballot_sync(0xFFFFFFFFu, key < dstar) & elw;
      const uint32_t tiew = __ballot_sync(0xFFFFFFFFu, key == dstar) & elw;
      if (tiew) {  // id-order inclusive prefix of the tie bytes
        const bool tie = (tiew >> lane) & 1u;
        const uint32_t fp = s.fp[k];
        // the word's tie bytes lie in (lo, hi]: every tie of the word fits when hi <= rem, none
        // when lo > rem (one word of the grid straddles rem: only it needs the in-word prefix)
        const unsigned long long lo = sh_tie_excl + word_tie[w], hi = sh_tie_excl + word_tie[w + 1];
        if (hi <= sel.rem) {
          if (tie) tie_kept += fp;
          kw |= tiew;
        } else if (lo <= sel.rem) {
          unsigned long long incl = tie ? fp : 0u;
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
          }
          incl += lo;
          const bool ok = tie && incl <= sel.rem;
          if (ok) tie_kept += fp;
          kw |= __ballot_sync(0xFFFFFFFFu, ok);
        }
      }
    }
    const uint32_t old = s.old_w[w];
    const uint32_t pfw = kw & ~old, evw = old & ~kw;
    if (lane == 0) {
      if (w < tw_here) bm_new[base / 32 + w] = kw;
      s.pf_w[w] = pfw;
      s.ev_w[w] = evw;
      n_el += __popc(elw);
    }
    if (pfw | evw) {  // list members in this word (list-bucket counts)
      const uint32_t bk = key >> 21;
      if ((pfw >> lane) & 1u) {
        h2d += s.fp[k];
        atomicAdd(&cnt_pf[bk], 1u);
        atomicMin(&mm_l[bk], key);
        atomicMin(&mm_l[NBL + bk], ~key);
        atomicOr(&lor_l[bk], key & 0x1FFFFFu);
      }
      if ((evw >> lane) & 1u) {
        atomicAdd(&cnt_ev[bk], 1u);
        atomicMin(&mm_l[2 * NBL + bk], key);
        atomicMin(&mm_l[3 * NBL + bk], ~key);
        atomicOr(&lor_l[NBL + bk], key & 0x1FFFFFu);
      }
    }
  }
  __syncthreads();
  STAMP_MAX(27)  // P4 word loop done
  // list bucket totals (global atomics, issued now: they drain while the members are
  // staged); the CTA's min / max key and OR of the low key bits per bucket go to its rows
  {
    uint32_t *tot_pf = d.f_tot + 2 * NBL * par, *tot_ev = d.f_tot + 2 * NBL * par + NBL;
    uint32_t *rm = d.f_cta_lmm + (uint64_t)c * 6 * NBL;
    const int b = threadIdx.x;  // NBL == FT
    const uint32_t a = cnt_pf[b], e = cnt_ev[b];
    if (a) {
      atomicAdd(&tot_pf[b], a);
      rm[b] = mm_l[b];
      rm[NBL + b] = mm_l[NBL + b];
      rm[2 * NBL + b] = lor_l[b];
    }
    if (e) {
      atomicAdd(&tot_ev[b], e);
      rm[3 * NBL + b] = mm_l[2 * NBL + b];
      rm[4 * NBL + b] = mm_l[3 * NBL + b];
      rm[5 * NBL + b] = lor_l[NBL + b];
    }
  }
  // This tile's list members in list order (prefetch ascending id, evict descending id) into
  // memb, and the bucket-major offsets of the staging area (one word / bucket per thread:
  // tw <= FT == NBL)
  uint32_t *off_pf = s.h + 2 * NBL, *off_ev = s.h + 3 * NBL;
  __shared__ uint32_t sh_mpf, sh_mev;
  // (the scan's barriers complete them; per thread: <= 12 agents of < 2^32 bytes each < 2^44;
  // n_el lives in lane 0 only)
  warp_add_u44(h2d, sacc + 4);
  warp_add_u44(tie_kept, sacc + 8);
  if (lane == 0 && n_el) atomicAdd(&sacc[10], n_el);
  // This tile's list members in list order (prefetch ascending id, evict descending id) into
  // memb, and the bucket-major offsets of the staging area (one word / bucket per thread:
  // tw <= FT == NBL)
  {
    const uint32_t w = threadIdx.x;
    const uint32_t pw = w < A.tw ? s.pf_w[w] : 0u, ew = w < A.tw ? s.ev_w[w] : 0u;
    // four scans in one: 16-bit fields of a 64-bit value (every prefix <= tile < 2^16)
    const unsigned long long pk = (unsigned long long)__popc(pw) | ((unsigned long long)__popc(ew) << 16) |
                                  ((unsigned long long)cnt_pf[w] << 32) | ((unsigned long long)cnt_ev[w] << 48);
    unsigned long long pv[1] = {pk}, pt[1];
    cta_scan1(pv, pt);
    const uint32_t v[4] = {(uint32_t)(pv[0] & 0xFFFFu), (uint32_t)((pv[0] >> 16) & 0xFFFFu),
                           (uint32_t)((pv[0] >> 32) & 0xFFFFu), (uint32_t)(pv[0] >> 48)};
    const uint32_t tt[2] = {(uint32_t)(pt[0] & 0xFFFFu), (uint32_t)((pt[0] >> 16) & 0xFFFFu)};
    off_pf[w] = v[2];
    off_ev[w] = v[3];
    if (threadIdx.x == 0) {
      sh_mpf = tt[0];
      sh_mev = tt[1];
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
  STAMP_MAX(17)  // member lists built
  const uint32_t m_pf = sh_mpf, m_ev = sh_mev;
  // staging slot of every member (bucket start + rank within its bucket in list order), warp
  // 0 prefetch, warp 1 evict, into fp[]; the bucket offsets serve as cursors (each ends at
  // its bucket's end: start = off - cnt)
  if (warp < 2) {
    const uint32_t *mem = s.memb + (warp == 0 ? 0 : m_pf);
    const uint32_t m = warp == 0 ? m_pf : m_ev;
    uint32_t *run = warp == 0 ? off_pf : off_ev;
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
  }
  __syncthreads();
  STAMP_MAX(19)  // in-bucket ranks
  // stage (key, id) bucket-major in this tile's range of the staging arrays: bucket b's
  // members at base + off[b] + rank, in list order
  for (uint32_t e = threadIdx.x; e < m_pf + m_ev; e += FT) {
    const uint32_t k = s.memb[e];
    const uint32_t key = s.keys[k];
    const uint32_t id = (uint32_t)(p.shard_begin + base + k);
    if (e < m_pf) {
      const uint64_t slot = base + s.fp[e];
      d.sort_ka[slot] = key;
      d.sort_va[slot] = id;
    } else {
      const uint64_t slot = base + s.fp[e];
      d.f_sk2[slot] = key;
      d.f_sv2[slot] = id;
    }
  }
  {  // rows: offset << 16 | count (tile <= FUSED_MAX_TILE < 2^16)
    const int b = threadIdx.x;  // NBL == FT
    d.f_cta_cpf[(uint64_t)c * NBL + b] = ((off_pf[b] - cnt_pf[b]) << 16) | cnt_pf[b];
    d.f_cta_cev[(uint64_t)c * NBL + b] = ((off_ev[b] - cnt_ev[b]) << 16) | cnt_ev[b];
  }
  STAMP_MAX(28)  // staged, rows published
  if (threadIdx.x < 4) {
    const unsigned long long v = threadIdx.x < 3 ? parts_u44(sacc + 4 + 2 * threadIdx.x) : sacc[10];
    if (v && threadIdx.x != 1) atomicAdd(&acc[1 + threadIdx.x], v);  // ([2] write-back bytes: end of P5)
  }
  if (c == 0 && threadIdx.x == 0) d.header[H_D2H] = 0ull;  // (summed by every CTA after B4)
  STAMP_MAX(12)
  STAMP0(5)
  wgrid.sync();  // (the world's CTAs: every instance's own when nw == 1)
  STAMP0(6)
  if (c == 0 && threadIdx.x == 32) {  // header (CTA 0, warp 1): the accumulators are complete; loads first
    unsigned long long a0 = 0, a3 = 0, a4 = 0;  // world sums: zero-distance bytes, tie bytes kept, eligible
    for (uint32_t r = 0; r < nw; ++r) {
      const unsigned long long *ar = W.acc[r] + 8 * par;
      a0 += ar[0];
      a3 += ar[3];
      a4 += ar[4];
    }
    const unsigned long long a1 = acc[1], a5 = acc[5];
    const uint32_t st0 = d.state->status;  // + BAD_KIN/BAD_RECORD of k_int_compact
    unsigned long long *H = d.header;
    const unsigned long long seq = H[H_SEQ];
    H[H_H2D] = a1;
    H[H_CUT_BITS] = all_fit ? 0xFFFFFFFFull : dstar;
    H[H_CUT_REM] = sel.rem;
    H[H_KEPT] = (p.budget - sel.rem) + (all_fit ? 0ull : a3);
    H[H_N_ELIG] = a4;
    uint32_t status = (uint32_t)a5 | st0;
    if (a0 > p.budget) status |= ST_INSUFFICIENT;
    H[H_STATUS] = status;
    H[H_SEQ] = seq + 1;
  }
  STAMP_MAX(30)  // B4 passed (last CTA)

  // A single-CTA instance (G == 1, the batched replicas of C5) holds every list member in its
  // own staging area, bucket-major (buckets ascending) and in list order within a bucket,
  // with P4's per-bucket counts, end offsets and min / max keys still in s.h: each member's
  // list position follows from its segment directly (single-valued segment: its staging
  // rank; otherwise by counting within the segment when every such segment holds <= 128
  // members), else one stable radix sort per list — instead of one P5 slot per nonempty
  // list bucket (tools/c5_probe.py: 30 slots of ~2 us for 473 members).
  // (batched launches only: a single context's group spans every SM)
  const bool one_cta = MAXB > 1 && G == 1 && 4 * max(m_pf, m_ev) <= 3 * A.tile;
  if constexpr (MAXB > 1) if (one_cta) {
    const uint32_t *mm = s.h + 10 * NBL;  // [4][NBL]: prefetch min, ~max, evict min, ~max
    bool big = false;
    for (uint32_t b = threadIdx.x; b < NBL; b += FT)
      big |= (s.h[b] > 128u && mm[b] != ~mm[NBL + b]) || (s.h[NBL + b] > 128u && mm[2 * NBL + b] != ~mm[3 * NBL + b]);
    big = __syncthreads_or(big);
#pragma unroll 1
    for (uint32_t list = 0; list < 2; ++list) {
      const uint32_t len = list == 0 ? m_pf : m_ev;
      if (len == 0) continue;
      const uint32_t *sk = list == 0 ? d.sort_ka : d.f_sk2, *sv = list == 0 ? d.sort_va : d.f_sv2;
      uint32_t *ka = s.keys, *ia = ka + len, *kb = ka + 2 * len, *ib = ka + 3 * len;  // 4 len <= 3 tile
      uint32_t *out = list == 0 ? d.pf_ids : d.ev_ids;
      for (uint32_t e = threadIdx.x; e < len; e += FT) {
        ka[e] = (list == 0 || !big) ? sk[e] : ~sk[e];
        ia[e] = sv[e];
      }
      __syncthreads();
      if (!big) {
        // prefetch: position = segment start + members with a smaller key or an equal key
        // earlier in staging (ascending id); evict (buckets and keys descending): members
        // of higher buckets + members with a larger key or an equal key earlier (descending id)
        for (uint32_t e = threadIdx.x; e < len; e += FT) {
          const uint32_t k = ka[e], bk = k >> 21;
          const uint32_t end = s.h[(2 + list) * NBL + bk], beg = end - s.h[list * NBL + bk];
          uint32_t pos = (list == 0 ? beg : len - end) + (e - beg);
          if (mm[2 * list * NBL + bk] != ~mm[(2 * list + 1) * NBL + bk]) {  // several distances
            pos = list == 0 ? beg : len - end;
            for (uint32_t x = beg; x < end; ++x) {
              const uint32_t kx = ka[x];
              pos += (list == 0 ? kx < k : kx > k) || (kx == k && x < e);
            }
          }
          out[pos] = ia[e];
        }
      } else {
        cta_sort_pairs(ka, ia, kb, ib, len, s.h);  // stable: ties keep the staging (list) order
        for (uint32_t e = threadIdx.x; e < len; e += FT) out[e] = ia[e];
      }
      __syncthreads();
    }
  }

  // ---------------- P5: list order.  A segment is the members of one list bucket, in list
  // order (prefetch: ascending key; evict: descending key); its position in the list follows
  // from the bucket totals.  Segments are cut into slices of CH elements, one slice per slot,
  // slots dealt round-robin to the CTAs.  A slot gathers its segment from the CTAs' staging
  // areas (CTA order = id order) and places
  //   SINGLE  (one distance in the segment): its slice as is (already in (distance, id) order);
  //   COUNT   (codes (key - min) >> g span <= RMAX values): its slice by a stable counting
  //           sort whose counts cover the whole segment;
  //   SORT1 / BIG (wider codes): the whole segment by a stable radix sort in shared / global
  //           memory (one slot).
  constexpr uint32_t RMAX = 2 * NBL;
  enum { M_NONE = 0, M_SINGLE, M_COUNT, M_SORT1, M_BIG };
  // per segment (index gp in list order: prefetch buckets ascending, then evict buckets
  // descending): first slot, list position, length
  uint32_t *slot_base = s.h + 6 * NBL, *seg_start = s.h + 8 * NBL, *seg_len = s.h + 10 * NBL;
  uint32_t npf, nev, CH;  // list lengths, slice length (every thread)
  __shared__ uint32_t sh_ns;
  {
    // thread t: segments 2t, 2t+1 (never on both lists: NBL is even)
    const uint32_t list = 2 * threadIdx.x < NBL ? 0u : 1u;
    const uint32_t *tot = d.f_tot + 2 * NBL * par + list * NBL;
    uint32_t len[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t gp = 2 * threadIdx.x + q;
      len[q] = tot[list == 0 ? gp : 2 * NBL - 1 - gp];
    }
    // one scan: list positions of the segments and their first slots (slices of CH = 512)
    CH = 512;
    const uint32_t ns0 = (len[0] + CH - 1) / CH, ns1 = (len[1] + CH - 1) / CH;
    // three scans in one: 21-bit fields of a 64-bit value (fused path: n_local <= 148 x 12288
    // < 2^21, slots <= n_local / 512 + 2048)
    const unsigned long long pk = (unsigned long long)(list == 0 ? len[0] + len[1] : 0u) |
                                  ((unsigned long long)(list == 1 ? len[0] + len[1] : 0u) << 21) |
                                  ((unsigned long long)(ns0 + ns1) << 42);
    unsigned long long pv[1] = {pk}, pt[1];
    cta_scan1(pv, pt);
    const uint32_t M21 = (1u << 21) - 1;
    const uint32_t v[3] = {(uint32_t)(pv[0] & M21), (uint32_t)((pv[0] >> 21) & M21), (uint32_t)(pv[0] >> 42)};
    const uint32_t tt[3] = {(uint32_t)(pt[0] & M21), (uint32_t)((pt[0] >> 21) & M21), (uint32_t)(pt[0] >> 42)};
    STAMP_MAX(31)  // totals loaded and scanned
    npf = tt[0];
    nev = tt[1];
    seg_start[2 * threadIdx.x] = v[list];
    seg_start[2 * threadIdx.x + 1] = v[list] + len[0];
    seg_len[2 * threadIdx.x] = len[0];
    seg_len[2 * threadIdx.x + 1] = len[1];
    slot_base[2 * threadIdx.x] = v[2];
    slot_base[2 * threadIdx.x + 1] = v[2] + ns0;
    if (threadIdx.x == 0) sh_ns = tt[2];
  }
  if (c == 0 && threadIdx.x == 0) {
    d.header[H_N_PF] = npf;
    d.header[H_N_EV] = nev;
  }
  __syncthreads();
  const uint32_t n_slots = one_cta ? 0u : sh_ns;
  // R13 write-back bytes of this tile's dirty evicted agents: loads issued now (up to two per
  // word in registers), summed after the slot loop (their latency hides behind P5) and added
  // to the header by a reduction
  uint32_t wbm = 0, wb0 = 0, wb1 = 0;
  if (threadIdx.x < A.tw) {
    wbm = s.ev_w[threadIdx.x] & s.dirty_w[threadIdx.x];
    const uint32_t *wbw = d.wb_bytes + base + 32 * threadIdx.x;
    if (wbm) {
      wb0 = wbw[__ffs(wbm) - 1];
      wbm &= wbm - 1;
    }
    if (wbm) {
      wb1 = wbw[__ffs(wbm) - 1];
      wbm &= wbm - 1;
    }
  }
  PROBE(if (c == 0 && threadIdx.x == 0) prof[16] = n_slots;)
  STAMP_MAX(13)  // P5 tables
  STAMP0(7)
  __shared__ uint32_t col_pre[FUSED_MAX_CTAS], col_src[FUSED_MAX_CTAS];
  __shared__ uint32_t sh_gp, sh_tmp;
  PROBE(const unsigned long long t_s0 = gtimer();)
  PROBE(unsigned long long dt[4] = {0, 0, 0, 0};)
  for (uint32_t j = c; j < n_slots; j += G) {
    PROBE(unsigned long long tq = gtimer();)
    {  // the segment holding slot j
      const uint32_t g0 = 2 * threadIdx.x;
      const uint32_t a = slot_base[g0], m = slot_base[g0 + 1], z = g0 + 2 < 2 * NBL ? slot_base[g0 + 2] : n_slots;
      if (a <= j && j < m) sh_gp = g0;
      if (m <= j && j < z) sh_gp = g0 + 1;
    }
    __syncthreads();
    const uint32_t gp = sh_gp;
    const uint32_t list = gp < NBL ? 0u : 1u, b = list == 0 ? gp : 2 * NBL - 1 - gp;
    const uint32_t len = seg_len[gp];
    const uint32_t si = j - slot_base[gp];
    // the segment's members in each CTA (list order of the CTAs: prefetch ascending, evict
    // descending): first position and staging address; the segment's min / max key and OR of
    // the low key bits
    // (warps holding CTA columns: G <= FUSED_MAX_CTAS <= 8 * 32; warp scans and REDUX, the
    // warp totals combined by every thread: two CTA barriers)
    uint32_t smin, smax, slo;
    {
      __shared__ uint32_t w_sum[8], w_mm[3][8];
      uint32_t cnt = 0, src = 0, mn = 0xFFFFFFFFu, nmx = 0xFFFFFFFFu, lo = 0, incl = 0;
      if ((int)threadIdx.x < (int)G) {
        const uint32_t q = list == 0 ? threadIdx.x : G - 1 - threadIdx.x;
        const uint32_t pk = (list == 0 ? d.f_cta_cpf : d.f_cta_cev)[(uint64_t)q * NBL + b];
        const uint32_t *rm = d.f_cta_lmm + (uint64_t)q * 6 * NBL + 3 * list * NBL + b;
        const uint32_t m0 = rm[0], m1 = rm[NBL], m2 = rm[2 * NBL];
        cnt = pk & 0xFFFFu;
        src = q * A.tile + (pk >> 16);
        if (cnt) {
          mn = m0;
          nmx = m1;
          lo = m2;
        }
      }
      // COUNT mode's code counters and per-warp code counts, cleared while the column loads
      // are in flight (ordered by the barriers below; the previous slot ended with one)
      for (uint32_t x = threadIdx.x; x < 4 * NBL; x += FT) s.h[x] = 0;            // h_all, h_bef
      for (uint32_t x = threadIdx.x; x < 4 * NBL; x += FT) s.h[12 * NBL + x] = 0;  // hw
      const uint32_t nwg = (G + 31) / 32;
      if ((uint32_t)warp < nwg) {
        incl = warp_incl_scan(cnt);
        mn = __reduce_min_sync(0xFFFFFFFFu, mn);
        nmx = __reduce_min_sync(0xFFFFFFFFu, nmx);
        lo = __reduce_or_sync(0xFFFFFFFFu, lo);
        if (lane == 31) {
          w_sum[warp] = incl;
          w_mm[0][warp] = mn;
          w_mm[1][warp] = nmx;
          w_mm[2][warp] = lo;
        }
      }
      __syncthreads();
      uint32_t a0 = 0xFFFFFFFFu, a1 = 0xFFFFFFFFu, a2 = 0u, pre = incl - cnt;
      for (uint32_t w2 = 0; w2 < nwg; ++w2) {
        a0 = min(a0, w_mm[0][w2]);
        a1 = min(a1, w_mm[1][w2]);
        a2 |= w_mm[2][w2];
        if (w2 < (uint32_t)warp) pre += w_sum[w2];
      }
      smin = a0;
      smax = ~a1;
      slo = a2;
      if ((int)threadIdx.x < (int)G) {
        col_pre[threadIdx.x] = pre;
        col_src[threadIdx.x] = src - pre;  // staging index of segment element e: col_src[o] + e
      }
      __syncthreads();
    }

    uint32_t mode, g = 0;
    if (smin == smax) mode = M_SINGLE;
    else {
      g = __ffs(slo) - 1;  // every key - min is a multiple of 2^g (same bits [31:21])
      mode = ((smax - smin) >> g) < RMAX ? M_COUNT : (4 * len <= 3 * A.tile ? M_SORT1 : M_BIG);
    }
    const uint32_t org = list == 0 ? smin : smax;  // code origin
    if (mode >= M_SORT1 && si > 0) {  // the segment's first slot sorts all of it
      __syncthreads();
      continue;
    }
    // staging index of segment element e: the last CTA o whose first position is <= e
    auto src_of = [&](uint32_t e) -> uint32_t {
      uint32_t lo = 0, hi = G;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (col_pre[mid] <= e) lo = mid;
        else hi = mid;
      }
      return col_src[lo] + e;
    };
    const uint32_t *sk = list == 0 ? d.sort_ka : d.f_sk2, *sv = list == 0 ? d.sort_va : d.f_sv2;
    uint32_t *out = (list == 0 ? d.pf_ids : d.ev_ids) + seg_start[gp];
    auto lap = [&](int i) {
      PROBE(const unsigned long long t = gtimer(); dt[i] += t - tq; tq = t;)
    };
    lap(0);
    const uint32_t e0 = si * CH, e1 = min(len, e0 + CH);
    if (mode == M_SINGLE) {
      for (uint32_t e = e0 + threadIdx.x; e < e1; e += FT) out[e] = sv[src_of(e)];
    } else if (mode == M_COUNT) {
      uint32_t *h_all = s.h, *h_bef = s.h + 2 * NBL, *sc = s.h + 4 * NBL, *sid = s.h + 5 * NBL;
      for (uint32_t e00 = 0; e00 < len; e00 += 4 * FT) {
        uint32_t key[4], id[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // loads first
          const uint32_t e = e00 + q * FT + threadIdx.x;
          if (e < len) {
            const uint32_t sidx = src_of(e);
            key[q] = sk[sidx];
            id[q] = (e >= e0 && e < e1) ? sv[sidx] : 0u;
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t e = e00 + q * FT + threadIdx.x;
          if (e < len) {
            const uint32_t code = (list == 0 ? key[q] - org : org - key[q]) >> g;
            atomicAdd(&h_all[code], 1u);
            if (e < e0) atomicAdd(&h_bef[code], 1u);
            else if (e < e1) {
              sc[e - e0] = code;
              sid[e - e0] = id[q];
            }
          }
        }
      }
      __syncthreads();
      lap(1);
      const uint32_t rseg = ((smax - smin) >> g) + 1, nsl = e1 - e0;
      if (rseg <= 128) {
        // position = start of the code + members before the slice + members of earlier warps
        // of the slice + earlier lanes of the warp (all warps at once: per-warp code counts);
        // the code starts are scanned by the last warp meanwhile (nsl <= CH: it holds no slice)
        uint32_t *hw = s.h + 12 * NBL;  // [32 warps][128 codes], cleared at the slot's start
        const uint32_t nw = (nsl + 31) / 32;
        const uint32_t x = warp * 32 + lane;
        const bool on = x < nsl;
        uint32_t code = 0xFFFFFFFFu, rin = 0;
        if (warp < nw) {
          code = on ? sc[x] : 0xFFFFFFFFu;
          const uint32_t peers = __match_any_sync(0xFFFFFFFFu, code);
          rin = __popc(peers & lanemask_lt());
          if (on && rin == 0) hw[warp * 128 + code] = __popc(peers);
        } else if (warp == FWARPS - 1) {
          uint32_t v[4], t = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            v[i] = h_all[4 * lane + i];
            t += v[i];
          }
          uint32_t ex = warp_incl_scan(t) - t;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            h_all[4 * lane + i] = ex;
            ex += v[i];
          }
        }
        __syncthreads();
        lap(2);
        for (uint32_t c2 = threadIdx.x; c2 < rseg; c2 += FT) {  // exclusive prefix over the warps
          uint32_t run = 0;
          for (uint32_t w2 = 0; w2 < nw; ++w2) {
            const uint32_t v = hw[w2 * 128 + c2];
            hw[w2 * 128 + c2] = run;
            run += v;
          }
        }
        __syncthreads();
        if (on) out[h_all[code] + h_bef[code] + hw[warp * 128 + code] + rin] = sid[x];
      } else {
        {  // exclusive scan of the code counts (2 bins per thread)
          const uint32_t v0 = h_all[2 * threadIdx.x], v1 = h_all[2 * threadIdx.x + 1];
          const uint32_t ex = block_excl_scan<uint32_t, FT>(v0 + v1, &sh_tmp);
          h_all[2 * threadIdx.x] = ex;
          h_all[2 * threadIdx.x + 1] = ex + v0;
        }
        __syncthreads();
        lap(2);
        if (warp == 0) {  // the slice in order, one warp: position = start + earlier members with the same code
          for (uint32_t x0 = 0; x0 < e1 - e0; x0 += 32) {
            const uint32_t x = x0 + lane;
            const bool on = x < e1 - e0;
            const uint32_t code = on ? sc[x] : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, code);
            if (on) out[h_all[code] + h_bef[code] + __popc(peers & lanemask_lt())] = sid[x];
            __syncwarp();
            if (on && (peers & lanemask_lt()) == 0) h_bef[code] += __popc(peers);
            __syncwarp();
          }
        }
      }
    } else {  // M_SORT1 / M_BIG: the whole segment
      uint32_t *ka, *ia, *kb, *ib;
      if (mode == M_SORT1) {  // 4 * len <= 3 * tile words of keys / fp / memb
        ka = s.keys;
        ia = ka + len;
        kb = ka + 2 * len;
        ib = ka + 3 * len;
      } else {  // disjoint global ranges: prefetch [0, npf), evict [npf, npf + nev)
        const uint32_t at = (list == 0 ? 0u : npf) + seg_start[gp];
        ka = d.sort_kb + at;
        ia = d.sort_vb + at;
        kb = d.f_sk3 + at;
        ib = d.f_sv3 + at;
      }
      for (uint32_t e = threadIdx.x; e < len; e += FT) {
        const uint32_t sidx = src_of(e);
        const uint32_t key = sk[sidx];
        ka[e] = (list == 0 ? key - org : org - key) >> g;  // order-preserving code
        ia[e] = sv[sidx];
      }
      __syncthreads();
      cta_sort_pairs(ka, ia, kb, ib, len, s.h);  // counters in s.h[0, 4096)
      for (uint32_t e = threadIdx.x; e < len; e += FT) out[e] = ia[e];
      PROBE(if (threadIdx.x == 0) atomicMax(&prof[18], (unsigned long long)len);)
    }
    __syncthreads();
    lap(3);
  }
  PROBE(if (threadIdx.x == 0) {
    atomicMax(&prof[21], gtimer() - t_s0);
    atomicMax(&prof[22], dt[0]);
    atomicMax(&prof[23], dt[1]);
    atomicMax(&prof[24], dt[2]);
    atomicMax(&prof[29], dt[3]);
  })
  {  // write-back bytes: the CTA's sum into acc[2]; the last CTA to arrive writes the header
    unsigned long long d2h = (unsigned long long)wb0 + wb1;
    while (wbm) {  // (rare: a word with more than two dirty evicted agents)
      d2h += d.wb_bytes[base + 32 * threadIdx.x + __ffs(wbm) - 1];
      wbm &= wbm - 1;
    }
    warp_add_u44(d2h, sacc + 6);  // (sacc[6, 8) are free since P4)
    __syncthreads();
    if (threadIdx.x == 0) {  // a reduction into the header (zeroed by CTA 0 before B4): no wait
      const unsigned long long v = parts_u44(sacc + 6);
      if (v) atomicAdd(&d.header[H_D2H], v);
    }
  }
  STAMP_MAX(1)
}

// host side
bool fused_supported(const Params &p, int grid, uint32_t *tile_out) {
  if ((p.world != 1 && !p.loopback) || grid <= 0 || grid > FUSED_MAX_CTAS) return false;
  uint64_t tile = (p.n_local + grid - 1) / grid;  // grid = CTAs of the instance
  tile = (tile + 31) / 32 * 32;
  if (tile == 0) tile = 32;
  if (tile > FUSED_MAX_TILE) return false;
  *tile_out = (uint32_t)tile;
  return true;
}

// Shared-memory budget of a launch: the tile arrays and histograms (fused_smem_bytes) plus the
// CTA-count column staging of the fast list placement (as many slots as fit, <= 128).
template <int MAXB>
static size_t smem_limit() {
  static size_t lim = 0;
  if (!lim) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, k_fused_plan<MAXB>) != cudaSuccess) return 0;
    lim = (size_t)optin > a.sharedSizeBytes ? (size_t)optin - a.sharedSizeBytes : 0;
  }
  return lim;
}

template <int MAXB>
static size_t launch_smem(uint32_t tile, uint32_t gsize, uint32_t *fastok) {
  const size_t base = fused_smem_bytes(tile), lim = smem_limit<MAXB>();
  size_t sm;
  if (gsize <= 1) {  // one CTA per instance: no bucket owners
    *fastok = 1;
    sm = base;
  } else {
    // bucket-owner staging: [G][RB] counts + [4][RB] totals / offsets
    const uint32_t RB = ((4096 + gsize - 1) / gsize + 3u) & ~3u;
    const size_t need = (size_t)4 * RB * (gsize + 4);
    *fastok = base + need <= lim ? 1u : 0u;  // else the two-barrier list path
    sm = base + (*fastok ? need : 0);
  }
#ifdef AB_P1_TMA
  // P1 record staging when the whole tile fits (the kernel checks %dynamic_smem_size)
  const size_t st = p1_staging_bytes(tile);
  if (st > sm && st <= lim) sm = st;
#endif
  return sm;
}

// 1 CTA of FT threads per SM must be resident for the whole grid (grid barrier).
template <int MAXB>
static bool prepare_one(uint32_t tile, uint32_t gsize) {
  const size_t lim = smem_limit<MAXB>();
  if (!lim || cudaFuncSetAttribute(k_fused_plan<MAXB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim) !=
                  cudaSuccess)
    return false;
  uint32_t fastok;
  const size_t sm = launch_smem<MAXB>(tile, gsize, &fastok);
  if (sm > lim) return false;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused_plan<MAXB>, FT, sm) != cudaSuccess) return false;
  return per_sm >= 1;
}

bool fused_prepare(int grid, uint32_t tile, uint32_t gsize) {
  return grid >= 1 && prepare_one<1>(tile, gsize) && prepare_one<FUSED_MAX_BATCH>(tile, gsize);
}

template <int MAXB>
static void launch_t(const FusedInst *insts, uint32_t n, uint32_t gsize, cudaStream_t s, bool coop, uint32_t wsize) {
  FusedArgs<MAXB> B;
  B.n_inst = n;
  B.wsize = wsize;
  B.gsize = gsize;
  uint32_t tile = 32;
  for (uint32_t i = 0; i < n; ++i) {
    B.inst[i] = insts[i];
    tile = insts[i].tile > tile ? insts[i].tile : tile;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n * gsize);
  cfg.blockDim = dim3(FT);
  cfg.dynamicSmemBytes = launch_smem<MAXB>(tile, gsize, &B.fastok);
  cfg.stream = s;
  // cooperative: the grid barrier needs every CTA resident at once; the launch is scheduled
  // (or fails) as a whole instead of leaving resident CTAs spinning on absent ones when other
  // work holds SMs (another context's plan, copy kernels, the caller's kernels)
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 2 : 1;  // (SCALESIM_F_EXCLUSIVE: PDL only)
  cudaLaunchKernelEx(&cfg, k_fused_plan<MAXB>, B);
}

int launch_fused_batch(const FusedInst *insts, uint32_t n, uint32_t gsize, cudaStream_t s, bool coop,
                       uint32_t wsize) {
  if (n == 1) launch_t<1>(insts, n, gsize, s, coop, 1);
  else launch_t<FUSED_MAX_BATCH>(insts, n, gsize, s, coop, wsize);
  return 1;
}

}  // namespace ss
