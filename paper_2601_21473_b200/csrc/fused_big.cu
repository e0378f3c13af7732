// fused_big.cu — the single-kernel plan of LARGE integer-distance contexts: more agents per SM
// than fused.cu's shared-memory tile holds (> FUSED_MAX_TILE = 12288 per CTA, i.e. above
// ~1.8M agents on 148 SMs), up to 2^19 agents per CTA (~77M per GPU).
//
// Same method and same bucket-owner list placement as fused.cu, but the
// per-agent state between the score pass and the emit pass lives in HBM: one 16-bit code per
// agent (level-1 bucket | eligible << 12 | dirty << 13), written by P1 and read once by P34.
//   P1   stream the CTA's records: distance, eligibility, bucket; byte and count histograms and
//        the eligible non-residents' byte histogram in shared memory; codes -> HBM
//   B1   grid barrier; select D* (warp 0) while the other warps stage this CTA's bucket-owner
//        columns; the prefetched bytes below the boundary from the non-resident histogram; owner
//        pass; this CTA's list-bucket positions from the owners
//   P34  one pass without CTA barriers: each warp streams its own word range from the highest
//        id down, a thread per word (coalesced 64-byte code rows, the next step's loads in
//        flight): masks by SWAR compares on 32-bit code pairs, kept / residency words, list
//        candidates, tie agents and evicted dirty agents appended to per-warp slabs; then the
//        tie group's id-order prefix (one CTA scan over the ties) and the write-back bytes
//   (e)  per list one stable sort of the candidates by bucket (list order kept within a
//        bucket); positions from per-bucket cursors (evict: up from the bucket's first
//        position; prefetch: down from its last, so that the list stays in ascending id order)
// Limits (status SCALESIM_ST_LIMIT, the step's plan is not produced): the boundary D* falls in
// a multi-valued bucket (>= 2048 ticks), or more than BIG_OVF_CAP (4096) eligible agents have
// finite distances >= 2048 ticks (or more than 128 in one CTA).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fused_common.cuh"

namespace ss {

#ifndef BIG_LB_V
#define BIG_LB_V 4
#endif
constexpr int BIG_LB = BIG_LB_V;     // records in flight per thread in P1 (two batches)

static uint32_t big_rb(uint32_t gsize) { return ((NB1 + gsize - 1) / gsize + 3u) & ~3u; }

// Region R of shared memory: P1's non-resident byte histogram, then P34's per-thread code rows
// (1024 x 64 B), the tie staging, the placement sort's counters and arrays, the overflow sort.
constexpr uint32_t BIG_R = 64 * FT;

size_t fused_big_smem_bytes(uint32_t gsize) {
  const uint32_t RB = big_rb(gsize);
  return (size_t)4 * 4 * NB1             // histograms / counts / need list, later cursors
         + (size_t)4 * RB * (gsize + 4)  // bucket-owner staging
         + (size_t)BIG_R                 // region R
         + 64;
}

__global__ void __launch_bounds__(FT, 1) k_fused_big(const __grid_constant__ FusedArgs<1> B) {
  const uint32_t c = blockIdx.x, G = B.gsize;
  const FusedInst &I = B.inst[0];
  __shared__ __align__(16) Params sp;
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
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const Params &p = sp;
  const Dev &d = p.d;
  const int par = (int)I.parity;
  const uint32_t tile = I.tile, ep = I.epoch & 0xFFFFu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  GridBar wgrid{d.f_bar + 2 + par, 0u, G};
  if (c == 0 && threadIdx.x == 0) {
    d.f_bar[2 + (par ^ 1)] = 0u;
    unsigned long long *H = d.header;
    H[H_N_PF] = H[H_N_EV] = H[H_H2D] = H[H_D2H] = H[H_KEPT] = H[H_N_ELIG] = H[H_STATUS] = 0ull;
  }
  unsigned long long *prof = d.f_prof;
  PROBE(if (threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    atomicMin(&prof[0], t);
  })
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint32_t *h = reinterpret_cast<uint32_t *>(smem_raw);  // [4 NB1]
  const uint32_t RB = ((NB1 + G - 1) / G + 3u) & ~3u;
  uint32_t *col = h + 4 * NB1;                            // [G][RB] + [4][RB]
  // region R after the owner staging (BIG_R bytes), several lives: P1's non-resident byte
  // histogram [2 NB1]; P34's per-thread code rows; the tie staging; the (e) sort counters and
  // arrays; the overflow sort's two lists
  uint8_t *R = reinterpret_cast<uint8_t *>(col + RB * (G + 4));
  uint32_t *nrb = reinterpret_cast<uint32_t *>(R);                       // [2 NB1] (16-bit halves)
  unsigned long long *la = reinterpret_cast<unsigned long long *>(R);    // [BIG_OVF_CAP]
  unsigned long long *lb = la + BIG_OVF_CAP;                             // [BIG_OVF_CAP]
  const uint64_t base = (uint64_t)c * tile;
  const uint32_t n_here =
      base >= p.n_local ? 0u : (uint32_t)((p.n_local - base) < tile ? (p.n_local - base) : tile);
  const uint32_t tw_here = (n_here + 31) / 32;
  unsigned long long *acc = d.f_acc + 8 * par;
  const uint32_t *bm_old = d.bm[p.cur];
  uint32_t *bm_new = d.bm[p.cur ^ 1];
  uint16_t *codes = d.big_codes + base;
  const uint4 *rec = p.rec + base;

  // ---------------- P1: score, histograms, codes
  for (int b = threadIdx.x; b < 3 * NB1; b += FT) h[b] = 0u;
  for (int b = threadIdx.x; b < 2 * NB1; b += FT) nrb[b] = 0u;
  constexpr uint32_t LOVF = 128;
  __shared__ uint4 s_ovf[LOVF];
  __shared__ uint32_t s_novf;
  __shared__ uint32_t sacc[24];
  if (threadIdx.x == 0) s_novf = 0;
  if (threadIdx.x < 24) sacc[threadIdx.x] = 0;
  __syncthreads();
  {
    const float hop_scale = p.hop_scale, th0 = p.theta[0], th1 = p.theta[1], th2 = p.theta[2];
    const int64_t now = I.now;
    const bool now32 = now >= 0 && now <= 0xFFFFFFFFll;
    const uint32_t nowl = (uint32_t)now;
    uint32_t st = 0;
    uint32_t *gkeys = p.keep_dist ? d.keys + base : nullptr;
    const uint32_t last = n_here ? n_here - 1 : 0u;
    constexpr int LB = BIG_LB;
    const uint32_t BS = LB * FT, nk = tw_here * 32;
    uint4 r[LB], r2[LB];
    uint32_t bw[LB], bw2[LB];  // the residency words, loaded with the records
    // (the tile is a multiple of 32 agents: the CTA's residency words start at base / 32)
    const uint32_t *bmt = bm_old + (base >> 5);
    const uint32_t twm1 = tw_here ? tw_here - 1 : 0u;
    auto load_into = [&](uint4 (&rr)[LB], uint32_t (&ww)[LB], uint32_t k0) {
#pragma unroll
      for (int j = 0; j < LB; ++j) {
        rr[j] = ld_stream(rec + min(k0 + j * FT + threadIdx.x, last));
        ww[j] = bmt[min((k0 + j * FT) / 32 + warp, twm1)];  // (warp-uniform)
      }
    };
    // One record; compiled two ways: CHECK (a batch that runs past the tile's end: `valid`
    // masks) and FAST (32-bit now, no distance copy: the class-0 arithmetic with nothing else
    // live; warps holding other classes still take the general definition)
    auto record = [&](const uint4 rj, const uint32_t rw, const uint32_t k, auto check_tag, auto fast_tag) {
      constexpr bool CHECK = decltype(check_tag)::value, FAST = decltype(fast_tag)::value;
      const bool valid = CHECK ? k < n_here : true;
      const bool res = valid && ((rw >> lane) & 1u);
      const uint32_t ph = rj.z & 3u, cl = (rj.z >> 2) & 3u;
      float dist, th;
      if (__ballot_sync(0xFFFFFFFFu, valid && cl != 0u)) {  // interaction / diffusion / malformed
        dist = valid ? distance_of(rj, now, hop_scale, d.dint, p.n_kin, st) : 0.0f;
        th = (cl & 2u) ? ((cl & 1u) ? 0.0f : th2) : ((cl & 1u) ? th1 : th0);
      } else {
        float d_action;
        if (FAST || now32) d_action = rj.x > nowl ? __uint2float_rn(rj.x - nowl) : 0.0f;
        else {
          const int64_t remain = (int64_t)rj.x - now;
          d_action = remain <= 0 ? 0.0f : __ll2float_rn(remain);
        }
        dist = (ph == 1u || ph == 2u) ? 0.0f : (ph == 3u ? __int_as_float(0x7F800000) : d_action);
        th = th0;
      }
      const uint32_t bits = valid ? __float_as_uint(dist) : 0u;
      const bool elig = valid && (res || dist == 0.0f || dist < th);
      const uint32_t q = ibucket(bits);
      if (elig) {
        atomicAdd(&h[q], rj.y & 0xFFFFu);
        atomicAdd(&h[NB1 + q], rj.y >> 16);
        atomicAdd(&h[2 * NB1 + q], res ? 0x10000u : 1u);
        if (!res) {  // eligible non-residents: the prefetched bytes follow from the boundary
          atomicAdd(&nrb[q], rj.y & 0xFFFFu);
          atomicAdd(&nrb[NB1 + q], rj.y >> 16);
        }
        if (ib_multi(q)) {
          const uint32_t jo = atomicAdd(&s_novf, 1u);
          if (jo < LOVF) s_ovf[jo] = make_uint4(bits, (uint32_t)(p.shard_begin + base + k), res ? 1u : 0u, 0u);
        }
      }
      // the agent's code: bucket | eligible << 12 | dirty << 13; within a word lane l's code sits
      // at 2 (l % 16) + l / 16, so that 32-bit pair j of the word holds agents j and j + 16
      // (P34 decodes pairs into masks without a bit permutation)
      if (valid) {
        codes[(k & ~31u) | ((lane & 15) << 1) | (lane >> 4)] =
            (uint16_t)(q | (elig ? 1u << 12 : 0u) | (((rj.z >> 4) & 1u) << 13));
        if (!FAST && gkeys) gkeys[k] = bits;
      }
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    const bool fast = now32 && gkeys == nullptr;
    if (n_here) load_into(r, bw, 0);
#pragma unroll 1
    for (uint32_t k0 = 0; k0 < nk; k0 += BS) {
      if (k0 + BS < nk) load_into(r2, bw2, k0 + BS);
      if (fast && k0 + BS <= n_here) {  // (CTA-uniform) a whole batch inside the tile
#pragma unroll
        for (int j = 0; j < LB; ++j) record(r[j], bw[j], k0 + j * FT + threadIdx.x, F_(), T_());
      } else {
#pragma unroll
        for (int j = 0; j < LB; ++j) {
          if (k0 + j * FT >= nk) break;  // (CTA-uniform)
          record(r[j], bw[j], k0 + j * FT + threadIdx.x, T_(), F_());
        }
      }
#pragma unroll
      for (int j = 0; j < LB; ++j) {
        r[j] = r2[j];
        bw[j] = bw2[j];
      }
    }
    st = __reduce_or_sync(0xFFFFFFFFu, st);
    if (lane == 0 && st) atomicOr(reinterpret_cast<unsigned int *>(&acc[5]), st);
  }
  __syncthreads();
  STAMP_MAX(25)  // P1 loop
  publish_hist(h, NB1, d.f_hist1 + NB1 * par, nullptr, d.f_rows1 + (uint64_t)c * NB1, d.f_hist1 + 2 * NB1 + 64 * par,
               false);
  reinterpret_cast<uint4 *>(d.f_crow + ((uint64_t)par * G + c) * NB1)[threadIdx.x] =
      reinterpret_cast<const uint4 *>(h + 2 * NB1)[threadIdx.x];  // (NB1 / 4 == FT)
  {
    const uint32_t nov = s_novf;
    if (nov) {
      __shared__ unsigned long long s_ovbase;
      if (threadIdx.x == 0)
        s_ovbase = atomicAdd(&acc[6], nov <= LOVF ? (unsigned long long)nov : BIG_OVF_CAP + 1ull);
      __syncthreads();
      const unsigned long long ob = s_ovbase;
      if (threadIdx.x < nov && nov <= LOVF && ob + threadIdx.x < BIG_OVF_CAP)
        d.f_ovf[(uint64_t)par * BIG_OVF_CAP + ob + threadIdx.x] = s_ovf[threadIdx.x];
    }
  }
  if (threadIdx.x == 0) {
    const unsigned long long zb = ((unsigned long long)h[NB1] << 16) + h[0];  // bucket 0: d == 0
    if (zb) atomicAdd(&acc[0], zb);
  }
  STAMP_MAX(26)  // published
  wgrid.sync();
  STAMP_MAX(4)   // B1
  // P34's word range of each warp (its codes into L2 while the select and the owners run)
  const uint32_t WPW = (tw_here + FWARPS - 1) / FWARPS;
  const uint32_t wlo = min(tw_here, (uint32_t)warp * WPW), whi = min(tw_here, wlo + WPW);
  // (the first P34_PF steps of 32 words, 2 KB each, from the top of the range down)
  constexpr uint32_t P34_PF = 4;
  if (lane == 0 && whi > wlo) {
    const uint32_t n0 = min(whi - wlo, 32 * P34_PF);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(codes + (uint64_t)(whi - n0) * 32), "r"(n0 * 64u)
                 : "memory");
  }

  // ---------------- select, bucket owners, list-bucket positions
  {
    const int q = par ^ 1;
    const uint32_t gt = c * FT + threadIdx.x, gs = G * FT;
    for (uint32_t b = gt; b < NB1; b += gs) {
      d.f_hist1[NB1 * q + b] = 0;
      if (b < 64) d.f_hist1[2 * NB1 + 64 * q + b] = 0;
    }
    if (gt < 8) d.f_acc[8 * q + gt] = 0;
  }
  const uint32_t o_lo = min((uint32_t)NB1, c * RB), o_n = min((uint32_t)NB1, o_lo + RB) - o_lo;
  const uint32_t QP = (G + 31) / 32;
  if (warp > 0) {
    const uint32_t ch = o_n / 4;
    for (uint32_t x = threadIdx.x - 32; x < G * ch; x += FT - 32) {
      const uint32_t qq = x / ch, k = x - qq * ch;
      cp_async16(col + qq * RB + 4 * k, d.f_crow + ((uint64_t)par * G + qq) * NB1 + o_lo + 4 * k);
    }
    cp_async_commit();
  }
  __shared__ unsigned long long sh_novf;
  if (threadIdx.x == 32) sh_novf = acc[6];
  __shared__ WorldPtrs sw;
  if (threadIdx.x == 0) {
    sw.nw = 1;
    sw.rank = 0;
    sw.h1[0] = d.f_hist1;
    sw.h2[0] = d.f_hist2;
    sw.h3[0] = d.f_hist3;
    sw.m1[0] = d.f_mm1;
    sw.m2[0] = d.f_mm2;
    sw.acc[0] = d.f_acc;
    sw.hdr[0] = d.header;
  }
  __syncthreads();
  Sel sel = {0, 0, 0, 0xFFFFFFFFu, 0, 0, 1, 0};
  select_level1_warp(sw, par, p.budget, sel, true, prof);
  const bool all_fit = sel.all_fit;
  const uint32_t dstar = sel.dstar;
  const uint32_t bs = all_fit ? (uint32_t)NB1 : sel.b_res;
  const bool ok = sh_novf <= BIG_OVF_CAP && (all_fit || (sel.done && sel.level_res == 1 && !ib_multi(bs)));
  cp_async_wait_all();
  __syncthreads();
  if (!ok) {  // outside this kernel's scope: the step's plan is not produced (documented limit)
    if (c == 0 && threadIdx.x == 0) {
      unsigned long long *H = d.header;
      H[H_STATUS] = ST_LIMIT;
      H[H_SEQ] = H[H_SEQ] + 1;
    }
    return;
  }
  // this CTA's prefetched bytes below the boundary bucket (every eligible non-resident there is
  // prefetched, R2); the tie group's kept non-residents are added in P34.
  unsigned long long h2d = 0;
  for (uint32_t b = threadIdx.x; b < bs; b += FT) h2d += ((unsigned long long)nrb[NB1 + b] << 16) + nrb[b];
  __syncthreads();
  // preceding CTAs' bytes at D* (tie prefix), and this CTA's own
  __shared__ unsigned long long sh_town;
  unsigned long long t_rows = 0;
  if (!all_fit && threadIdx.x < c) t_rows = d.f_rows1[(uint64_t)threadIdx.x * NB1 + bs];
  if (!all_fit && threadIdx.x == FT - 1) sh_town = d.f_rows1[(uint64_t)c * NB1 + bs];
  if (all_fit && threadIdx.x == FT - 1) sh_town = 0;
  // bucket owner pass (as fused.cu)
  {
    uint32_t *tn = col + G * RB, *tr = tn + RB;
    for (uint32_t j = warp; j < o_n; j += FWARPS) {
      uint32_t a = 0, e = 0;
      for (uint32_t i = 0; i < QP; ++i) {
        const uint32_t q = lane * QP + i;
        if (q < G) {
          const uint32_t v = col[q * RB + j];
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
    for (uint32_t j = warp; j < o_n; j += FWARPS) {
      uint32_t w_n = 0, w_r = 0;  // the range's buckets before j (prefetch) / after j (evict)
      for (uint32_t l0 = 0; l0 < o_n; l0 += 32) {
        const uint32_t l = l0 + lane;
        w_n += __reduce_add_sync(0xFFFFFFFFu, (l < o_n && l < j) ? tn[l] : 0u);
        w_r += __reduce_add_sync(0xFFFFFFFFu, (l < o_n && l > j) ? tr[l] : 0u);
      }
      const uint32_t t_r = tr[j];
      unsigned long long *P = d.f_pos + ((uint64_t)par * NB1 + o_lo + j) * FUSED_MAX_CTAS;
      uint32_t ca = 0, ce = 0;
      for (uint32_t q0 = 0; q0 < G; q0 += 32) {
        const uint32_t q = q0 + lane;
        const uint32_t v = q < G ? col[q * RB + j] : 0u;
        const uint32_t a = v & 0xFFFFu, e = v >> 16;
        const uint32_t ia = warp_incl_scan(a), ie = warp_incl_scan(e);
        // (only the entries a consumer reads: its list buckets, and CTA 0's / the last CTA's)
        const uint32_t b = o_lo + j;
        const bool used =
#ifdef NO_OWNER_SKIP
            true;
#else
            (b < bs ? a != 0u : (b > bs ? e != 0u : v != 0u)) || q == 0 || q == G - 1;
#endif
        if (q < G && used) st_relaxed_u64(&P[q], pack_ep(ep, w_n + ca + ia - a, w_r + t_r - (ce + ie)));
        ca += __shfl_sync(0xFFFFFFFFu, ia, 31);
        ce += __shfl_sync(0xFFFFFFFFu, ie, 31);
      }
    }
  }
  warp_add_u64(t_rows, sacc + 20);
  // the buckets where this CTA has list candidates (multi-valued ones: the overflow CTA)
  uint32_t *lcnt = h + 2 * NB1, *need = h + 3 * NB1;
  __shared__ uint32_t sh_m;
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
  const uint32_t m_need = sh_m;
  STAMP_MAX(41)  // select, owner pass, need list
  const unsigned long long tie_pre = parts_u64(sacc + 20), tie_own = sh_town;
  // positions: range starts from the owners' totals, then each list bucket's offsets for this
  // CTA; prefetch cursors count down from the bucket's last position (candidates come in
  // descending id order), evict cursors up from the first
  uint32_t *h32 = h;  // [0, NB1): prefetch cursors, [NB1, 2 NB1): evict cursors
  __shared__ uint32_t sh_spf, sh_sev, sh_mvpf, sh_mvev;
  {
    uint32_t *rps = col, *rpe = col + G;
    const unsigned long long *Pc = d.f_pos + (uint64_t)par * NB1 * FUSED_MAX_CTAS + c;
    const unsigned long long pv0 =
        threadIdx.x < m_need ? ld_relaxed_u64(Pc + (uint64_t)need[threadIdx.x] * FUSED_MAX_CTAS) : 0ull;
    unsigned long long rv = 0;
    if (threadIdx.x < G) rv = poll_ep(&d.f_rt[par * FUSED_MAX_CTAS + threadIdx.x], ep, d.header);
    const uint32_t ra = (uint32_t)(rv >> 24) & 0xFFFFFFu, re = (uint32_t)rv & 0xFFFFFFu;
    unsigned long long pk[1] = {(unsigned long long)ra | ((unsigned long long)re << 32)}, tt[1];
    cta_scan1(pk, tt);
    const uint32_t r_tot = (uint32_t)(tt[0] >> 32);
    if (threadIdx.x < G) {
      rps[threadIdx.x] = (uint32_t)pk[0];
      rpe[threadIdx.x] = r_tot - (uint32_t)(pk[0] >> 32) - re;
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < m_need; j += FT) {
      const uint32_t b = need[j];
      unsigned long long v = j == threadIdx.x ? pv0 : ld_relaxed_u64(Pc + (uint64_t)b * FUSED_MAX_CTAS);
      if ((uint32_t)(v >> 48) != ep) v = poll_ep(Pc + (uint64_t)b * FUSED_MAX_CTAS, ep, d.header);
      const uint32_t nr = lcnt[b] & 0xFFFFu;
      h32[b] = rps[b / RB] + ((uint32_t)(v >> 24) & 0xFFFFFFu) + nr - 1u;  // (wraps when nr == 0: unused)
      h32[NB1 + b] = rpe[b / RB] + ((uint32_t)v & 0xFFFFFFu);
    }
    auto pos_pf = [&](uint32_t b) {
      const unsigned long long v = poll_ep(&d.f_pos[((uint64_t)par * NB1 + b) * FUSED_MAX_CTAS], ep, d.header);
      return rps[b / RB] + ((uint32_t)(v >> 24) & 0xFFFFFFu);
    };
    auto pos_ev = [&](uint32_t b) {
      const unsigned long long v = poll_ep(&d.f_pos[((uint64_t)par * NB1 + b) * FUSED_MAX_CTAS + G - 1], ep, d.header);
      return rpe[b / RB] + ((uint32_t)v & 0xFFFFFFu);
    };
    if (c == 0 && threadIdx.x == 0) {
      sh_spf = bs < (uint32_t)NB1 ? pos_pf(bs) : (uint32_t)tt[0];
      sh_sev = bs < (uint32_t)NB1 ? pos_ev(bs) : 0u;
    }
    if (c == G - 1 && threadIdx.x == 32) {
      sh_mvpf = pos_pf(IB_EXACT);
      sh_mvev = pos_ev(IB_INF - 1);
    }
    __syncthreads();
  }

  STAMP_MAX(17)  // positions
  // ---------------- P34: one pass, each warp over its own word range from the highest id down
  // (no CTA barrier inside: the warps' code loads overlap).  Two words per step: half-warp h
  // holds word hw - 1 + h, lane j of a half the 32-bit pair j of its word (agents j and j + 16,
  // P1's lane permutation); ballots assemble the word masks.  Decisions that need the other
  // warps (the tie group's id-order prefix) are deferred: tie agents, and the evicted dirty
  // agents whose write-back bytes are summed, go to per-warp lists and are resolved after the
  // pass.  List candidates (bucket << 20 | kept << 19 | k) go to per-warp slabs of the tile's
  // scratch range, each in descending id order; the placement reads them warp 31 first.
  PROBE(unsigned long long dta = 0, dtb = 0, dtc = 0, dtd = 0, tq = gtimer();)
#define LAP(v) PROBE(if (threadIdx.x == 0) { const unsigned long long t_ = gtimer(); v += t_ - tq; tq = t_; })
  unsigned long long tie_kept = 0, d2h = 0;
  uint32_t n_el = 0, n_pfb = 0, n_evb = 0;
  const unsigned long long rem = sel.rem;
  const bool cta_mv = s_novf > 0;  // this CTA holds eligible agents in multi-valued buckets
  // the words holding them (from P1's list of this CTA's such agents: at most LOVF): only those
  // words decode the multi-valued mask
  __shared__ uint32_t s_mvw[FUSED_BIG_MAX_TILE / 1024];
  if (cta_mv) {  // (CTA-uniform)
    for (uint32_t x = threadIdx.x; x < FUSED_BIG_MAX_TILE / 1024; x += FT) s_mvw[x] = 0;
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < min(s_novf, LOVF); x += FT) {
      const uint32_t k = s_ovf[x].y - (uint32_t)(p.shard_begin + base);
      atomicOr(&s_mvw[k >> 10], 1u << ((k >> 5) & 31u));
    }
    __syncthreads();
  }
  __shared__ uint32_t s_wbn[FWARPS];  // the warps' write-back list lengths
  if (lane == 0) s_wbn[warp] = 0;
  __syncwarp();
  const uint32_t slab = wlo * 32;  // this warp's slab in the tile-range scratch arrays
  uint32_t *w_pf = d.sort_ka + base + slab, *w_ev = d.sort_va + base + slab;  // candidates
  uint32_t *w_tk = d.pfa_key + base + slab, *w_tp = d.pfa_val + base + slab;  // ties: k | res, dirty; slab pos
  uint32_t *w_wb = d.f_sk3 + base + slab;                                     // evicted dirty (not ties)
  uint32_t o_pf = 0, o_ev = 0, o_t = 0, o_w = 0;  // (warp-uniform)
  {
    // thread-per-word: step s of warp w covers the 32 words [whi - 32 (s + 1), whi - 32 s), lane
    // l the word whi - 32 s - 32 + l (coalesced 64-byte rows); the lane's four 16-byte loads of
    // the next step go out before this step is decoded
    const uint4 *codes4 = reinterpret_cast<const uint4 *>(codes);
    uint8_t *const myrow = R + 64u * threadIdx.x;  // (region R is free during the pass: 1024 x 64 B)
    const uint32_t *bmt = bm_old + (base >> 5);
    const uint32_t nst = (whi - wlo + 31) / 32;
    uint4 c4[4];
    uint32_t crm = 0;
    auto load_step = [&](uint32_t t) {
      const int wd = (int)whi - 32 * ((int)t + 1) + lane;
#pragma unroll
      for (int u = 0; u < 4; ++u) c4[u] = make_uint4(0, 0, 0, 0);
      crm = 0;
      if (t < nst && wd >= (int)wlo) {
#pragma unroll
        for (int u = 0; u < 4; ++u) c4[u] = codes4[(uint32_t)wd * 4 + u];
        crm = bmt[wd];
      }
    };
    load_step(0);
    constexpr uint32_t G12 = 0x10001000u;
    const uint32_t B0 = bs * 0x10001u, B1 = (bs + 1u) * 0x10001u;  // (bs < 4096 unless all fit)
#pragma unroll 1
    for (uint32_t t = 0; t < nst; ++t) {
      const uint4 q0 = c4[0], q1 = c4[1], q2 = c4[2], q3 = c4[3];
      const uint32_t rmw = crm;
      {  // the word's codes also into the thread's 64-byte row of region R (16-byte units swizzled:
         // a quarter warp's stores hit eight distinct bank groups), read back by the candidates
        const uint32_t sz = (threadIdx.x >> 1) & 3u;
        uint4 *row4 = reinterpret_cast<uint4 *>(myrow);
        row4[0 ^ sz] = q0;
        row4[1 ^ sz] = q1;
        row4[2 ^ sz] = q2;
        row4[3 ^ sz] = q3;
      }
      load_step(t + 1);
      if (lane == 0 && t + P34_PF < nst) {  // step t + P34_PF into L2 (the range's codes do not all fit L2 at once)
        const int w1 = (int)whi - 32 * (int)(t + P34_PF), w0 = max((int)wlo, w1 - 32);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(codes + (uint64_t)w0 * 32), "r"((uint32_t)(w1 - w0) * 64u)
                     : "memory");
      }
      const int wd = (int)whi - 32 * ((int)t + 1) + lane;
      const bool on = wd >= (int)wlo;
      auto pair = [&](int jj) -> uint32_t {
        const uint4 &qq = jj < 4 ? q0 : (jj < 8 ? q1 : (jj < 12 ? q2 : q3));
        const int r = jj & 3;
        return r == 0 ? qq.x : (r == 1 ? qq.y : (r == 2 ? qq.z : qq.w));
      };
#define SWAR_SH(v, j) ((j) <= 12 ? (v) >> (12 - (j)) : (v) << ((j) - 12))
      uint32_t em = 0, lm = 0, tm = 0, mv = 0;
      if (all_fit) {
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) em |= SWAR_SH(pair(jj) & G12, jj);
        lm = em;
      } else {
        uint32_t ge0 = 0, ge1 = 0;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const uint32_t W = pair(jj), X = (W & 0x0FFF0FFFu) | G12;
          em |= SWAR_SH(W & G12, jj);
          ge0 |= SWAR_SH((X - B0) & G12, jj);
          ge1 |= SWAR_SH((X - B1) & G12, jj);
        }
        lm = em & ~ge0;
        tm = em & ge0 & ~ge1;
      }
      if (cta_mv && on && ((s_mvw[(uint32_t)wd >> 5] >> (wd & 31)) & 1u)) {  // (rare: a word with such agents)
        uint32_t m0 = 0, m1 = 0;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const uint32_t X = (pair(jj) & 0x0FFF0FFFu) | G12;
          m0 |= SWAR_SH((X - (uint32_t)IB_EXACT * 0x10001u) & G12, jj);
          m1 |= SWAR_SH((X - (uint32_t)IB_INF * 0x10001u) & G12, jj);
        }
        mv = em & m0 & ~m1;
      }
#undef SWAR_SH
      if (!on) em = lm = tm = mv = 0;
      const uint32_t rm = on ? rmw : 0u;
      const uint32_t pm = em & ~rm & ~mv & (lm | tm), ec = rm & ~lm & ~mv;
      const uint32_t evk = rm & ~lm & ~tm;  // evicted whatever the cut (write-back bytes if dirty)
      if (on) {
        bm_new[(base >> 5) + wd] = lm;  // (kept ties OR'ed in after the pass)
        n_el += __popc(em);
      }
      // list offsets of this step in descending id order: the higher lanes first
      const uint32_t npm = __popc(pm), nec = __popc(ec), ntm = __popc(tm), nwb = 0;
      const unsigned long long c01 = (unsigned long long)npm | ((unsigned long long)nec << 32);
      const unsigned long long c23 = (unsigned long long)ntm | ((unsigned long long)nwb << 32);
      unsigned long long i01 = c01, i23 = c23;  // inclusive suffix sums (lanes >= l)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long x01 = __shfl_down_sync(0xFFFFFFFFu, i01, o);
        const unsigned long long x23 = __shfl_down_sync(0xFFFFFFFFu, i23, o);
        if (lane + o < 32) {
          i01 += x01;
          i23 += x23;
        }
      }
      const unsigned long long t01 = __shfl_sync(0xFFFFFFFFu, i01, 0), t23 = __shfl_sync(0xFFFFFFFFu, i23, 0);
      uint32_t bpf = o_pf + (uint32_t)(i01 - c01), bev = o_ev + (uint32_t)((i01 - c01) >> 32);
      uint32_t bt = o_t + (uint32_t)(i23 - c23);
      o_pf += (uint32_t)t01;
      o_ev += (uint32_t)(t01 >> 32);
      o_t += (uint32_t)t23;
      const uint32_t kb = (uint32_t)wd * 32 - slab;  // (slab-relative id of the word's agent 0)
      // the word's candidates, ties and write-backs, from its highest agent down; a code's place
      // in the word: agent a sits in pair a % 16, half a / 16
      for (uint32_t m = pm | ec | tm | evk; m; ) {
        const uint32_t a = 31 - __clz(m);
        m &= ~(1u << a);
        // (the code from the thread's shared-memory row: pair a % 16 in unit (a % 16) / 4, swizzled)
        const uint32_t jj = a & 15u, un = (jj >> 2) ^ ((threadIdx.x >> 1) & 3u);
        const uint32_t code = *reinterpret_cast<const uint16_t *>(myrow + un * 16 + (jj & 3u) * 4 + (a >> 4) * 2);
        const uint32_t q = code & 0xFFFu, dirty = (code >> 13) & 1u, bit = 1u << a;
        uint32_t cpos = 0xFFFFFFFFu;
        if (pm & bit) {
          w_pf[bpf] = (q << 20) | (((lm >> a) & 1u) << 19) | (kb + a);
          cpos = bpf++;
        } else if (ec & bit) {
          w_ev[bev] = (q << 20) | (kb + a);
          cpos = (bev++) | 0x80000000u;
        }
        if (tm & bit) {
          w_tk[bt] = (kb + a + slab) | (((rm >> a) & 1u) << 31) | (dirty << 30);
          w_tp[bt++] = cpos;
        }
        if ((evk & bit) && dirty) w_wb[atomicAdd(&s_wbn[warp], 1u)] = kb + a + slab;  // (order irrelevant: a sum)
      }
    }
  }
  __syncwarp();
  o_w = s_wbn[warp];
  // write-back bytes of the warp's other evicted dirty agents (R13): its list, 32 loads at a time
  for (uint32_t i0 = 0; i0 < o_w; i0 += 128) {  // (four independent loads in flight per lane)
    uint32_t ix[4], v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ix[u] = i0 + 32u * u + lane < o_w ? w_wb[i0 + 32u * u + lane] : 0xFFFFFFFFu;
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ix[u] != 0xFFFFFFFFu ? d.wb_bytes[base + ix[u]] : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) d2h += v[u];
  }
  LAP(dta)
  // the warps' list lengths: candidates / ties / write-backs
  __shared__ uint32_t s_cnt[4][FWARPS], s_pre[4][FWARPS + 1];
  if (lane == 0) {
    s_cnt[0][warp] = o_pf;
    s_cnt[1][warp] = o_ev;
    s_cnt[2][warp] = o_t;
    s_cnt[3][warp] = o_w;
  }
  __syncthreads();
  if (warp < 4) {  // [0], [1]: warp 31 first (list order); [2], [3]: warp 0 first (ascending id)
    const uint32_t src = warp < 2 ? (uint32_t)(FWARPS - 1 - lane) : (uint32_t)lane;
    const uint32_t c = s_cnt[warp][src], inc = warp_incl_scan(c);
    s_pre[warp][lane] = inc - c;
    if (lane == 31) s_pre[warp][FWARPS] = inc;
  }
  __syncthreads();
  // ties in ascending id order (warp w's list reversed, after the lower warps'); their bytes'
  // inclusive prefix decides each one (kept iff tie_pre + prefix <= rem, P:241 R3).  Each warp
  // stages its ties (entry, candidate place, bytes) at their ascending positions in shared
  // memory (region R, free now), TCAP at a time
  {
    const uint32_t nt = s_pre[2][FWARPS];
    constexpr uint32_t TCAP = 4096;  // ties per round (3 x 16 KB of R)
    uint32_t *t_e = reinterpret_cast<uint32_t *>(R), *t_c = t_e + TCAP, *t_f = t_c + TCAP;
    __shared__ unsigned long long s_tot;
    unsigned long long carry = 0;
    const uint32_t my_n = s_cnt[2][warp], my_pre = s_pre[2][warp];
    for (uint32_t g0 = 0; g0 < nt; g0 += TCAP) {  // (CTA-uniform)
      for (uint32_t i = lane; i < my_n; i += 32) {
        const uint32_t g = my_pre + (my_n - 1 - i);
        if (g < g0 || g >= g0 + TCAP) continue;
        const uint32_t e = w_tk[i], cp = w_tp[i];
        t_e[g - g0] = e;
        t_c[g - g0] = cp == 0xFFFFFFFFu ? cp : (cp & 0x80000000u) | (slab + (cp & 0x7FFFFFFFu));  // (tile-relative)
        t_f[g - g0] = rec[e & 0x7FFFFu].y;
      }
      __syncthreads();
      const uint32_t nr = min(TCAP, nt - g0);
      for (uint32_t x0 = 0; x0 < nr; x0 += FT) {  // (CTA-uniform)
        const uint32_t x = x0 + threadIdx.x;
        const uint32_t fp = x < nr ? t_f[x] : 0u;
        const unsigned long long ex = block_excl_scan<unsigned long long, FT>((unsigned long long)fp, &s_tot);
        if (x < nr) {
          const bool kept = tie_pre + carry + ex + fp <= rem;
          const uint32_t e = t_e[x], cp = t_c[x], k = e & 0x7FFFFu;
          const bool res = (e >> 31) & 1u, dirty = (e >> 30) & 1u;
          if (kept) {
            atomicOr(&bm_new[(base >> 5) + (k >> 5)], 1u << (k & 31));
            if (cp != 0xFFFFFFFFu) atomicOr((cp >> 31) ? &d.sort_va[base + (cp & 0x7FFFFFFFu)] : &d.sort_ka[base + cp], 1u << 19);
            tie_kept += fp;
            if (!res) {
              h2d += fp;
              ++n_pfb;
            }
          } else if (res) {
            ++n_evb;
            if (dirty) d2h += d.wb_bytes[base + k];
          }
        }
        carry += s_tot;
      }
      __syncthreads();
    }
  }
  LAP(dtb)
  __syncthreads();  // (the tie patches of the candidate entries are visible to the placement)
  // (e) placement: per list, a stable sort of the candidates by bucket (list order kept within a
  // bucket); a candidate's rank in its bucket = sorted index - the bucket's first index; evict
  // positions count up from the bucket's cursor, prefetch positions down from its last one
  // (only kept candidates are members).  The sort runs in shared memory (region R: counters +
  // four arrays) when the list fits, else on HBM scratch.
  const uint32_t *cur_pf = h32, *cur_ev = h32 + NB1;
  auto place = [&](uint32_t x, uint32_t pos, bool pf) {  // x: a member's candidate entry
    if (pos >= p.n_local) {  // (cannot happen: flagged instead of writing out of bounds)
      atomicOr(reinterpret_cast<unsigned int *>(&d.header[H_STATUS]), ST_SYNC);
      return;
    }
    (pf ? d.pf_ids : d.ev_ids)[pos] = (uint32_t)(p.shard_begin + base + (x & 0x7FFFFu));
  };
  {
    constexpr uint32_t SMAX = (BIG_R / 4 - SB_CNT) / 2;  // entries sortable in R
    uint32_t *start = h + 2 * NB1;  // [NB1] first sorted index per bucket (the counts are no longer needed)
    uint32_t *cnt = reinterpret_cast<uint32_t *>(R);  // SB_CNT sort counters
    for (int lst = 0; lst < 2; ++lst) {
      const uint32_t n = s_pre[lst][FWARPS];
      if (n == 0) continue;  // (CTA-uniform)
      const uint32_t *src = lst == 0 ? d.sort_ka + base : d.sort_va + base;
      uint32_t *xa, *xb;  // the entries (bucket << 20 | kept << 19 | k), sorted by bucket
      if (n <= SMAX) {
        xa = cnt + SB_CNT;
        xb = xa + SMAX;
      } else {
        xa = d.sort_kb + base;
        xb = d.sort_vb + base;
      }
      {  // the slabs, warp 31's first: each warp copies its own
        const uint32_t mine = s_cnt[lst][warp], at = s_pre[lst][FWARPS - 1 - warp];
        for (uint32_t i = lane; i < mine; i += 32) {
          const uint32_t x0 = src[slab + i];
          xa[at + i] = (x0 & 0xFFF80000u) | (slab + (x0 & 0x7FFFFu));  // (tile-relative k)
        }
      }
      __syncthreads();
      PROBE(const unsigned long long ts0 = gtimer();)
      cta_sort_buckets(xa, xb, n, cnt);
      PROBE(if (threadIdx.x == 0) {
        atomicMax(&prof[50 + lst], gtimer() - ts0);
        atomicMax(&prof[52 + lst], (unsigned long long)n);
      })
      for (uint32_t i = threadIdx.x; i < n; i += FT)
        if (i == 0 || (xa[i - 1] >> 20) != (xa[i] >> 20)) start[xa[i] >> 20] = i;
      __syncthreads();
      const uint32_t *cur = lst == 0 ? cur_pf : cur_ev;
      for (uint32_t i = threadIdx.x; i < n; i += FT) {
        const uint32_t x = xa[i], b = x >> 20, rk = i - start[b];
        // members: kept prefetch candidates, evict candidates the cut does not keep
        if (((x >> 19) & 1u) == (lst == 0 ? 1u : 0u)) place(x, lst == 0 ? cur[b] - rk : cur[b] + rk, lst == 0);
      }
      __syncthreads();
    }
  }
  LAP(dtc)
  PROBE(if (threadIdx.x == 0) {
    atomicMax(&prof[22], dta);
    atomicMax(&prof[23], dtb);
    atomicMax(&prof[24], dtc);
    atomicMax(&prof[29], dtd);
  })
  STAMP_MAX(39)  // P34 done
  // the agents in multi-valued buckets (all CTAs'): one CTA sorts them -- prefetch members
  // (non-residents below b*) ascending by (key, id) after the value buckets below 2048, evict
  // members (residents above b*) descending after the +inf bucket (bitonic sorts of packed
  // (key, id) in shared memory; the chunk arrays are free now)
  if (c == G - 1 && sh_novf > 0) {
    const uint32_t nov = (uint32_t)sh_novf;
    __shared__ uint32_t sh_na, sh_nb;
    if (threadIdx.x == 0) sh_na = sh_nb = 0;
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < nov; x += FT) {
      const uint4 q = d.f_ovf[(uint64_t)par * BIG_OVF_CAP + x];
      const uint32_t b = ibucket(q.x);
      if (!q.z && b < bs) la[atomicAdd(&sh_na, 1u)] = ((unsigned long long)q.x << 32) | q.y;
      else if (q.z && b > bs) lb[atomicAdd(&sh_nb, 1u)] = ~(((unsigned long long)q.x << 32) | q.y);
    }
    __syncthreads();
    const uint32_t na = sh_na, nb = sh_nb;
    for (int lst = 0; lst < 2; ++lst) {
      unsigned long long *v = lst == 0 ? la : lb;
      const uint32_t m = lst == 0 ? na : nb;
      if (m == 0) continue;
      uint32_t N = 1;
      while (N < m) N <<= 1;
      for (uint32_t x = m + threadIdx.x; x < N; x += FT) v[x] = ~0ull;
      __syncthreads();
      for (uint32_t k = 2; k <= N; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          for (uint32_t i = threadIdx.x; i < N; i += FT) {
            const uint32_t ij = i ^ j;
            if (ij > i) {
              const unsigned long long a = v[i], bb = v[ij];
              if ((a > bb) == ((i & k) == 0)) {
                v[i] = bb;
                v[ij] = a;
              }
            }
          }
          __syncthreads();
        }
      uint32_t *out = lst == 0 ? d.pf_ids + sh_mvpf : d.ev_ids + sh_mvev;
      for (uint32_t x = threadIdx.x; x < m; x += FT) out[x] = (uint32_t)(lst == 0 ? v[x] : ~v[x]);
      __syncthreads();
    }
  }
  // sums into the header (zeroed before B1)
  warp_add_u44(h2d, sacc + 4);
  warp_add_u44(tie_kept, sacc + 8);
  warp_add_u44(d2h, sacc + 6);
  n_el = __reduce_add_sync(0xFFFFFFFFu, n_el);  // (every thread counted its words)

  n_pfb = __reduce_add_sync(0xFFFFFFFFu, n_pfb);
  n_evb = __reduce_add_sync(0xFFFFFFFFu, n_evb);
  if (lane == 0) {
    if (n_el) atomicAdd(&sacc[10], n_el);
    if (n_pfb) atomicAdd(&sacc[11], n_pfb);
    if (n_evb) atomicAdd(&sacc[12], n_evb);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long *H = d.header;
    const unsigned long long v_h2d = parts_u44(sacc + 4), v_tie = parts_u44(sacc + 8), v_wb = parts_u44(sacc + 6);
    if (v_h2d) atomicAdd(&H[H_H2D], v_h2d);
    if (v_tie) atomicAdd(&H[H_KEPT], v_tie);
    if (v_wb) atomicAdd(&H[H_D2H], v_wb);
    if (sacc[10]) atomicAdd(&H[H_N_ELIG], (unsigned long long)sacc[10]);
    if (sacc[11]) atomicAdd(&H[H_N_PF], (unsigned long long)sacc[11]);
    if (sacc[12]) atomicAdd(&H[H_N_EV], (unsigned long long)sacc[12]);
    if (c == 0) {
      if (sh_spf) atomicAdd(&H[H_N_PF], (unsigned long long)sh_spf);
      if (sh_sev) atomicAdd(&H[H_N_EV], (unsigned long long)sh_sev);
      atomicAdd(&H[H_KEPT], p.budget - rem);
      uint32_t status = (uint32_t)acc[5] | d.state->status;
      if (acc[0] > p.budget) status |= ST_INSUFFICIENT;
      H[H_CUT_BITS] = all_fit ? 0xFFFFFFFFull : dstar;
      H[H_CUT_REM] = rem;
      atomicOr(reinterpret_cast<unsigned int *>(&H[H_STATUS]), status);
      H[H_SEQ] = H[H_SEQ] + 1;
    }
    PROBE(atomicMax(&prof[1], gtimer());)
  }
}

bool fused_big_prepare(uint32_t gsize) {
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return false;
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, k_fused_big) != cudaSuccess) return false;
  const size_t sm = fused_big_smem_bytes(gsize);
  if (sm + a.sharedSizeBytes > (size_t)optin) return false;
  if (cudaFuncSetAttribute(k_fused_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
    return false;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused_big, FT, sm) != cudaSuccess) return false;
  return per_sm >= 1;
}

int launch_fused_big(const FusedInst &inst, uint32_t gsize, cudaStream_t s, bool coop) {
  FusedArgs<1> B;
  B.n_inst = 1;
  B.gsize = gsize;
  B.fastok = 1;
  B.wsize = 1;
  B.inst[0] = inst;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(gsize);
  cfg.blockDim = dim3(FT);
  cfg.dynamicSmemBytes = fused_big_smem_bytes(gsize);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 2 : 1;
  cudaLaunchKernelEx(&cfg, k_fused_big, B);
  return 1;
}

}  // namespace ss
