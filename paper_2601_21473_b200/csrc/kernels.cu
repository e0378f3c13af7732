// kernels.cu — sm_100a kernels of the ScaleSim planner (multi-kernel path, v1).
//
// Step = score (a1, a1', a2) -> radix select of the boundary distance (a3) -> id-order tie
// scan and emit (a4, a5) -> list compaction + stable radix sort by distance (a5) -> block
// expansion / page assignment (a5) -> page copies pinned host <-> HBM (a6).
// See DESIGN.md §7 for the kernel list, the data layout and the roofline of each kernel.
//
// Floating point: the distance arithmetic uses explicit round-to-nearest intrinsics so
// that nvcc cannot contract into FMA; the same op sequence as PAPER Eq. 2 reading R7.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace ss {

// ------------------------------------------------------------------------------------
// plan init: clear per-plan accumulators

__global__ void k_plan_init(Params p) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < 2048) {
    p.d.hist1[t] = 0;
    p.d.mm1[t] = 0xFFFFFFFFu;
    p.d.mm1[2048 + t] = 0xFFFFFFFFu;
  }
  if (t < 1024) {
    p.d.hist2[t] = 0;
    p.d.hist3[t] = 0;
    p.d.mm2[t] = 0xFFFFFFFFu;
    p.d.mm2[1024 + t] = 0xFFFFFFFFu;
  }
  if (t == 0) {
    SelState z = {};
    z.level = 1;
    z.sort_and[0] = z.sort_and[1] = 0xFFFFFFFFu;
    *p.d.state = z;
    p.d.hist1[2048] = 0;  // zero-distance bytes slot (exchanged with the histogram)
  }
  // the header is not cleared: every field is rewritten by the plan that owns it
}

// ------------------------------------------------------------------------------------
// a1': interaction participants (ACTING INT agents with finite kinematics) and pair-min

__global__ void __launch_bounds__(NT) k_int_compact(Params p, int64_t now) {
  uint32_t st = 0;
  // bounding box and largest speed of the participants, for the a1' grid (interaction.cu)
  int32_t bx0 = 0x7FFFFFFF, by0 = 0x7FFFFFFF, bx1 = (int32_t)0x80000000, by1 = (int32_t)0x80000000;
  uint32_t bvm = 0;
  for (uint64_t k = blockIdx.x * (uint64_t)NT + threadIdx.x; k < p.n_kin; k += (uint64_t)gridDim.x * NT)
    p.d.dint[k] = __int_as_float(0x7F800000);
  for (uint64_t base = blockIdx.x * (uint64_t)NT; base < p.n_local; base += (uint64_t)gridDim.x * NT) {
    const uint64_t i = base + threadIdx.x;
    bool part = false;
    float4 kv = make_float4(0, 0, 0, 0);
    uint32_t ki = 0;
    float dact = 0.0f;
    if (i < p.n_local) {
      const uint4 r = ld_stream(p.rec + i);
      const int64_t remain = (int64_t)r.x - now;  // D_action, as in distance_of
      dact = remain <= 0 ? 0.0f : __ll2float_rn(remain);
      if (phase_of(r) == 0u && class_of(r) == 1u) {
        if (r.w >= p.n_kin) {
          st |= ST_BAD_RECORD;
        } else {
          kv = p.kin[r.w];
          ki = r.w;
          if (isfinite(kv.x) && isfinite(kv.y) && isfinite(kv.z) && isfinite(kv.w)) part = true;
          else st |= ST_BAD_KIN;
        }
      }
    }
    const uint32_t m = __ballot_sync(FULL, part);
    if (m) {
      const int lane = threadIdx.x & 31;
      uint32_t base_slot = 0;
      if (lane == __ffs(m) - 1) base_slot = atomicAdd(&p.d.state->int_count, __popc(m));
      base_slot = __shfl_sync(FULL, base_slot, __ffs(m) - 1);
      if (part) {
        const uint32_t slot = base_slot + __popc(m & lanemask_lt());
        p.d.ilist_kin[slot] = kv;
        p.d.ilist_idx[slot] = ki;
        p.d.ilist_dact[slot] = dact;
        bx0 = min(bx0, fkey(kv.x));
        by0 = min(by0, fkey(kv.y));
        bx1 = max(bx1, fkey(kv.x));
        by1 = max(by1, fkey(kv.y));
        bvm = max(bvm, __float_as_uint(sqrtf(kv.z * kv.z + kv.w * kv.w)));
      }
    }
  }
  st = __reduce_or_sync(FULL, st);
  if ((threadIdx.x & 31) == 0 && st) atomicOr(&p.d.state->status, st);
  if (p.n_kin >= GRID_MIN_PARTICIPANTS) {
    __shared__ int32_t sb[4];
    __shared__ uint32_t svm;
    if (threadIdx.x == 0) {
      sb[0] = sb[1] = 0x7FFFFFFF;
      sb[2] = sb[3] = (int32_t)0x80000000;
      svm = 0;
    }
    __syncthreads();
    bx0 = __reduce_min_sync(FULL, bx0);
    by0 = __reduce_min_sync(FULL, by0);
    bx1 = __reduce_max_sync(FULL, bx1);
    by1 = __reduce_max_sync(FULL, by1);
    bvm = __reduce_max_sync(FULL, bvm);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&sb[0], bx0);
      atomicMin(&sb[1], by0);
      atomicMax(&sb[2], bx1);
      atomicMax(&sb[3], by1);
      atomicMax(&svm, bvm);
    }
    __syncthreads();
    if (threadIdx.x == 0 && sb[0] != 0x7FFFFFFF) {
      GridHdr *g = reinterpret_cast<GridHdr *>(p.d.grid_hdr);
      atomicMin(&g->acc_x0, sb[0]);
      atomicMin(&g->acc_y0, sb[1]);
      atomicMax(&g->acc_x1, sb[2]);
      atomicMax(&g->acc_y1, sb[3]);
      atomicMax(&g->acc_vmax, svm);
    }
  }
}

// Eq. 2, reading R6/R7: t_ij = (r.r) / (-(r.w)), r = p_j - p_i, w = v_j - v_i,
// only for approaching pairs (r.w < 0).  min_j over other participants.  The division is
// skipped only when it provably cannot lower the running minimum (g2 > RU(best * den)
// implies fl(g2/den) >= best), so the result is the exact min of the rounded quotients.
__global__ void __launch_bounds__(NT) k_pairmin(Params p) {
  __shared__ float4 tile[NT];
  const uint32_t count = p.d.state->int_count;
  const uint32_t i = blockIdx.x * NT + threadIdx.x;
  if (blockIdx.x * NT >= count) return;
  const bool mine = i < count;
  const float4 ki = mine ? p.d.ilist_kin[i] : make_float4(0, 0, 0, 0);
  float best = __int_as_float(0x7F800000);
  for (uint32_t j0 = 0; j0 < count; j0 += NT) {
    __syncthreads();
    if (j0 + threadIdx.x < count) tile[threadIdx.x] = p.d.ilist_kin[j0 + threadIdx.x];
    __syncthreads();
    const uint32_t jn = min((uint32_t)NT, count - j0);
    if (mine) {
      for (uint32_t jj = 0; jj < jn; ++jj) {
        const float4 kj = tile[jj];
        const float dx = __fsub_rn(kj.x, ki.x);
        const float dy = __fsub_rn(kj.y, ki.y);
        const float dvx = __fsub_rn(kj.z, ki.z);
        const float dvy = __fsub_rn(kj.w, ki.w);
        const float rw = __fadd_rn(__fmul_rn(dx, dvx), __fmul_rn(dy, dvy));
        if (rw < 0.0f && (j0 + jj) != i) {
          const float g2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
          const float den = -rw;
          if (!(g2 > __fmul_ru(best, den))) {
            const float t = __fdiv_rn(g2, den);
            if (t < best) best = t;
          }
        }
      }
    }
  }
  if (mine) p.d.dint[p.d.ilist_idx[i]] = best;
}

// ------------------------------------------------------------------------------------
// a1 + a2: score, key, eligibility, byte-weighted level-1 histogram with per-bucket min/max

__global__ void __launch_bounds__(NT) k_score(Params p, int64_t now) {
  // byte-weighted level-1 histogram in shared memory as 16-bit halves (native 32-bit
  // shared atomics, exact), with per-bucket min key and min complemented key
  __shared__ uint32_t sh_lo[2048], sh_hi[2048], sh_min[2048], sh_nmax[2048];
  for (int b = threadIdx.x; b < 2048; b += NT) {
    sh_lo[b] = 0;
    sh_hi[b] = 0;
    sh_min[b] = 0xFFFFFFFFu;
    sh_nmax[b] = 0xFFFFFFFFu;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t st = 0;
  unsigned long long zero_bytes = 0;
  const uint32_t *bm_old = p.d.bm[p.cur];
  for (uint64_t base = blockIdx.x * (uint64_t)NT; base < p.n_local; base += (uint64_t)gridDim.x * NT) {
    const uint64_t i = base + threadIdx.x;
    const bool valid = i < p.n_local;
    uint4 r = make_uint4(0, 0, 0, 0);
    uint32_t word = 0;
    if (valid) {
      r = ld_stream(p.rec + i);
      word = bm_old[i >> 5];
    }
    const bool res = valid && ((word >> (i & 31)) & 1u);
    const float d = !valid ? 0.0f
                    : (p.explicit_dist ? explicit_distance_of(r, st)
                                       : distance_of(r, now, p.hop_scale, p.d.dint, p.n_kin, st));
    const uint32_t bits = __float_as_uint(d);
    const bool elig = valid && (res || d == 0.0f || d < (p.explicit_dist ? p.theta[0] : theta_of(p, class_of(r))));
    if (valid) p.d.keys[i] = bits;
    const uint32_t eb = __ballot_sync(FULL, elig);
    if (lane == 0 && (i >> 5) < p.n_words) p.d.elig[i >> 5] = eb;
    if (valid && d == 0.0f) zero_bytes += r.y;
    if (elig) {
      const uint32_t b = bits >> 20;
      atomicAdd(&sh_lo[b], r.y & 0xFFFFu);
      atomicAdd(&sh_hi[b], r.y >> 16);
      atomicMin(&sh_min[b], bits);
      atomicMin(&sh_nmax[b], ~bits);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 2048; b += NT) {
    const unsigned long long v = ((unsigned long long)sh_hi[b] << 16) + sh_lo[b];
    if (v != 0 || sh_min[b] != 0xFFFFFFFFu) {
      atomicAdd(&p.d.hist1[b], v);
      atomicMin(&p.d.mm1[b], sh_min[b]);
      atomicMin(&p.d.mm1[2048 + b], sh_nmax[b]);
    }
  }
  const unsigned long long zb = block_sum(zero_bytes);
  if (threadIdx.x == 0 && zb) atomicAdd(&p.d.hist1[2048], zb);
  st = __reduce_or_sync(FULL, st);
  if (lane == 0 && st) atomicOr(&p.d.state->status, st);
}

__global__ void k_copy_keys(Params p, float *out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.n_local; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = __uint_as_float(p.d.keys[i]);
}

// ------------------------------------------------------------------------------------
// a3: select.  One block of NT threads scans the 2^w buckets of the current level and finds
// the first bucket b with below + cum(<=b) > B (the boundary of the budget).

__global__ void __launch_bounds__(NT) k_select(Params p, int level) {
  SelState *S = p.d.state;
  if (S->done) return;
  const int w = level == 1 ? L1_BITS : (level == 2 ? L2_BITS : L3_BITS);
  const int shift = level == 1 ? 20 : (level == 2 ? 10 : 0);
  const uint32_t nb = 1u << w;
  const unsigned long long *h = level == 1 ? p.d.hist1 : (level == 2 ? p.d.hist2 : p.d.hist3);
  const uint32_t *mm = level == 1 ? p.d.mm1 : (level == 2 ? p.d.mm2 : nullptr);
  const unsigned long long below = S->below;
  __shared__ unsigned long long sh_total, sh_prev;
  __shared__ uint32_t sh_first;
  if (threadIdx.x == 0) sh_first = 0xFFFFFFFFu;
  __syncthreads();
  // each thread owns nb/NT consecutive buckets
  const uint32_t per = nb / NT;
  unsigned long long loc = 0;
  for (uint32_t k = 0; k < per; ++k) loc += h[threadIdx.x * per + k];
  unsigned long long tot;
  const unsigned long long ex = block_excl_scan(loc, &sh_total);
  tot = sh_total;
  unsigned long long run = below + ex;
  for (uint32_t k = 0; k < per; ++k) {
    const uint32_t b = threadIdx.x * per + k;
    const unsigned long long prev = run;
    run += h[b];
    if (run > p.budget && prev <= p.budget) {  // exactly one bucket crosses (sums are monotone)
      sh_first = b;
      sh_prev = prev;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (level == 1) {
      S->total = tot;
      if (p.d.hist1[2048] > p.budget) S->status |= ST_INSUFFICIENT;
      S->zero_bytes = p.d.hist1[2048];
    }
    const uint32_t b = sh_first;
    if (b == 0xFFFFFFFFu) {
      // level 1 only: everything eligible fits
      S->all_fit = 1;
      S->done = 1;
      S->dstar = 0xFFFFFFFFu;
      S->rem = p.budget - (below + tot);
      S->level = 4;
    } else {
      const unsigned long long cum_before = sh_prev;
      S->below = cum_before;
      S->prefix |= b << shift;
      const bool single = mm != nullptr && mm[b] == ~mm[nb + b];
      if (level == 3 || single) {
        S->dstar = (level == 3) ? S->prefix : mm[b];
        S->rem = p.budget - cum_before;
        S->done = 1;
        S->level = 4;
      } else {
        S->level = level + 1;
      }
    }
  }
}

// Histogram of the next digit over the keys inside the boundary bucket (levels 2 and 3).
__global__ void __launch_bounds__(NT) k_hist(Params p, int level) {
  const SelState *S = p.d.state;
  if (S->done || S->level != (unsigned)level) return;
  __shared__ uint32_t sh_lo[1024], sh_hi[1024], sh_min[1024], sh_nmax[1024];
  for (int b = threadIdx.x; b < 1024; b += NT) {
    sh_lo[b] = 0;
    sh_hi[b] = 0;
    sh_min[b] = 0xFFFFFFFFu;
    sh_nmax[b] = 0xFFFFFFFFu;
  }
  __syncthreads();
  const int hi_shift = level == 2 ? 20 : 10;
  const int shift = level == 2 ? 10 : 0;
  const uint32_t want = S->prefix >> hi_shift;
  for (uint64_t i = blockIdx.x * (uint64_t)NT + threadIdx.x; i < p.n_local; i += (uint64_t)gridDim.x * NT) {
    const bool el = (p.d.elig[i >> 5] >> (i & 31)) & 1u;
    const uint32_t bits = p.d.keys[i];
    if (el && (bits >> hi_shift) == want) {
      const uint32_t fp = p.rec[i].y;
      const uint32_t b = (bits >> shift) & 1023u;
      atomicAdd(&sh_lo[b], fp & 0xFFFFu);
      atomicAdd(&sh_hi[b], fp >> 16);
      atomicMin(&sh_min[b], bits);
      atomicMin(&sh_nmax[b], ~bits);
    }
  }
  __syncthreads();
  unsigned long long *gh = level == 2 ? p.d.hist2 : p.d.hist3;
  for (int b = threadIdx.x; b < 1024; b += NT) {
    const unsigned long long v = ((unsigned long long)sh_hi[b] << 16) + sh_lo[b];
    if (v != 0 || sh_min[b] != 0xFFFFFFFFu) {
      atomicAdd(&gh[b], v);
      if (level == 2) {
        atomicMin(&p.d.mm2[b], sh_min[b]);
        atomicMin(&p.d.mm2[1024 + b], sh_nmax[b]);
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// a4: tie group (d == D*) bytes per tile, in id order, then the exclusive scan over tiles

__global__ void __launch_bounds__(NT) k_tie_partial(Params p) {
  const SelState *S = p.d.state;
  const uint64_t t0 = (uint64_t)blockIdx.x * TILE;
  unsigned long long s = 0;
  if (!S->all_fit) {
    const uint32_t dstar = S->dstar;
    for (uint32_t k = threadIdx.x; k < TILE; k += NT) {
      const uint64_t i = t0 + k;
      if (i < p.n_local && ((p.d.elig[i >> 5] >> (i & 31)) & 1u) && p.d.keys[i] == dstar) s += p.rec[i].y;
    }
  }
  s = block_sum(s);
  if (threadIdx.x == 0) p.d.tile_tie[blockIdx.x] = s;
}

// single block: exclusive scan of u64/u32 arrays of length n (NT threads, chunked)
template <typename T>
__device__ void block_scan_array(const T *in, T *out, uint64_t n, T *total_out) {
  __shared__ T sh_tot;
  T carry = 0;
  for (uint64_t base = 0; base < n; base += NT) {
    const uint64_t i = base + threadIdx.x;
    const T v = i < n ? in[i] : T(0);
    const T ex = block_excl_scan(v, &sh_tot);
    __syncthreads();
    const T tot = sh_tot;
    if (i < n) out[i] = carry + ex;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}

__global__ void __launch_bounds__(NT) k_tie_scan(Params p) {
  __shared__ unsigned long long tot;
  block_scan_array<unsigned long long>(p.d.tile_tie, p.d.tile_tie_excl, p.n_tiles, &tot);
  __syncthreads();
  if (threadIdx.x == 0) {
    p.d.state->tie_local = tot;
    if (p.world == 1) p.d.gather[0] = tot;
  }
}

// a4 + a5: kept decision, new residency bitmap, per-tile change counts.
__global__ void __launch_bounds__(NT) k_emit(Params p) {
  const SelState *S = p.d.state;
  const uint64_t t0 = (uint64_t)blockIdx.x * TILE;
  const bool all_fit = S->all_fit;
  const uint32_t dstar = S->dstar;
  const unsigned long long rem = S->rem;
  unsigned long long rank_excl = 0;
  for (int r = 0; r < p.rank; ++r) rank_excl += p.d.gather[r];
  unsigned long long carry = p.d.tile_tie_excl[blockIdx.x] + rank_excl;
  const uint32_t *bm_old = p.d.bm[p.cur];
  uint32_t *bm_new = p.d.bm[p.cur ^ 1];
  uint32_t n_pf = 0, n_ev = 0, n_el = 0;
  unsigned long long h2d = 0, tie_kept = 0;
  __shared__ unsigned long long sh_tot;
  const int lane = threadIdx.x & 31;
  for (uint32_t k0 = 0; k0 < TILE; k0 += NT) {
    const uint64_t i = t0 + k0 + threadIdx.x;
    const bool valid = i < p.n_local;
    bool el = false, tie = false;
    uint32_t key = KEY_NONE, fp = 0;
    if (valid) {
      el = (p.d.elig[i >> 5] >> (i & 31)) & 1u;
      key = p.d.keys[i];
      tie = el && !all_fit && key == dstar;
      if (tie) fp = p.rec[i].y;
    }
    const unsigned long long ex = block_excl_scan((unsigned long long)fp, &sh_tot);
    __syncthreads();
    const unsigned long long incl = carry + ex + fp;
    carry += sh_tot;
    const bool kept = el && (all_fit || key < dstar || (tie && incl <= rem));
    if (tie && kept) tie_kept += fp;
    const uint32_t kw = __ballot_sync(FULL, kept);
    const uint32_t ew = __ballot_sync(FULL, el);
    const uint64_t wi = i >> 5;
    uint32_t old = 0;
    if (wi < p.n_words) old = bm_old[wi];
    if (lane == 0 && wi < p.n_words && (t0 + k0 + (threadIdx.x & ~31u)) < p.n_local) {
      bm_new[wi] = kw;
      n_pf += __popc(kw & ~old);
      n_ev += __popc(old & ~kw);
      n_el += __popc(ew);
    }
    const bool pf = kept && !((old >> lane) & 1u);
    if (pf) h2d += p.rec[i].y;
    __syncthreads();
  }
  n_pf = block_sum(n_pf);
  n_ev = block_sum(n_ev);
  n_el = block_sum(n_el);
  h2d = block_sum(h2d);
  tie_kept = block_sum(tie_kept);
  if (threadIdx.x == 0) {
    p.d.tile_pf[blockIdx.x] = n_pf;
    p.d.tile_ev[blockIdx.x] = n_ev;
    p.d.tile_elig[blockIdx.x] = n_el;
    p.d.tile_h2d[blockIdx.x] = h2d;
    p.d.tile_tiekept[blockIdx.x] = tie_kept;
  }
}

__global__ void __launch_bounds__(NT) k_count_scan(Params p) {
  __shared__ uint32_t tot_pf, tot_ev, tot_el;
  __shared__ unsigned long long tot_h2d, tot_tk;
  block_scan_array<uint32_t>(p.d.tile_pf, p.d.tile_pf_excl, p.n_tiles, &tot_pf);
  __syncthreads();
  block_scan_array<uint32_t>(p.d.tile_ev, p.d.tile_ev_excl, p.n_tiles, &tot_ev);
  __syncthreads();
  unsigned long long a = 0, b = 0;
  uint32_t c = 0;
  for (uint64_t t = threadIdx.x; t < p.n_tiles; t += NT) {
    a += p.d.tile_h2d[t];
    b += p.d.tile_tiekept[t];
    c += p.d.tile_elig[t];
  }
  a = block_sum(a);
  b = block_sum(b);
  c = block_sum(c);
  if (threadIdx.x == 0) {
    tot_h2d = a;
    tot_tk = b;
    tot_el = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    SelState *S = p.d.state;
    S->tie_kept = tot_tk;
    unsigned long long *H = p.d.header;
    H[H_N_PF] = tot_pf;
    H[H_N_EV] = tot_ev;
    H[H_H2D] = tot_h2d;
    H[H_CUT_BITS] = S->all_fit ? 0xFFFFFFFFull : S->dstar;
    H[H_CUT_REM] = S->rem;
    H[H_KEPT] = S->all_fit ? (p.budget - S->rem) : (p.budget - S->rem) + tot_tk;
    H[H_N_ELIG] = tot_el;
    H[H_STATUS] = S->status;
    H[H_SEQ] += 1;
  }
}

// ------------------------------------------------------------------------------------
// a5: list compaction in id order (prefetch ascending id, evict descending id), then a
// stable LSD radix sort by distance bits (prefetch: ascending d; evict: descending d via
// the complemented key) -> ascending / descending (d, id) order.

__global__ void __launch_bounds__(64) k_compact(Params p) {
  const uint64_t w0 = (uint64_t)blockIdx.x * (TILE / 32);
  const uint64_t wi = w0 + threadIdx.x;
  const uint32_t *bm_old = p.d.bm[p.cur];
  const uint32_t *bm_new = p.d.bm[p.cur ^ 1];
  uint32_t pfw = 0, evw = 0;
  if (wi < p.n_words) {
    const uint32_t o = bm_old[wi], n = bm_new[wi];
    pfw = n & ~o;
    evw = o & ~n;
  }
  __shared__ uint32_t sh_pf[64], sh_ev[64];
  sh_pf[threadIdx.x] = __popc(pfw);
  sh_ev[threadIdx.x] = __popc(evw);
  __syncthreads();
  uint32_t epf = 0, eev = 0;
  for (uint32_t k = 0; k < threadIdx.x; ++k) {
    epf += sh_pf[k];
    eev += sh_ev[k];
  }
  uint32_t pos = p.d.tile_pf_excl[blockIdx.x] + epf;
  const uint32_t n_ev_tot = (uint32_t)p.d.header[H_N_EV];
  uint32_t epos = p.d.tile_ev_excl[blockIdx.x] + eev;
  SelState *S = p.d.state;
  uint32_t or_pf = 0, and_pf = 0xFFFFFFFFu, or_ev = 0, and_ev = 0xFFFFFFFFu;
  while (pfw) {
    const int b = __ffs(pfw) - 1;
    pfw &= pfw - 1;
    const uint32_t i = (uint32_t)(wi * 32 + b);
    const uint32_t key = p.d.keys[i];
    p.d.sort_ka[pos] = key;
    p.d.sort_va[pos] = i;
    or_pf |= key;
    and_pf &= key;
    ++pos;
  }
  while (evw) {
    const int b = __ffs(evw) - 1;
    evw &= evw - 1;
    const uint32_t i = (uint32_t)(wi * 32 + b);
    const uint32_t key = ~p.d.keys[i];
    const uint32_t slot = n_ev_tot - 1 - epos;
    p.d.pfa_key[slot] = key;  // evict list staging (second buffer set)
    p.d.pfa_val[slot] = i;
    or_ev |= key;
    and_ev &= key;
    ++epos;
  }
  or_pf = __reduce_or_sync(FULL, or_pf);
  and_pf = __reduce_and_sync(FULL, and_pf);
  or_ev = __reduce_or_sync(FULL, or_ev);
  and_ev = __reduce_and_sync(FULL, and_ev);
  if ((threadIdx.x & 31) == 0) {
    if (or_pf) atomicOr(&S->sort_or[0], or_pf);
    if (and_pf != 0xFFFFFFFFu) atomicAnd(&S->sort_and[0], and_pf);
    if (or_ev) atomicOr(&S->sort_or[1], or_ev);
    if (and_ev != 0xFFFFFFFFu) atomicAnd(&S->sort_and[1], and_ev);
  }
}

// digit d of pass q: bits [0,11), [11,22), [22,32)
__device__ __forceinline__ uint32_t digit_of(uint32_t key, int pass) {
  return pass == 0 ? (key & 2047u) : pass == 1 ? ((key >> 11) & 2047u) : (key >> 22);
}
__device__ __forceinline__ uint32_t digit_mask(int pass) {
  return pass == 0 ? 0x7FFu : pass == 1 ? (0x7FFu << 11) : (0x3FFu << 22);
}
__device__ __forceinline__ bool pass_needed(const SelState *S, int list, int pass) {
  const uint32_t varying = S->sort_or[list] ^ S->sort_and[list];
  return (varying & digit_mask(pass)) != 0;
}

struct SortIO {
  const uint32_t *kin, *vin;
  uint32_t *kout, *vout;
};

__global__ void __launch_bounds__(NT) k_sort_hist(Params p, int list, int pass, SortIO io) {
  const uint32_t count = (uint32_t)p.d.header[list == 0 ? H_N_PF : H_N_EV];
  const uint32_t n_chunks = (count + SORT_CH - 1) / SORT_CH;
  if (blockIdx.x >= n_chunks || !pass_needed(p.d.state, list, pass)) return;
  __shared__ uint32_t h[2048];
  for (int b = threadIdx.x; b < 2048; b += NT) h[b] = 0;
  __syncthreads();
  const uint32_t c0 = blockIdx.x * SORT_CH;
  for (uint32_t k = threadIdx.x; k < SORT_CH; k += NT) {
    const uint32_t e = c0 + k;
    if (e < count) atomicAdd(&h[digit_of(io.kin[e], pass)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 2048; b += NT) p.d.sort_cnt[(uint64_t)b * n_chunks + blockIdx.x] = h[b];
}

__global__ void __launch_bounds__(NT) k_sort_scan(Params p, int list, int pass) {
  const uint32_t count = (uint32_t)p.d.header[list == 0 ? H_N_PF : H_N_EV];
  const uint32_t n_chunks = (count + SORT_CH - 1) / SORT_CH;
  if (n_chunks == 0 || !pass_needed(p.d.state, list, pass)) return;
  block_scan_array<uint32_t>(p.d.sort_cnt, p.d.sort_cnt, (uint64_t)2048 * n_chunks, nullptr);
}

__global__ void __launch_bounds__(NT) k_sort_scatter(Params p, int list, int pass, SortIO io) {
  const uint32_t count = (uint32_t)p.d.header[list == 0 ? H_N_PF : H_N_EV];
  const uint32_t n_chunks = (count + SORT_CH - 1) / SORT_CH;
  if (blockIdx.x >= n_chunks) return;
  const uint32_t c0 = blockIdx.x * SORT_CH;
  if (!pass_needed(p.d.state, list, pass)) {  // identity copy keeps the buffer schedule static
    for (uint32_t k = threadIdx.x; k < SORT_CH; k += NT) {
      const uint32_t e = c0 + k;
      if (e < count) {
        io.kout[e] = io.kin[e];
        io.vout[e] = io.vin[e];
      }
    }
    return;
  }
  __shared__ uint32_t run[2048];
  for (int b = threadIdx.x; b < 2048; b += NT) run[b] = p.d.sort_cnt[(uint64_t)b * n_chunks + blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t k0 = 0; k0 < SORT_CH; k0 += NT) {
    const uint32_t e = c0 + k0 + threadIdx.x;
    const bool valid = e < count;
    const uint32_t key = valid ? io.kin[e] : 0u;
    const uint32_t val = valid ? io.vin[e] : 0u;
    const uint32_t dg = valid ? digit_of(key, pass) : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(FULL, dg);
    const uint32_t rank = __popc(peers & lanemask_lt());
    const bool leader = (peers & lanemask_lt()) == 0;
    for (int w = 0; w < NT / 32; ++w) {
      if (warp == w && valid) {
        const uint32_t pos = run[dg] + rank;
        io.kout[pos] = key;
        io.vout[pos] = val;
      }
      __syncwarp();
      if (warp == w && valid && leader) run[dg] += __popc(peers);
      __syncthreads();
    }
  }
}

__global__ void k_sort_finish(Params p, int list, const uint32_t *vals) {
  const uint32_t count = (uint32_t)p.d.header[list == 0 ? H_N_PF : H_N_EV];
  uint32_t *out = list == 0 ? p.d.pf_ids : p.d.ev_ids;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x)
    out[e] = (uint32_t)(vals[e] + p.shard_begin);
}

// ------------------------------------------------------------------------------------
// a5: block expansion and deterministic page assignment.
// Chunk c of a list covers entries [c*EXP_CH, (c+1)*EXP_CH).  exp_sum layout:
//   [0][chunk] evict pages, [1][chunk] evict write-back pages, [2][chunk] prefetch pages

__device__ __forceinline__ void agent_pages(const Params &p, uint32_t a, bool dirty, uint32_t &pages,
                                            uint32_t &wb_pages) {
  const uint64_t b0 = p.blk_ptr[a], b1 = p.blk_ptr[a + 1];
  pages = (uint32_t)(p.d.page_first[b1] - p.d.page_first[b0]);
  wb_pages = 0;
  if (dirty)
    for (uint64_t b = b0; b < b1; ++b)
      if (p.blk_kind[b] != 0) wb_pages += (uint32_t)(p.d.page_first[b + 1] - p.d.page_first[b]);
}

__global__ void __launch_bounds__(NT) k_exp_count(Params p, uint64_t max_chunks) {
  const uint32_t n_pf = (uint32_t)p.d.header[H_N_PF], n_ev = (uint32_t)p.d.header[H_N_EV];
  const uint32_t e = blockIdx.x * EXP_CH + threadIdx.x;
  uint32_t evp = 0, evw = 0, pfp = 0;
  unsigned long long wb_bytes = 0;
  if (e < n_ev) {
    const uint32_t a = p.d.ev_ids[e] - (uint32_t)p.shard_begin;
    const bool dirty = p.ev_dirty ? p.ev_dirty[e] != 0 : ((p.rec[a].z >> 4) & 1u);
    agent_pages(p, a, dirty, evp, evw);
    if (dirty)  // R13: KV + HIST blocks of a dirty evicted agent are written back
      for (uint64_t b = p.blk_ptr[a]; b < p.blk_ptr[a + 1]; ++b)
        if (p.blk_kind[b] != 0) wb_bytes += p.blk_size[b];
  }
  if (e < n_pf) {
    const uint32_t a = p.d.pf_ids[e] - (uint32_t)p.shard_begin;
    uint32_t dummy;
    agent_pages(p, a, false, pfp, dummy);
  }
  const unsigned long long s0 = block_sum((unsigned long long)evp);
  const unsigned long long s1 = block_sum((unsigned long long)evw);
  const unsigned long long s2 = block_sum((unsigned long long)pfp);
  const unsigned long long s3 = block_sum(wb_bytes);
  if (threadIdx.x == 0) {
    p.d.exp_sum[blockIdx.x] = s0;
    p.d.exp_sum[max_chunks + blockIdx.x] = s1;
    p.d.exp_sum[2 * max_chunks + blockIdx.x] = s2;
    p.d.exp_sum[3 * max_chunks + blockIdx.x] = s3;
  }
}

__global__ void __launch_bounds__(NT) k_exp_scan(Params p, uint64_t max_chunks) {
  const uint32_t n_pf = (uint32_t)p.d.header[H_N_PF], n_ev = (uint32_t)p.d.header[H_N_EV];
  const uint64_t nc = (max(n_pf, n_ev) + EXP_CH - 1) / EXP_CH;
  __shared__ unsigned long long t0, t1, t2, t3;
  block_scan_array<unsigned long long>(p.d.exp_sum, p.d.exp_excl, nc, &t0);
  __syncthreads();
  block_scan_array<unsigned long long>(p.d.exp_sum + max_chunks, p.d.exp_excl + max_chunks, nc, &t1);
  __syncthreads();
  block_scan_array<unsigned long long>(p.d.exp_sum + 2 * max_chunks, p.d.exp_excl + 2 * max_chunks, nc, &t2);
  __syncthreads();
  block_scan_array<unsigned long long>(p.d.exp_sum + 3 * max_chunks, p.d.exp_excl + 3 * max_chunks, nc, &t3);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long *H = p.d.header;
    H[H_D2H] = t3;
    if (p.n_dev_pages == 0) return;  // logical sizes (NO_TRANSFER): byte accounting only
    unsigned long long *desc = p.d.desc[p.desc_buf];
    const unsigned long long head = p.d.pool[0], tail = p.d.pool[1];
    H[H_N_D2H] = t1;
    H[H_N_H2D] = t2;
    desc[0] = t1;
    desc[1] = t2;
    // prefetched pages popped below the old tail were free before this step's releases: their
    // loads do not wait for the write-backs (D2H and H2D then run concurrently)
    desc[2] = t2 < tail - head ? t2 : tail - head;
    desc[3] = 0;
    // free pages after releasing = tail + t0 - head; the prefetch must fit (always true when
    // dev pages >= budget pages; flagged otherwise)
    if (t2 > tail + t0 - head) {
      p.d.state->status |= ST_NO_PAGES;
      H[H_STATUS] |= ST_NO_PAGES;
    }
    H[H_POOL_HEAD] = head + t2;
    H[H_POOL_TAIL] = tail + t0;
  }
}

// release (evict) or assign (prefetch) the pages of one list chunk
template <bool RELEASE>
__global__ void __launch_bounds__(NT) k_pages(Params p, uint64_t max_chunks) {
  const uint32_t count = (uint32_t)p.d.header[RELEASE ? H_N_EV : H_N_PF];
  const uint32_t c0 = blockIdx.x * EXP_CH;
  if (c0 >= count || (p.d.header[H_STATUS] & ST_NO_PAGES)) return;
  __shared__ unsigned long long sh_off[EXP_CH], sh_wb[EXP_CH];
  __shared__ unsigned long long sh_t;
  const uint32_t e = c0 + threadIdx.x;
  uint32_t a = 0, pages = 0, wb = 0;
  bool dirty = false;
  if (e < count) {
    a = (RELEASE ? p.d.ev_ids[e] : p.d.pf_ids[e]) - (uint32_t)p.shard_begin;
    dirty = RELEASE && (p.ev_dirty ? p.ev_dirty[e] != 0 : ((p.rec[a].z >> 4) & 1u));
    agent_pages(p, a, dirty, pages, wb);
  }
  const unsigned long long ex = block_excl_scan((unsigned long long)pages, &sh_t);
  __syncthreads();
  const unsigned long long exw = block_excl_scan((unsigned long long)wb, &sh_t);
  __syncthreads();
  const unsigned long long chunk_off = p.d.exp_excl[(RELEASE ? 0 : 2 * max_chunks) + blockIdx.x];
  sh_off[threadIdx.x] = chunk_off + ex;
  sh_wb[threadIdx.x] = (RELEASE ? p.d.exp_excl[max_chunks + blockIdx.x] : 0ull) + exw;
  __syncthreads();
  const unsigned long long head = p.d.pool[0], tail = p.d.pool[1];
  const unsigned long long npg = p.n_dev_pages;
  unsigned long long *desc = p.d.desc[p.desc_buf] + DESC_HDR;  // pairs after the counters
  unsigned long long *d2h = desc;
  unsigned long long *h2d = desc + 2 * p.desc_cap;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t n_here = min(count - c0, EXP_CH);
  for (uint32_t k = warp; k < n_here; k += NT / 32) {
    const uint32_t ag = (RELEASE ? p.d.ev_ids[c0 + k] : p.d.pf_ids[c0 + k]) - (uint32_t)p.shard_begin;
    const bool dty = RELEASE && (p.ev_dirty ? p.ev_dirty[c0 + k] != 0 : ((p.rec[ag].z >> 4) & 1u));
    unsigned long long off = sh_off[k];
    unsigned long long woff = sh_wb[k];
    for (uint64_t b = p.blk_ptr[ag]; b < p.blk_ptr[ag + 1]; ++b) {
      const unsigned long long pf0 = p.d.page_first[b];
      const uint32_t np = (uint32_t)(p.d.page_first[b + 1] - pf0);
      const bool wbk = dty && p.blk_kind[b] != 0;
      const unsigned long long hoff = p.blk_host_off[b];
      for (uint32_t q = lane; q < np; q += 32) {
        if (RELEASE) {
          const uint32_t pg = p.d.page_table[pf0 + q];
          p.d.ring[(tail + off + q) % npg] = pg;
          p.d.page_table[pf0 + q] = PAGE_NONE;
          if (wbk) {
            d2h[2 * (woff + q)] = hoff + (unsigned long long)q * p.page_bytes;
            d2h[2 * (woff + q) + 1] = pg;
          }
        } else {
          const uint32_t pg = p.d.ring[(head + off + q) % npg];
          p.d.page_table[pf0 + q] = pg;
          h2d[2 * (off + q)] = hoff + (unsigned long long)q * p.page_bytes;
          h2d[2 * (off + q) + 1] = pg;
        }
      }
      off += np;
      if (wbk) woff += np;
    }
  }
}

__global__ void k_pool_update(Params p) {
  p.d.pool[0] = p.d.header[H_POOL_HEAD];
  p.d.pool[1] = p.d.header[H_POOL_TAIL];
}

// init: pages for the initially resident agents in id order (block order, page order)
__global__ void k_init_pages_count(Params p, const uint32_t *res, uint64_t *cnt) {
  // serial over agents in a single thread: init-time only
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  unsigned long long head = 0;
  for (uint64_t a = 0; a < p.n_local; ++a) {
    if (!((res[a >> 5] >> (a & 31)) & 1u)) continue;
    for (uint64_t b = p.blk_ptr[a]; b < p.blk_ptr[a + 1]; ++b)
      for (unsigned long long q = p.d.page_first[b]; q < p.d.page_first[b + 1]; ++q) {
        p.d.page_table[q] = p.d.ring[head % p.n_dev_pages];
        ++head;
      }
  }
  p.d.pool[0] = head;
  p.d.pool[1] = p.n_dev_pages;
  *cnt = head;
}

__global__ void k_init_ring(Params p, const uint32_t *res) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.d.pool[0] = 0;              // FIFO of free pages: all pages, in index order
    p.d.pool[1] = p.n_dev_pages;
  }
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < p.n_dev_pages; q += (uint64_t)gridDim.x * blockDim.x)
    p.d.ring[q] = (uint32_t)q;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < p.n_words; w += (uint64_t)gridDim.x * blockDim.x) {
    p.d.bm[0][w] = res ? res[w] : 0u;
    p.d.bm[1][w] = 0u;
  }
}

__global__ void k_init_page_table(Params p, uint64_t n_block_pages) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n_block_pages; q += (uint64_t)gridDim.x * blockDim.x)
    p.d.page_table[q] = PAGE_NONE;
}

// ------------------------------------------------------------------------------------
// a6: page copies.  One CTA per 64 KiB page per iteration: every thread issues all its
// 128-bit loads (16 per thread for 64 KiB) before its stores, so a CTA keeps a whole page
// in flight across PCIe; the grid is small (the copy overlaps the next plan).

// MODE 0: write-backs (device page -> host), all; MODE 1: loads (host -> device page)
// [0, n_indep); MODE 2: loads [n_indep, n_h2d) (after the write-backs).  Each descriptor moves
// `slot` bytes: host page bytes [off, off + slot) <-> device slot pg (slot = page_bytes, off = 0;
// TP-sliced: this rank's slice of the page).
template <int MODE>
__global__ void __launch_bounds__(NT) k_copy_pages(const unsigned long long *desc_base, uint8_t *host, uint8_t *dev,
                                                  uint64_t slot, uint64_t off, uint64_t desc_cap) {
  constexpr bool D2H = MODE == 0;
  const unsigned long long lo = MODE == 2 ? desc_base[2] : 0ull;
  const unsigned long long hi = MODE == 0 ? desc_base[0] : (MODE == 1 ? desc_base[2] : desc_base[1]);
  const unsigned long long *desc = desc_base + DESC_HDR + (D2H ? 0 : 2 * desc_cap);
  const uint32_t vec_per_page = (uint32_t)(slot / 16);
  for (unsigned long long k = lo + blockIdx.x; k < hi; k += gridDim.x) {
    const unsigned long long hoff = desc[2 * k] + off;
    const unsigned long long pg = desc[2 * k + 1];
    const uint4 *src = reinterpret_cast<const uint4 *>(D2H ? dev + pg * slot : host + hoff);
    uint4 *dst = reinterpret_cast<uint4 *>(D2H ? host + hoff : dev + pg * slot);
    for (uint32_t v0 = 0; v0 < vec_per_page; v0 += NT * 16) {
      uint4 buf[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint32_t v = v0 + u * NT + threadIdx.x;
        if (v < vec_per_page) buf[u] = ld_stream(src + v);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint32_t v = v0 + u * NT + threadIdx.x;
        if (v < vec_per_page) dst[v] = buf[u];
      }
    }
  }
}

// TMA variant: one thread per CTA drives bulk copies (cp.async.bulk) through a ring of shared-
// memory chunks: global (host-mapped or device) -> shared with an mbarrier completion, then
// shared -> global as a bulk group; no register staging, 128 KB in flight per CTA.
constexpr uint32_t TMA_CH = 16384, TMA_NB = 8;
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(32) k_copy_pages_tma(const unsigned long long *desc_base, uint8_t *host, uint8_t *dev,
                                                      uint64_t slot, uint64_t off, uint64_t desc_cap) {
  constexpr bool D2H = MODE == 0;
  extern __shared__ __align__(128) uint8_t tbuf[];
  __shared__ __align__(8) unsigned long long bar[TMA_NB];
  if (threadIdx.x != 0) return;
  const unsigned long long lo = MODE == 2 ? desc_base[2] : 0ull;
  const unsigned long long hi = MODE == 0 ? desc_base[0] : (MODE == 1 ? desc_base[2] : desc_base[1]);
  const unsigned long long *desc = desc_base + DESC_HDR + (D2H ? 0 : 2 * desc_cap);
  // chunk size: 16 KB, or the whole slot when it is smaller (slot % 16 == 0, and slot % 16 KB == 0
  // when larger: checked by the launcher)
  const uint32_t CH = slot < TMA_CH ? (uint32_t)slot : TMA_CH;
  const uint32_t cpp = (uint32_t)(slot / CH);  // chunks per slot
  const unsigned long long mine = hi > lo + blockIdx.x ? (hi - lo - blockIdx.x + gridDim.x - 1) / gridDim.x : 0ull;
  const unsigned long long n = mine * cpp;  // this CTA's chunks: its pages in order, chunks in order
  if (n == 0) return;
  for (uint32_t i = 0; i < TMA_NB; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto src_dst = [&](unsigned long long j, const uint8_t *&src, uint8_t *&dst) {
    const unsigned long long k = lo + blockIdx.x + (j / cpp) * gridDim.x, co = (j % cpp) * CH;
    const unsigned long long hoff = desc[2 * k] + off, pg = desc[2 * k + 1];
    src = (D2H ? dev + pg * slot : host + hoff) + co;
    dst = (D2H ? host + hoff : dev + pg * slot) + co;
  };
  auto load = [&](unsigned long long j) {
    const uint8_t *src;
    uint8_t *dst;
    src_dst(j, src, dst);
    const uint32_t b = smem_u32(&bar[j % TMA_NB]), sm = smem_u32(tbuf + (j % TMA_NB) * TMA_CH);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm),
                 "l"(src), "r"(CH), "r"(b)
                 : "memory");
  };
  for (unsigned long long j = 0; j < n && j < TMA_NB; ++j) load(j);
  for (unsigned long long j = 0; j < n; ++j) {
    const uint32_t b = smem_u32(&bar[j % TMA_NB]), ph = (uint32_t)((j / TMA_NB) & 1);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok)
                   : "r"(b), "r"(ph)
                   : "memory");
    const uint8_t *src;
    uint8_t *dst;
    src_dst(j, src, dst);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(tbuf + (j % TMA_NB) * TMA_CH)), "r"(CH)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the previous chunk's store has read its buffer: refill that buffer
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    if (j >= 1 && j - 1 + TMA_NB < n) load(j - 1 + TMA_NB);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------------------------
// launchers

static inline int ceil_div(uint64_t a, uint64_t b) { return (int)((a + b - 1) / b); }
static inline int tiles_grid(const Params &p) { return p.n_tiles > 0 ? (int)p.n_tiles : 1; }

int launch_plan_init(const Params &p, cudaStream_t s) {
  k_plan_init<<<8, NT, 0, s>>>(p);
  return 1;
}

int launch_interaction(const Params &p, int64_t now, cudaStream_t s, int grid) {
  if (p.n_kin == 0) return 0;
  const int g = min(grid, max(1, ceil_div(max(p.n_local, p.n_kin), NT)));
  k_int_compact<<<g, NT, 0, s>>>(p, now);
  if (p.n_kin >= GRID_MIN_PARTICIPANTS) return 1 + launch_grid_pairmin(p, s, grid);
  k_pairmin<<<max(1, ceil_div(p.n_kin, NT)), NT, 0, s>>>(p);
  return 2;
}

int launch_score(const Params &p, int64_t now, float *dist_out, cudaStream_t s, int grid) {
  int n = launch_interaction(p, now, s, grid);
  const int g = min(grid / 2, max(1, ceil_div(p.n_local, NT)));  // 2 blocks per SM: fewer histogram flushes
  k_score<<<g, NT, 0, s>>>(p, now);
  ++n;
  if (dist_out) {
    k_copy_keys<<<min(grid, max(1, ceil_div(p.n_local, NT))), NT, 0, s>>>(p, dist_out);
    ++n;
  }
  return n;
}

int launch_select(const Params &p, int level, cudaStream_t s) {
  k_select<<<1, NT, 0, s>>>(p, level);
  return 1;
}

int launch_hist(const Params &p, int level, cudaStream_t s, int grid) {
  k_hist<<<min(grid, max(1, ceil_div(p.n_local, NT))), NT, 0, s>>>(p, level);
  return 1;
}

int launch_tie(const Params &p, cudaStream_t s) {
  k_tie_partial<<<tiles_grid(p), NT, 0, s>>>(p);
  k_tie_scan<<<1, NT, 0, s>>>(p);
  return 2;
}

int launch_emit(const Params &p, cudaStream_t s) {
  k_emit<<<tiles_grid(p), NT, 0, s>>>(p);
  k_count_scan<<<1, NT, 0, s>>>(p);
  return 2;
}

int launch_lists(const Params &p, cudaStream_t s) {
  int n = 0;
  k_compact<<<tiles_grid(p), 64, 0, s>>>(p);
  ++n;
  const int max_chunks = max(1, ceil_div(p.n_local, SORT_CH));
  for (int list = 0; list < 2; ++list) {
    uint32_t *ka = list == 0 ? p.d.sort_ka : p.d.pfa_key;
    uint32_t *va = list == 0 ? p.d.sort_va : p.d.pfa_val;
    uint32_t *kb = p.d.sort_kb, *vb = p.d.sort_vb;
    // A -> B -> A -> B
    for (int pass = 0; pass < 3; ++pass) {
      SortIO io;
      if (pass == 1) io = SortIO{kb, vb, ka, va};
      else io = SortIO{ka, va, kb, vb};
      k_sort_hist<<<max_chunks, NT, 0, s>>>(p, list, pass, io);
      k_sort_scan<<<1, NT, 0, s>>>(p, list, pass);
      k_sort_scatter<<<max_chunks, NT, 0, s>>>(p, list, pass, io);
      n += 3;
    }
    k_sort_finish<<<min(1184, max_chunks * 8), NT, 0, s>>>(p, list, vb);
    ++n;
  }
  return n;
}

int launch_expand(const Params &p, cudaStream_t s) {
  const uint64_t max_chunks = (uint64_t)max(1, ceil_div(p.n_local, EXP_CH));
  k_exp_count<<<(int)max_chunks, NT, 0, s>>>(p, max_chunks);
  k_exp_scan<<<1, NT, 0, s>>>(p, max_chunks);
  if (p.n_dev_pages == 0) return 2;
  k_pages<true><<<(int)max_chunks, NT, 0, s>>>(p, max_chunks);
  k_pages<false><<<(int)max_chunks, NT, 0, s>>>(p, max_chunks);
  k_pool_update<<<1, 1, 0, s>>>(p);
  return 5;
}

int launch_transfer(const Params &p, cudaStream_t s, int ctas) {
  const unsigned long long *desc = p.d.desc[p.desc_buf];
  k_copy_pages<0><<<ctas, NT, 0, s>>>(desc, p.host_arena, p.dev_arena, p.slot_bytes, p.slice_off, p.desc_cap);
  k_copy_pages<1><<<ctas, NT, 0, s>>>(desc, p.host_arena, p.dev_arena, p.slot_bytes, p.slice_off, p.desc_cap);
  k_copy_pages<2><<<ctas, NT, 0, s>>>(desc, p.host_arena, p.dev_arena, p.slot_bytes, p.slice_off, p.desc_cap);
  return 3;
}

// write-backs on s, independent loads concurrently on s2, dependent loads on s after the
// write-backs; the caller joins s2 back into s
int launch_transfer_split(const Params &p, cudaStream_t s, cudaStream_t s2, int ctas) {
  const unsigned long long *desc = p.d.desc[p.desc_buf];
  // bulk copies when pages are whole 16 KB chunks (A/B: the same link fraction as the
  // register-staged copy, profiles/r02_copy_tma_ab.log, with one thread and no registers per CTA)
#ifndef COPY_REGS
  if (p.slot_bytes % 16 == 0 && (p.slot_bytes <= TMA_CH || p.slot_bytes % TMA_CH == 0)) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_copy_pages_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, TMA_CH * TMA_NB);
      cudaFuncSetAttribute(k_copy_pages_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, TMA_CH * TMA_NB);
      cudaFuncSetAttribute(k_copy_pages_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, TMA_CH * TMA_NB);
      attr = true;
    }
    k_copy_pages_tma<0><<<ctas, 32, TMA_CH * TMA_NB, s>>>(desc, p.host_arena, p.dev_arena, p.slot_bytes, p.slice_off, p.desc_cap);
    k_copy_pages_tma<1><<<ctas, 32, TMA_CH * TMA_NB, s2>>>(desc, p.host_arena, p.dev_arena, p.slot_bytes, p.slice_off, p.desc_cap);
    k_copy_pages_tma<2><<<ctas, 32, TMA_CH * TMA_NB, s>>>(desc, p.host_arena, p.dev_arena, p.slot_bytes, p.slice_off, p.desc_cap);
    return 3;
  }
#endif
  k_copy_pages<0><<<ctas, NT, 0, s>>>(desc, p.host_arena, p.dev_arena, p.slot_bytes, p.slice_off, p.desc_cap);
  k_copy_pages<1><<<ctas, NT, 0, s2>>>(desc, p.host_arena, p.dev_arena, p.slot_bytes, p.slice_off, p.desc_cap);
  k_copy_pages<2><<<ctas, NT, 0, s>>>(desc, p.host_arena, p.dev_arena, p.slot_bytes, p.slice_off, p.desc_cap);
  return 3;
}

int launch_init_pages(const Params &p, const uint32_t *resident_init, cudaStream_t s) {
  k_init_ring<<<256, NT, 0, s>>>(p, resident_init);
  if (p.n_dev_pages == 0) return 1;
  return 1;
}

int launch_copy_dist(const Params &p, float *dist_out, cudaStream_t s) {
  k_copy_keys<<<256, NT, 0, s>>>(p, dist_out);
  return 1;
}

__global__ void k_fix_kept(Params p) {
  const SelState *S = p.d.state;
  p.d.header[H_KEPT] = S->all_fit ? (p.budget - S->rem) : (p.budget - S->rem) + S->tie_kept;
}

__global__ void k_mask_tail(Params p) {
  if (p.n_local % 32 != 0 && p.n_words > 0) p.d.bm[0][p.n_words - 1] &= (1u << (p.n_local % 32)) - 1u;
}

int launch_fix_kept(const Params &p, cudaStream_t s) {
  k_fix_kept<<<1, 1, 0, s>>>(p);
  return 1;
}

int launch_mask_tail(const Params &p, cudaStream_t s) {
  k_mask_tail<<<1, 1, 0, s>>>(p);
  return 1;
}

// exported for api.cpp (init-time page table)
void launch_init_page_table(const Params &p, uint64_t n_block_pages, const uint32_t *res, uint64_t *cnt_dev,
                            cudaStream_t s) {
  k_init_page_table<<<256, NT, 0, s>>>(p, n_block_pages);
  if (res) k_init_pages_count<<<1, 1, 0, s>>>(p, res, cnt_dev);
}

void launch_init_transfer(const Params &p, cudaStream_t s, int ctas) { launch_transfer(p, s, ctas); }

// ------------------------------------------------------------------------------------
// Loopback worlds (SCALESIM_F_LOOPBACK): the exchanges of §8(e) through device
// memory, one launch for the world.  Per-step inputs (records, kinematics) by value; every
// other field of rank r from its device parameter copy.
struct WRank {
  const Params *pd;
  const uint4 *rec;
};
struct WArgs {
  uint32_t G;
  int64_t now;
  WRank r[FUSED_MAX_WORLD];
};

static WArgs world_args(const Params *const *ps, uint32_t G, int64_t now) {
  WArgs w = {};
  w.G = G;
  w.now = now;
  for (uint32_t r = 0; r < G; ++r) {
    w.r[r].pd = reinterpret_cast<const Params *>(ps[r]->d.params_dev);
    w.r[r].rec = ps[r]->rec;
  }
  return w;
}

// §8(e) "an all-gather of kin for active INT agents": rank s's participants (k_int_compact's
// list) copied into every rank's world list at s's offset (participants of lower ranks first);
// block (d, s) of chunk x.  wcnt[d][r] = offset of rank r, wcnt[d][G] = the world's count.
__global__ void __launch_bounds__(NT) k_kin_allgather(WArgs w) {
  const uint32_t dr = blockIdx.y, sr = blockIdx.z;
  const Dev &dd = w.r[dr].pd->d;
  uint32_t off = 0, tot = 0;
  for (uint32_t r = 0; r < w.G; ++r) {
    const uint32_t n = w.r[r].pd->n_kin ? w.r[r].pd->d.state->int_count : 0u;
    if (r < sr) off += n;
    tot += n;
  }
  if (blockIdx.x == 0 && sr == 0 && threadIdx.x == 0) {
    uint32_t o = 0;
    for (uint32_t r = 0; r < w.G; ++r) {
      dd.wcnt[r] = o;
      o += w.r[r].pd->n_kin ? w.r[r].pd->d.state->int_count : 0u;
    }
    dd.wcnt[w.G] = tot;
  }
  const Params &ps = *w.r[sr].pd;
  if (ps.n_kin == 0 || w.r[dr].pd->n_kin == 0) return;  // (a rank without interaction agents scans nothing)
  const uint32_t n = ps.d.state->int_count;
  for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) dd.wkin[off + i] = ps.d.ilist_kin[i];
}

// Eq. 2 over the world's participants: rank r's participant i against every
// participant j of the world but itself (j == wcnt[r] + i); the same rounding and division
// filter as k_pairmin, so D_int is the exact min of the rounded quotients at any world size.
__global__ void __launch_bounds__(NT) k_pairmin_world(Params p) {
  __shared__ float4 tile[NT];
  const uint32_t count = p.d.state->int_count, total = p.d.wcnt[p.world], self = p.d.wcnt[p.rank];
  const uint32_t i = blockIdx.x * NT + threadIdx.x;
  if (blockIdx.x * NT >= count) return;
  const bool mine = i < count;
  const float4 ki = mine ? p.d.ilist_kin[i] : make_float4(0, 0, 0, 0);
  float best = __int_as_float(0x7F800000);
  for (uint32_t j0 = 0; j0 < total; j0 += NT) {
    __syncthreads();
    if (j0 + threadIdx.x < total) tile[threadIdx.x] = p.d.wkin[j0 + threadIdx.x];
    __syncthreads();
    const uint32_t jn = min((uint32_t)NT, total - j0);
    if (mine) {
      for (uint32_t jj = 0; jj < jn; ++jj) {
        const float4 kj = tile[jj];
        const float dx = __fsub_rn(kj.x, ki.x);
        const float dy = __fsub_rn(kj.y, ki.y);
        const float dvx = __fsub_rn(kj.z, ki.z);
        const float dvy = __fsub_rn(kj.w, ki.w);
        const float rw = __fadd_rn(__fmul_rn(dx, dvx), __fmul_rn(dy, dvy));
        if (rw < 0.0f && (j0 + jj) != self + i) {
          const float g2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
          const float den = -rw;
          if (!(g2 > __fmul_ru(best, den))) {
            const float t = __fdiv_rn(g2, den);
            if (t < best) best = t;
          }
        }
      }
    }
  }
  if (mine) p.d.dint[p.d.ilist_idx[i]] = best;
}

int launch_world_interaction(const Params *const *ps, uint32_t G, int64_t now, cudaStream_t s) {
  int n = 0;
  uint64_t most = 0;
  for (uint32_t r = 0; r < G; ++r) {
    if (ps[r]->n_kin == 0) continue;
    const int g = max(1, min(1184, ceil_div(max(ps[r]->n_local, ps[r]->n_kin), NT)));
    k_int_compact<<<g, NT, 0, s>>>(*ps[r], now);
    ++n;
    most = ps[r]->n_kin > most ? ps[r]->n_kin : most;
  }
  if (n == 0) return 0;
  const WArgs w = world_args(ps, G, now);
  k_kin_allgather<<<dim3(max(1, min(64, ceil_div(most, NT))), G, G), NT, 0, s>>>(w);
  ++n;
  for (uint32_t r = 0; r < G; ++r) {
    if (ps[r]->n_kin == 0) continue;
    k_pairmin_world<<<max(1, ceil_div(ps[r]->n_kin, NT)), NT, 0, s>>>(*ps[r]);
    ++n;
  }
  return n;
}

// §8(e) step 4, "all-gather of per-rank prefetch/evict id lists" merged into the global lists:
// rank r's entry i of a list (its shard's members in list order) sits in the global list at
//   i + sum over the other ranks r' of the entries of r' that precede it in list order,
// i.e. (prefetch, ascending (d, id)) r' < r: keys <= k, r' > r: keys < k; (evict, descending
// (d, id)) r' > r: keys >= k, r' < r: keys > k -- ranks own contiguous ascending id ranges.
// The keys are the distance bits, recomputed from the records by the definition (a1).
__device__ __forceinline__ uint32_t world_key(const Params &P, const uint4 *rec, uint32_t id, int64_t now) {
  const uint4 r = rec[id - (uint32_t)P.shard_begin];
  uint32_t st = 0;
  const float d = P.explicit_dist ? explicit_distance_of(r, st) : distance_of(r, now, P.hop_scale, P.d.dint, P.n_kin, st);
  return __float_as_uint(d);
}

__global__ void __launch_bounds__(NT) k_tp_keys(WArgs w) {
  const uint32_t r = blockIdx.y, lst = blockIdx.z;
  const Params &P = *w.r[r].pd;
  const uint32_t n = (uint32_t)P.d.header[lst == 0 ? H_N_PF : H_N_EV];
  const uint32_t *ids = lst == 0 ? P.d.pf_ids : P.d.ev_ids;
  uint32_t *key = lst == 0 ? P.d.tp_kpf : P.d.tp_kev;
  for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) key[i] = world_key(P, w.r[r].rec, ids[i], w.now);
}

// one entry per 8 lanes (lane g searches rank g's list), 128 entries per block
__global__ void __launch_bounds__(1024) k_tp_merge(WArgs w) {
  const uint32_t r = blockIdx.y, lst = blockIdx.z;
  const Params &P = *w.r[r].pd;
  const uint32_t n = (uint32_t)P.d.header[lst == 0 ? H_N_PF : H_N_EV];
  const uint32_t g = threadIdx.x & 7u;
  const uint32_t i = blockIdx.x * 128 + (threadIdx.x >> 3);
  if (blockIdx.x == 0 && r == 0 && lst == 0 && threadIdx.x < w.G) {  // merged counts into every rank
    unsigned long long npf = 0, nev = 0;
    for (uint32_t q = 0; q < w.G; ++q) {
      npf += w.r[q].pd->d.header[H_N_PF];
      nev += w.r[q].pd->d.header[H_N_EV];
    }
    unsigned long long *H = w.r[threadIdx.x].pd->d.tp_hdr;
    H[H_N_PF] = npf;
    H[H_N_EV] = nev;
    H[H_STATUS] = 0;
  }
  if (blockIdx.x * 128 >= n) return;  // (block-uniform)
  const bool on = i < n;
  uint32_t k = 0, id = 0;
  if (on) {
    k = (lst == 0 ? P.d.tp_kpf : P.d.tp_kev)[i];
    id = (lst == 0 ? P.d.pf_ids : P.d.ev_ids)[i];
  }
  uint32_t cnt = 0;
  if (on && g < w.G) {
    if (g == r) {
      cnt = i;
    } else {
      const Params &Q = *w.r[g].pd;
      const uint32_t m = (uint32_t)Q.d.header[lst == 0 ? H_N_PF : H_N_EV];
      const uint32_t *kq = lst == 0 ? Q.d.tp_kpf : Q.d.tp_kev;
      // count of the leading entries of rank g's list that precede (k, id): a prefix of its list
      const bool lower = g < r;
      uint32_t lo = 0, hi = m;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1, kk = kq[mid];
        const bool before = lst == 0 ? (lower ? kk <= k : kk < k) : (lower ? kk > k : kk >= k);
        if (before) lo = mid + 1;
        else hi = mid;
      }
      cnt = lo;
    }
  }
  cnt += __shfl_xor_sync(FULL, cnt, 1);
  cnt += __shfl_xor_sync(FULL, cnt, 2);
  cnt += __shfl_xor_sync(FULL, cnt, 4);
  if (!on || g >= w.G) return;
  // lane g writes rank g's copy (the all-gather's destination)
  const Dev &dd = w.r[g].pd->d;
  if (lst == 0) {
    dd.tp_pf[cnt] = id;
  } else {
    dd.tp_ev[cnt] = id;
    dd.tp_dirty[cnt] = (uint8_t)((w.r[r].rec[id - (uint32_t)P.shard_begin].z >> 4) & 1u);
  }
}

int launch_tp_merge(const Params *const *ps, uint32_t G, int64_t now, cudaStream_t s) {
  uint64_t most = 1;
  for (uint32_t r = 0; r < G; ++r) most = ps[r]->n_local > most ? ps[r]->n_local : most;
  const WArgs w = world_args(ps, G, now);
  k_tp_keys<<<dim3(max(1, min(148, ceil_div(most, NT))), G, 2), NT, 0, s>>>(w);
  k_tp_merge<<<dim3(ceil_div(most, 128), G, 2), 1024, 0, s>>>(w);
  return 2;
}

// after the expansion of the merged lists: this rank's header carries the world's page counts
// (its transfer moves slice `rank` of each listed page) and a pool shortage
__global__ void k_tp_finish(Params p) {
  const unsigned long long *T = p.d.tp_hdr;
  unsigned long long *H = p.d.header;
  H[H_N_D2H] = T[H_N_D2H];
  H[H_N_H2D] = T[H_N_H2D];
  H[H_POOL_HEAD] = T[H_POOL_HEAD];
  H[H_POOL_TAIL] = T[H_POOL_TAIL];
  if (T[H_STATUS] & ST_NO_PAGES) {
    H[H_STATUS] |= ST_NO_PAGES;
    p.d.state->status |= ST_NO_PAGES;
  }
}

int launch_tp_finish(const Params &p, cudaStream_t s) {
  k_tp_finish<<<1, 1, 0, s>>>(p);
  return 1;
}

// The collectives of the multi-kernel world > 1 path between ranks that share one
// device, each rank driven by its own host thread (SCALESIM_F_THREADS): out = reduction over the
// G ranks' buffers (kind 0: sum of u64, 1: min of u32), or the all-gather of one u64 per rank.
struct XIn {
  const void *in[FUSED_MAX_WORLD];
};
__global__ void __launch_bounds__(NT) k_xreduce(void *out, XIn x, uint32_t G, uint64_t n, int kind) {
  for (uint64_t i = blockIdx.x * (uint64_t)NT + threadIdx.x; i < n; i += (uint64_t)gridDim.x * NT) {
    if (kind == 0) {
      unsigned long long v = 0;
      for (uint32_t r = 0; r < G; ++r) v += static_cast<const unsigned long long *>(x.in[r])[i];
      static_cast<unsigned long long *>(out)[i] = v;
    } else {
      uint32_t v = 0xFFFFFFFFu;
      for (uint32_t r = 0; r < G; ++r) v = min(v, static_cast<const uint32_t *>(x.in[r])[i]);
      static_cast<uint32_t *>(out)[i] = v;
    }
  }
}
__global__ void k_xgather(unsigned long long *out, XIn x, uint32_t G) {
  if (threadIdx.x < G) out[threadIdx.x] = *static_cast<const unsigned long long *>(x.in[threadIdx.x]);
}

int launch_xreduce(void *out, const void *const *ins, uint32_t G, uint64_t n, int kind, cudaStream_t s) {
  XIn x = {};
  for (uint32_t r = 0; r < G; ++r) x.in[r] = ins[r];
  k_xreduce<<<max(1, min(64, ceil_div(n, NT))), NT, 0, s>>>(out, x, G, n, kind);
  return 1;
}
int launch_xgather(unsigned long long *out, const void *const *ins, uint32_t G, cudaStream_t s) {
  XIn x = {};
  for (uint32_t r = 0; r < G; ++r) x.in[r] = ins[r];
  k_xgather<<<1, 32, 0, s>>>(out, x, G);
  return 1;
}

}  // namespace ss

namespace ss {
// Incremental inputs (scalesim_stage_updates / scalesim_step_updates): the step's changed
// agent records scattered into the context's resident record array.  One thread per update;
// ids outside this shard are skipped and counted into *err (host-mapped, rare path).
__global__ void k_apply_updates(uint4 *rec, const uint32_t *ids, const uint4 *upd, uint32_t n, uint64_t shard_begin,
                                uint64_t n_local, uint32_t *err) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t a = (uint64_t)ids[i] - shard_begin;  // (ids below the shard wrap past n_local)
    if (a < n_local) rec[a] = upd[i];
    else atomicAdd(err, 1u);
  }
}
int launch_apply_updates(uint4 *rec, const uint32_t *ids, const uint4 *upd, uint32_t n, uint64_t shard_begin,
                         uint64_t n_local, uint32_t *err, cudaStream_t s) {
  if (n == 0) return 0;
  k_apply_updates<<<max(1, min(4 * 148, ceil_div(n, NT))), NT, 0, s>>>(rec, ids, upd, n, shard_begin, n_local, err);
  return 1;
}
}  // namespace ss

namespace ss {
// Host read-back of a step (scalesim_step_host / scalesim_step_updates): the header and both
// lists written straight into host-mapped pinned memory, then a completion word (the step's
// sequence number) the host polls instead of synchronising the stream.  Each CTA fences its
// writes at system scope before taking a ticket; the last CTA writes the word.
__global__ void k_readback(const unsigned long long *hdr, const uint32_t *pf, const uint32_t *ev,
                           unsigned long long *out_hdr, uint32_t *out_pf, uint32_t *out_ev,
                           volatile unsigned long long *done_word, unsigned long long seq, unsigned int *tickets) {
  const unsigned long long n_pf = hdr[H_N_PF], n_ev = hdr[H_N_EV];
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, ts = (uint64_t)gridDim.x * blockDim.x;
  if (t0 < 16) out_hdr[t0] = hdr[t0];
  // 16-byte stores (a warp writes 512 contiguous bytes of host memory): 4-byte stores over the
  // host link cost ~4x (measured: 15.8 us for C4's ~60 KB of lists, r02_v77)
  auto copy = [&](const uint32_t *src, uint32_t *dst, unsigned long long n) {
    const uint64_t n4 = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) ? 0 : n / 4;
    for (uint64_t i = t0; i < n4; i += ts) reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
    for (uint64_t i = 4 * n4 + t0; i < n; i += ts) dst[i] = src[i];
  };
  copy(pf, out_pf, n_pf);
  copy(ev, out_ev, n_ev);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(tickets, 1u) == gridDim.x - 1) {
    *tickets = 0u;  // (the next launch on this stream starts after this one)
    __threadfence_system();
    *done_word = seq;
  }
}
int launch_readback(const unsigned long long *hdr, const uint32_t *pf, const uint32_t *ev, unsigned long long *out_hdr,
                    uint32_t *out_pf, uint32_t *out_ev, unsigned long long *done_word, unsigned long long seq,
                    unsigned int *tickets, cudaStream_t s) {
  k_readback<<<32, 256, 0, s>>>(hdr, pf, ev, out_hdr, out_pf, out_ev, done_word, seq, tickets);
  return 1;
}
}  // namespace ss
