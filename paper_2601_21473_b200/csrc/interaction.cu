// interaction.cu — a1' (Eq. 2; readings R6, R7) with exact spatial pruning
// (NEXT #4): the participants (ACTING interaction agents) are bucketed into a uniform grid
// and every participant searches rings of cells outward from its own, stopping once no pair
// in the remaining rings can beat its running minimum.
//
// Why it is exact (R7: distances bit-identical to the all-pairs scan).  For a pair at gap
// |r| with relative velocity w, t = (r.r)/(-(r.w)) >= |r|/|w| >= |r|/(|v_i| + |v_j|)
// (Cauchy-Schwarz, triangle inequality), and the rounded quotient the scan computes is
// >= that bound x (1 - 13u), u = 2^-24.  A ring whose cells are all at least dmin away is
// skipped only when dmin > best x (|v_i| + vmax) x (1 + 1e-5), so every skipped pair's rounded
// quotient exceeds best and could not lower it.  best starts at D_action (the agent's
// distance is min(D_action, D_interaction), Eq. 1), so pairs that cannot matter for the
// distance are never computed.  Cell assignment and ring bounds are computed in double from
// the f32 coordinates, so a point lies in its cell up to double rounding (covered by the
// 1e-9 relative slack).  The per-pair arithmetic and the division filter are those of the
// all-pairs kernel (kernels.cu k_pairmin), so the minimum is the same rounded value.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "internal.h"

namespace ss {

constexpr int GT = 1024;  // threads of the single-block grid setup / scan kernels

__device__ __forceinline__ uint32_t cell_of(const GridHdr &g, float x, float y) {
  int cx = (int)floor(((double)x - g.xmin) / g.h), cy = (int)floor(((double)y - g.ymin) / g.h);
  cx = cx < 0 ? 0 : (cx >= (int)g.ncx ? (int)g.ncx - 1 : cx);
  cy = cy < 0 ? 0 : (cy >= (int)g.ncy ? (int)g.ncy - 1 : cy);
  return (uint32_t)cy * g.ncx + (uint32_t)cx;
}

// grid shape from the accumulated bounding box and speed (k_int_compact); re-arms the
// accumulators for the next step and clears the cell counters (one block)
__global__ void __launch_bounds__(GT) k_grid_setup(Params p) {
  __shared__ uint32_t s_nc;
  GridHdr *gp = reinterpret_cast<GridHdr *>(p.d.grid_hdr);
  if (threadIdx.x == 0) {
    GridHdr g = *gp;
    const uint32_t count = p.d.state->int_count;
    g.count = count;
    g.n_heavy = 0;
    const bool any = count > 0 && g.acc_x0 != 0x7FFFFFFF;
    g.xmin = any ? (double)fkey_inv(g.acc_x0) : 0.0;
    g.ymin = any ? (double)fkey_inv(g.acc_y0) : 0.0;
    const double ex = any ? (double)fkey_inv(g.acc_x1) - g.xmin : 0.0;
    const double ey = any ? (double)fkey_inv(g.acc_y1) - g.ymin : 0.0;
    const double e = fmax(ex, ey);
    uint32_t side = (uint32_t)floor(sqrt((double)count / 2.0));
    side = side < 1 ? 1 : (side > GRID_MAX_SIDE ? GRID_MAX_SIDE : side);
    g.h = e > 0.0 ? e / side * (1.0 + 1e-6) : 1.0;
    g.ncx = (uint32_t)fmin((double)side, floor(ex / g.h) + 1.0);
    g.ncy = (uint32_t)fmin((double)side, floor(ey / g.h) + 1.0);
    // the speed was rounded once in float (sqrtf): a relative margin covers it
    g.vmax = (double)__uint_as_float(g.acc_vmax) * (1.0 + 1e-6);
    g.acc_x0 = g.acc_y0 = 0x7FFFFFFF;
    g.acc_x1 = g.acc_y1 = (int32_t)0x80000000;
    g.acc_vmax = 0;
    *gp = g;
    s_nc = g.ncx * g.ncy;
  }
  __syncthreads();
  const uint32_t nc = s_nc;
  for (uint32_t c = threadIdx.x; c < ((nc + 3u) & ~3u); c += GT) p.d.cell_cnt[c] = 0;  // whole uint4 groups
}

__global__ void __launch_bounds__(NT) k_grid_count(Params p) {
  const GridHdr g = *reinterpret_cast<const GridHdr *>(p.d.grid_hdr);
  for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < g.count; i += gridDim.x * NT) {
    const float4 k = p.d.ilist_kin[i];
    const uint32_t c = cell_of(g, k.x, k.y);
    p.d.g_cell[i] = c;
    atomicAdd(&p.d.cell_cnt[c], 1u);
  }
}

// exclusive scan of the cell counts into cell_start (cell_start[ncells] = count); the counts
// become fill counters.  Thread t owns a contiguous run of cells (uint4 loads): one pass
// sums, a block scan, a second pass (L2-resident re-reads) writes.
__global__ void __launch_bounds__(GT) k_grid_scan(Params p) {
  static_assert(GRID_MAX_SIDE * GRID_MAX_SIDE <= 16 * GT, "at most 4 uint4 cell groups per thread");
  const GridHdr g = *reinterpret_cast<const GridHdr *>(p.d.grid_hdr);
  const uint32_t nc = g.ncx * g.ncy, n4 = (nc + 3) / 4;  // uint4 groups (counts beyond nc are 0)
  const uint32_t q0 = threadIdx.x * 4;
  const uint4 *src = reinterpret_cast<const uint4 *>(p.d.cell_cnt);
  uint4 v[4];
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = q0 + k < n4 ? src[q0 + k] : make_uint4(0, 0, 0, 0);
    sum += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  __shared__ uint32_t tot;
  uint32_t ex = block_excl_scan<uint32_t, GT>(sum, &tot);
  uint4 *dst = reinterpret_cast<uint4 *>(p.d.cell_start);
  uint4 *cnt = reinterpret_cast<uint4 *>(p.d.cell_cnt);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (q0 + k < n4) {
      uint4 o;
      o.x = ex;
      o.y = o.x + v[k].x;
      o.z = o.y + v[k].y;
      o.w = o.z + v[k].z;
      ex = o.w + v[k].w;
      dst[q0 + k] = o;
      cnt[q0 + k] = make_uint4(0, 0, 0, 0);
    }
  }
  if (threadIdx.x == 0) p.d.cell_start[nc] = g.count;
}

__global__ void __launch_bounds__(NT) k_grid_scatter(Params p) {
  const GridHdr g = *reinterpret_cast<const GridHdr *>(p.d.grid_hdr);
  for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < g.count; i += gridDim.x * NT) {
    const uint32_t c = p.d.g_cell[i];
    const uint32_t s = p.d.cell_start[c] + atomicAdd(&p.d.cell_cnt[c], 1u);
    p.d.g_kin[s] = p.d.ilist_kin[i];
    p.d.g_ent[s] = i;
  }
}

// Candidates j of participant (ki, slot s) in sorted slots [lo, hi): the pair arithmetic of
// the all-pairs kernel (kernels.cu k_pairmin) and its division filter.
__device__ __forceinline__ void scan_range(const float4 *__restrict__ gk, uint32_t lo, uint32_t hi, uint32_t s,
                                           float4 ki, float &best) {
#pragma unroll 4
  for (uint32_t j = lo; j < hi; ++j) {
    const float4 kj = gk[j];
    const float dx = __fsub_rn(kj.x, ki.x);
    const float dy = __fsub_rn(kj.y, ki.y);
    const float dvx = __fsub_rn(kj.z, ki.z);
    const float dvy = __fsub_rn(kj.w, ki.w);
    const float rw = __fadd_rn(__fmul_rn(dx, dvx), __fmul_rn(dy, dvy));
    if (rw < 0.0f && j != s) {
      const float g2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
      const float den = -rw;
      if (!(g2 > __fmul_ru(best, den))) {
        const float t = __fdiv_rn(g2, den);
        if (t < best) best = t;
      }
    }
  }
}

// The same over a range split across the lanes of a warp (lane l: lo + l, lo + l + 32, ...).
__device__ __forceinline__ void scan_range_lanes(const float4 *__restrict__ gk, uint32_t lo, uint32_t hi, uint32_t s,
                                                 float4 ki, float &best, uint32_t lane) {
  for (uint32_t j = lo + lane; j < hi; j += 32) {
    const float4 kj = gk[j];
    const float dx = __fsub_rn(kj.x, ki.x);
    const float dy = __fsub_rn(kj.y, ki.y);
    const float dvx = __fsub_rn(kj.z, ki.z);
    const float dvy = __fsub_rn(kj.w, ki.w);
    const float rw = __fadd_rn(__fmul_rn(dx, dvx), __fmul_rn(dy, dvy));
    if (rw < 0.0f && j != s) {
      const float g2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
      const float den = -rw;
      if (!(g2 > __fmul_ru(best, den))) {
        const float t = __fdiv_rn(g2, den);
        if (t < best) best = t;
      }
    }
  }
}

// One participant per thread (cell order).  Square windows of Chebyshev radius 0, 1, 2, 4, ...
// around its cell; cells are row-major and slots follow cell order, so the cells of one row
// of a window are one contiguous slot range (two loads for its bounds).  After window R the
// search stops once the distance to the outside of the window exceeds best x (|v_i| + vmax).
constexpr int PT = 64;  // threads per block: ~one participant per 32 spread over every SM
constexpr int R_THREAD = 2;  // windows beyond this radius continue warp-wide (k_grid_heavy)
__global__ void __launch_bounds__(PT) k_grid_pairmin(Params p) {
  const GridHdr g = *reinterpret_cast<const GridHdr *>(p.d.grid_hdr);
  const float4 *__restrict__ gk = p.d.g_kin;
  const uint32_t *__restrict__ cs = p.d.cell_start;
  const int ncx = (int)g.ncx, ncy = (int)g.ncy;
  for (uint32_t s = blockIdx.x * PT + threadIdx.x; s < g.count; s += gridDim.x * PT) {
    const float4 ki = gk[s];
    const uint32_t e = p.d.g_ent[s];
    float best = p.d.ilist_dact[e];  // D_action: pairs that cannot go below it do not matter (Eq. 1)
    const double xi = (double)ki.x, yi = (double)ki.y;
    const double vsum = ((double)sqrtf(ki.z * ki.z + ki.w * ki.w) * (1.0 + 1e-6) + g.vmax) * (1.0 + 1e-5);
    int cx = (int)floor((xi - g.xmin) / g.h), cy = (int)floor((yi - g.ymin) / g.h);
    cx = cx < 0 ? 0 : (cx >= ncx ? ncx - 1 : cx);
    cy = cy < 0 ? 0 : (cy >= ncy ? ncy - 1 : cy);
    const uint32_t own = (uint32_t)cy * g.ncx + (uint32_t)cx;
    scan_range(gk, cs[own], cs[own + 1], s, ki, best);
    const int rcap = max(max(cx, ncx - 1 - cx), max(cy, ncy - 1 - cy));  // window covering the grid
    int R = 0;
    bool done = false;
    while (R < rcap) {
      // distance from the participant to the outside of window R
      const double dl = xi - (g.xmin + (double)(cx - R) * g.h), dr = (g.xmin + (double)(cx + R + 1) * g.h) - xi;
      const double dd = yi - (g.ymin + (double)(cy - R) * g.h), du = (g.ymin + (double)(cy + R + 1) * g.h) - yi;
      const double dmin = fmin(fmin(dl, dr), fmin(dd, du)) - 1e-9 * g.h;
      if (dmin > 0.0 && dmin * (1.0 - 1e-9) > (double)best * vsum) {
        done = true;
        break;
      }
      if (R >= R_THREAD) break;  // a long search: handed to a warp
      const int nR = R == 0 ? 1 : min(2 * R, rcap);
      const int y0 = max(cy - nR, 0), y1 = min(cy + nR, ncy - 1);
      const int xa = max(cx - nR, 0), xb = min(cx + nR, ncx - 1);
      for (int y = y0; y <= y1; ++y) {
        const uint32_t row = (uint32_t)y * g.ncx;
        if (y < cy - R || y > cy + R) {  // a new row: the window's full width
          scan_range(gk, cs[row + xa], cs[row + xb + 1], s, ki, best);
        } else {  // a row of window R: the two new side segments
          if (xa <= cx - R - 1) scan_range(gk, cs[row + xa], cs[row + cx - R], s, ki, best);
          if (cx + R + 1 <= xb) scan_range(gk, cs[row + cx + R + 1], cs[row + xb + 1], s, ki, best);
        }
      }
      R = nR;
    }
    p.d.dint[p.d.ilist_idx[e]] = best;  // final, or the running minimum the warp continues from
    if (!done && R < rcap) {
      GridHdr *gp = reinterpret_cast<GridHdr *>(p.d.grid_hdr);
      p.d.heavy[atomicAdd(&gp->n_heavy, 1u)] = s;
    }
  }
}

// The searches that outgrew window R_THREAD, one warp each: every row range of the next
// windows is split over the lanes (coalesced); the lanes' minima are combined before each
// stopping test.  A lane's filter uses its own running minimum, which is never below the
// warp's, so it only skips quotients that cannot become the final minimum.
__global__ void __launch_bounds__(256) k_grid_heavy(Params p) {
  const GridHdr g = *reinterpret_cast<const GridHdr *>(p.d.grid_hdr);
  const float4 *__restrict__ gk = p.d.g_kin;
  const uint32_t *__restrict__ cs = p.d.cell_start;
  const int ncx = (int)g.ncx, ncy = (int)g.ncy;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp_g = (blockIdx.x * 256 + threadIdx.x) / 32, n_warps = gridDim.x * 256 / 32;
  for (uint32_t hi = warp_g; hi < g.n_heavy; hi += n_warps) {
    const uint32_t s = p.d.heavy[hi];
    const float4 ki = gk[s];
    const uint32_t e = p.d.g_ent[s];
    float *out = p.d.dint + p.d.ilist_idx[e];
    float best = *out;
    const double xi = (double)ki.x, yi = (double)ki.y;
    const double vsum = ((double)sqrtf(ki.z * ki.z + ki.w * ki.w) * (1.0 + 1e-6) + g.vmax) * (1.0 + 1e-5);
    int cx = (int)floor((xi - g.xmin) / g.h), cy = (int)floor((yi - g.ymin) / g.h);
    cx = cx < 0 ? 0 : (cx >= ncx ? ncx - 1 : cx);
    cy = cy < 0 ? 0 : (cy >= ncy ? ncy - 1 : cy);
    const int rcap = max(max(cx, ncx - 1 - cx), max(cy, ncy - 1 - cy));
    int R = R_THREAD;
    while (R < rcap) {
      best = __uint_as_float(__reduce_min_sync(0xFFFFFFFFu, __float_as_uint(best)));  // d >= 0: bits order
      const double dl = xi - (g.xmin + (double)(cx - R) * g.h), dr = (g.xmin + (double)(cx + R + 1) * g.h) - xi;
      const double dd = yi - (g.ymin + (double)(cy - R) * g.h), du = (g.ymin + (double)(cy + R + 1) * g.h) - yi;
      const double dmin = fmin(fmin(dl, dr), fmin(dd, du)) - 1e-9 * g.h;
      if (dmin > 0.0 && dmin * (1.0 - 1e-9) > (double)best * vsum) break;
      const int nR = min(2 * R, rcap);
      const int y0 = max(cy - nR, 0), y1 = min(cy + nR, ncy - 1);
      const int xa = max(cx - nR, 0), xb = min(cx + nR, ncx - 1);
      for (int y = y0; y <= y1; ++y) {
        const uint32_t row = (uint32_t)y * g.ncx;
        if (y < cy - R || y > cy + R) {
          const uint32_t lo = cs[row + xa], hi2 = cs[row + xb + 1];
          scan_range_lanes(gk, lo, hi2, s, ki, best, lane);
        } else {
          if (xa <= cx - R - 1) scan_range_lanes(gk, cs[row + xa], cs[row + cx - R], s, ki, best, lane);
          if (cx + R + 1 <= xb) scan_range_lanes(gk, cs[row + cx + R + 1], cs[row + xb + 1], s, ki, best, lane);
        }
      }
      R = nR;
    }
    best = __uint_as_float(__reduce_min_sync(0xFFFFFFFFu, __float_as_uint(best)));
    if (lane == 0) *out = best;
  }
}

int launch_grid_pairmin(const Params &p, cudaStream_t s, int grid) {
  const int g = min(grid, max(1, (int)((p.n_kin + NT - 1) / NT)));
  k_grid_setup<<<1, GT, 0, s>>>(p);
  k_grid_count<<<g, NT, 0, s>>>(p);
  k_grid_scan<<<1, GT, 0, s>>>(p);
  k_grid_scatter<<<g, NT, 0, s>>>(p);
  k_grid_pairmin<<<max(1, (int)((p.n_kin + PT - 1) / PT)), PT, 0, s>>>(p);
  k_grid_heavy<<<grid * 2, 256, 0, s>>>(p);
  return 6;
}

}  // namespace ss
