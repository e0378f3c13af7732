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

struct GridHdr {
  double xmin, ymin, h, vmax;
  uint32_t ncx, ncy, count, pad;
};

__device__ __forceinline__ uint32_t cell_of(const GridHdr &g, float x, float y) {
  int cx = (int)floor(((double)x - g.xmin) / g.h), cy = (int)floor(((double)y - g.ymin) / g.h);
  cx = cx < 0 ? 0 : (cx >= (int)g.ncx ? (int)g.ncx - 1 : cx);
  cy = cy < 0 ? 0 : (cy >= (int)g.ncy ? (int)g.ncy - 1 : cy);
  return (uint32_t)cy * g.ncx + (uint32_t)cx;
}

// bounding box, max speed, grid shape; clears the cell counters (one block)
__global__ void __launch_bounds__(GT) k_grid_setup(Params p) {
  __shared__ double red[4][GT / 32];
  __shared__ GridHdr sg;
  const uint32_t count = p.d.state->int_count;
  double x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY, vm = 0.0;
  for (uint32_t i = threadIdx.x; i < count; i += GT) {
    const float4 k = p.d.ilist_kin[i];
    x0 = fmin(x0, (double)k.x);
    y0 = fmin(y0, (double)k.y);
    x1 = fmax(x1, (double)k.x);
    y1 = fmax(y1, (double)k.y);
    vm = fmax(vm, sqrt((double)k.z * k.z + (double)k.w * k.w));
  }
  double v[4] = {x0, y0, -x1, -y1};
  for (int q = 0; q < 4; ++q)
    for (int o = 16; o > 0; o >>= 1) v[q] = fmin(v[q], __shfl_xor_sync(FULL, v[q], o));
  for (int o = 16; o > 0; o >>= 1) vm = fmax(vm, __shfl_xor_sync(FULL, vm, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double vmr[GT / 32];
  if (lane == 0) {
    for (int q = 0; q < 4; ++q) red[q][warp] = v[q];
    vmr[warp] = vm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < GT / 32; ++w) {
      for (int q = 0; q < 4; ++q) red[q][0] = fmin(red[q][0], red[q][w]);
      vmr[0] = fmax(vmr[0], vmr[w]);
    }
    GridHdr g;
    g.count = count;
    g.xmin = count ? red[0][0] : 0.0;
    g.ymin = count ? red[1][0] : 0.0;
    const double ex = count ? -red[2][0] - g.xmin : 0.0, ey = count ? -red[3][0] - g.ymin : 0.0;
    const double e = fmax(ex, ey);
    uint32_t side = (uint32_t)floor(sqrt((double)count / 2.0));
    side = side < 1 ? 1 : (side > GRID_MAX_SIDE ? GRID_MAX_SIDE : side);
    g.h = e > 0.0 ? e / side * (1.0 + 1e-6) : 1.0;
    g.ncx = (uint32_t)fmin((double)side, floor(ex / g.h) + 1.0);
    g.ncy = (uint32_t)fmin((double)side, floor(ey / g.h) + 1.0);
    g.vmax = vmr[0] * (1.0 + 1e-6);
    g.pad = 0;
    sg = g;
    *reinterpret_cast<GridHdr *>(p.d.grid_hdr) = g;
  }
  __syncthreads();
  const uint32_t nc = sg.ncx * sg.ncy;
  for (uint32_t c = threadIdx.x; c < nc; c += GT) p.d.cell_cnt[c] = 0;
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
// become fill counters
__global__ void __launch_bounds__(GT) k_grid_scan(Params p) {
  const GridHdr g = *reinterpret_cast<const GridHdr *>(p.d.grid_hdr);
  const uint32_t nc = g.ncx * g.ncy;
  const uint32_t per = (nc + GT - 1) / GT, c0 = threadIdx.x * per;
  uint32_t sum = 0;
  for (uint32_t c = c0; c < c0 + per && c < nc; ++c) sum += p.d.cell_cnt[c];
  __shared__ uint32_t tot;
  uint32_t ex = block_excl_scan<uint32_t, GT>(sum, &tot);
  for (uint32_t c = c0; c < c0 + per && c < nc; ++c) {
    const uint32_t v = p.d.cell_cnt[c];
    p.d.cell_start[c] = ex;
    ex += v;
    p.d.cell_cnt[c] = 0;
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

// one participant per thread (cell order: neighbouring threads search overlapping cells)
__global__ void __launch_bounds__(NT) k_grid_pairmin(Params p) {
  const GridHdr g = *reinterpret_cast<const GridHdr *>(p.d.grid_hdr);
  for (uint32_t s = blockIdx.x * NT + threadIdx.x; s < g.count; s += gridDim.x * NT) {
    const float4 ki = p.d.g_kin[s];
    const uint32_t e = p.d.g_ent[s];
    float best = p.d.ilist_dact[e];  // D_action: pairs that cannot go below it do not matter (Eq. 1)
    const double si = sqrt((double)ki.z * ki.z + (double)ki.w * ki.w);
    const double vsum = (si + g.vmax) * (1.0 + 1e-5);
    const int cx = (int)floor(((double)ki.x - g.xmin) / g.h), cy = (int)floor(((double)ki.y - g.ymin) / g.h);
    const int ccx = cx < 0 ? 0 : (cx >= (int)g.ncx ? (int)g.ncx - 1 : cx);
    const int ccy = cy < 0 ? 0 : (cy >= (int)g.ncy ? (int)g.ncy - 1 : cy);
    const int rmax = (int)max(g.ncx, g.ncy);
    for (int r = 0; r <= rmax; ++r) {
      if (r > 0) {
        // every cell of ring r lies beyond these four lines around the participant
        const double xi = (double)ki.x, yi = (double)ki.y;
        const double dl = xi - (g.xmin + (double)(ccx - r + 1) * g.h), dr = (g.xmin + (double)(ccx + r) * g.h) - xi;
        const double dd = yi - (g.ymin + (double)(ccy - r + 1) * g.h), du = (g.ymin + (double)(ccy + r) * g.h) - yi;
        const double dmin = fmin(fmin(dl, dr), fmin(dd, du)) - 1e-9 * g.h;
        if (dmin > 0.0 && dmin * (1.0 - 1e-9) > (double)best * vsum) break;
      }
      for (int y = ccy - r; y <= ccy + r; ++y) {
        if (y < 0 || y >= (int)g.ncy) continue;
        const bool edge_row = (y == ccy - r || y == ccy + r);
        for (int x = ccx - r; x <= ccx + r; x += (edge_row || r == 0) ? 1 : 2 * r) {
          if (x < 0 || x >= (int)g.ncx) continue;
          const uint32_t c = (uint32_t)y * g.ncx + (uint32_t)x;
          const uint32_t j1 = p.d.cell_start[c + 1];
          for (uint32_t j = p.d.cell_start[c]; j < j1; ++j) {
            if (j == s) continue;
            const float4 kj = p.d.g_kin[j];
            const float dx = __fsub_rn(kj.x, ki.x);
            const float dy = __fsub_rn(kj.y, ki.y);
            const float dvx = __fsub_rn(kj.z, ki.z);
            const float dvy = __fsub_rn(kj.w, ki.w);
            const float rw = __fadd_rn(__fmul_rn(dx, dvx), __fmul_rn(dy, dvy));
            if (rw < 0.0f) {
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
    }
    p.d.dint[p.d.ilist_idx[e]] = best;
  }
}

int launch_grid_pairmin(const Params &p, cudaStream_t s, int grid) {
  const int g = min(grid, max(1, (int)((p.n_kin + NT - 1) / NT)));
  k_grid_setup<<<1, GT, 0, s>>>(p);
  k_grid_count<<<g, NT, 0, s>>>(p);
  k_grid_scan<<<1, GT, 0, s>>>(p);
  k_grid_scatter<<<g, NT, 0, s>>>(p);
  k_grid_pairmin<<<max(1, (int)((p.n_kin + NT - 1) / NT)), NT, 0, s>>>(p);
  return 5;
}

}  // namespace ss
