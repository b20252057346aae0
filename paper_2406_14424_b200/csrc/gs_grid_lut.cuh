// gs_grid_lut.cuh — threshold-grid bin lookup shared by the grid-sweep
// histogram kernels (gs_sweep.cu, gs_grid4.cu).
//
// A record's bin for model j is b_j = #{g in G_j : g <= cert[r, j]}: then
// cert >= G_j[k] <=> b_j > k, the inclusive gate of the reference walk
// (/root/reference/pkg/src/gearserve/kernels.py:50-52).
//
// Per CTA, every forwarding model's grid is bucketed by a monotone f64 map
// q(x) onto kLutBuckets buckets.  Grid values with q(g) < q(x) are all <= x
// and those with q(g) > q(x) are all > x, so the exact count lies in [lb, ub)
// of x's bucket and only the grid values sharing the bucket (usually none or
// one) are compared.  This replaces a 7-step binary search of bank-conflicted
// 64-bit shared loads per model.
#pragma once

#include "gs_common.cuh"

namespace gs {

constexpr int kLutBuckets = 2048;

__device__ __forceinline__ int lut_bucket(double x, double lo, double hi, double scale) {
  if (!(x >= lo)) return 0;  // below the grid (or NaN)
  if (x >= hi) return kLutBuckets - 1;
  const int q = (int)((x - lo) * scale);
  return q > kLutBuckets - 1 ? kLutBuckets - 1 : q;
}

// #{g[i] <= x} for strictly increasing g (n >= 1).  Branch-free: the trip
// count depends on n only, so a warp never diverges in the search.
__device__ __forceinline__ int upper_count(const double* g, int n, double x) {
  int base = 0, len = n;
  while (len > 1) {
    const int half = len >> 1;
    base = (g[base + half - 1] <= x) ? base + half : base;
    len -= half;
  }
  return base + (g[base] <= x ? 1 : 0);
}

// Shared-memory bin tables of D models: the grids (f64) and per model one
// bucket table of (lb | ub << 16) entries.
struct BinTables {
  const double* grid;     // smem, concatenated grids
  const uint32_t* lut;    // smem, [D][kLutBuckets]
  const int32_t* goff;    // grid offsets (kernel params)
  double lo[GS_MAX_MODELS], hi[GS_MAX_MODELS], scale[GS_MAX_MODELS];

  __device__ __forceinline__ int bin(int j, double x) const {
    const uint32_t e = lut[j * kLutBuckets + lut_bucket(x, lo[j], hi[j], scale[j])];
    const int lb = (int)(e & 0xffffu), ub = (int)(e >> 16);
    return lb + (ub > lb ? upper_count(grid + goff[j] + lb, ub - lb, x) : 0);
  }
};

// Build the bin tables of models 0..D-1 in shared memory.  Every thread of
// the block must call it (it synchronises).  s_grid holds n_grid doubles,
// s_lut D * kLutBuckets words, s_par 3 * D doubles.  THREADS = blockDim.x.
template <int THREADS>
__device__ __forceinline__ BinTables build_bin_tables(const double* grids, const int32_t* goff,
                                                      const int32_t* glen, int D, int n_grid,
                                                      double* s_grid, uint32_t* s_lut,
                                                      double* s_par) {
  static_assert(kLutBuckets % THREADS == 0 || THREADS % kLutBuckets == 0, "bucket split");
  for (int i = threadIdx.x; i < n_grid; i += THREADS) s_grid[i] = grids[i];
  for (int i = threadIdx.x; i < D * kLutBuckets; i += THREADS) s_lut[i] = 0u;
  __syncthreads();
  if ((int)threadIdx.x < D) {
    const int j = threadIdx.x;
    const double* g = s_grid + goff[j];
    const int n = glen[j];
    s_par[j] = g[0];
    s_par[GS_MAX_MODELS + j] = g[n - 1];
    s_par[2 * GS_MAX_MODELS + j] = n > 1 ? (double)kLutBuckets / (g[n - 1] - g[0]) : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < D; ++j) {
    const double lo = s_par[j], hi = s_par[GS_MAX_MODELS + j], sc = s_par[2 * GS_MAX_MODELS + j];
    for (int i = threadIdx.x; i < glen[j]; i += THREADS)
      atomicAdd(s_lut + j * kLutBuckets + lut_bucket(s_grid[goff[j] + i], lo, hi, sc), 1u);
  }
  __syncthreads();
  // per model: exclusive scan of the bucket counts -> (lb, ub), whole block
  {
    __shared__ uint32_t s_wsum[THREADS / 32];
    constexpr int per = kLutBuckets >= THREADS ? kLutBuckets / THREADS : 1;
    const int warp = threadIdx.x >> 5, lane = (int)lane_id();
    for (int j = 0; j < D; ++j) {
      uint32_t* L = s_lut + j * kLutBuckets + threadIdx.x * per;
      const bool own = (int)threadIdx.x * per < kLutBuckets;
      uint32_t c[per], tot = 0;
#pragma unroll
      for (int q = 0; q < per; ++q) {
        c[q] = own ? L[q] : 0u;
        tot += c[q];
      }
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_wsum[warp] = incl;
      __syncthreads();
      uint32_t run = incl - tot;
      for (int w = 0; w < warp; ++w) run += s_wsum[w];
      if (own) {
#pragma unroll
        for (int q = 0; q < per; ++q) {
          L[q] = run | ((run + c[q]) << 16);
          run += c[q];
        }
      }
      __syncthreads();
    }
  }
  BinTables t;
  t.grid = s_grid;
  t.lut = s_lut;
  t.goff = goff;
#pragma unroll
  for (int j = 0; j < GS_MAX_MODELS; ++j) {
    t.lo[j] = j < D ? s_par[j] : 0.0;
    t.hi[j] = j < D ? s_par[GS_MAX_MODELS + j] : 0.0;
    t.scale[j] = j < D ? s_par[2 * GS_MAX_MODELS + j] : 0.0;
  }
  return t;
}

}  // namespace gs
