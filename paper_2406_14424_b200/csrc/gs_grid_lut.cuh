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

// Shared-memory bin tables of D models (four-model path).  The bucket map
// is one clamp of a truncated affine f64 map: monotone non-decreasing in x
// (each rounded step is), NaN -> bucket 0 (cvt.rzi of NaN is 0, and NaN >=
// g is false for every g, so its bin 0 is exact), +-inf saturate.  An entry
// holds the bucket's first grid index and how many grid values it holds
// (usually 0 or 1), so a lookup is one LDS plus at most one f64 compare.
__device__ __forceinline__ int bucket_of(double x, double lo, double scale) {
  const int q = (int)__dmul_rn(__dadd_rn(x, -lo), scale);
  return min(max(q, 0), kLutBuckets - 1);
}

template <int D>
struct BinTables {
  const double* grid;   // smem, concatenated grids of models 0..D-1
  const uint32_t* lut;  // smem, [D][kLutBuckets]: first index | count << 16
  int goff[D];
  double lo[D], scale[D];

  __device__ __forceinline__ int bin(int j, double x) const {
    const uint32_t e = lut[j * kLutBuckets + bucket_of(x, lo[j], scale[j])];
    const int lb = (int)(e & 0xffffu), c = (int)(e >> 16);
    const double* g = grid + goff[j] + lb;
    if (c == 0) return lb;
    if (c == 1) return lb + (g[0] <= x ? 1 : 0);
    return lb + upper_count(g, c, x);
  }
};

// Build the tables in shared memory; every thread of the block calls it (two
// barriers).  s_grid holds the D grids, s_lut D * kLutBuckets words.  Every
// thread derives lo / scale itself.  Per model, a thread owns kLutBuckets /
// THREADS consecutive buckets: one binary search (over the monotone bucket
// index of the grid values) finds the first grid index of its first bucket,
// then it walks its buckets and the grid values inside them.  The work is
// balanced however unevenly the grid values fall into buckets.
template <int D, int THREADS>
__device__ __forceinline__ BinTables<D> build_bin_tables(const double* grids, const int32_t* glen,
                                                         double* s_grid, uint32_t* s_lut) {
  static_assert(kLutBuckets % THREADS == 0, "bucket split");
  constexpr int per = kLutBuckets / THREADS;
  BinTables<D> t;
  int n_grid = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    t.goff[j] = n_grid;
    n_grid += glen[j];
  }
  for (int i = threadIdx.x; i < n_grid; i += THREADS) s_grid[i] = grids[i];
  __syncthreads();
  const int q0 = threadIdx.x * per;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double* g = s_grid + t.goff[j];
    const int n = glen[j];
    const double lo = g[0];
    const double scale = n > 1 ? (double)kLutBuckets / (g[n - 1] - g[0]) : 0.0;
    t.lo[j] = lo;
    t.scale[j] = scale;
    // k = #{grid values whose bucket < q0}
    int k = 0, len = n;
    while (len > 0) {
      const int half = len >> 1;
      if (bucket_of(g[k + half], lo, scale) < q0) {
        k += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    uint32_t* L = s_lut + j * kLutBuckets;
#pragma unroll
    for (int q = q0; q < q0 + per; ++q) {
      int c = 0;
      while (k + c < n && bucket_of(g[k + c], lo, scale) == q) ++c;
      L[q] = (uint32_t)k | ((uint32_t)c << 16);
      k += c;
    }
  }
  __syncthreads();
  t.grid = s_grid;
  t.lut = s_lut;
  return t;
}

}  // namespace gs
