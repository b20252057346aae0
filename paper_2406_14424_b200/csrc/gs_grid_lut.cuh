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
//
// The integer part is taken with the 2^52 magic-number trick instead of a
// f64 -> s32 conversion (the conversion unit is the slow path): y is first
// clamped to [-1, kLutBuckets] (NaN -> -1), so y + 2^52 is exact and its low
// mantissa bits are round-to-nearest(y) — a monotone map, which is all the
// bucketing needs (grid values and records go through the same function).
__device__ __forceinline__ int bucket_of(double x, double lo, double scale) {
  double y = __dmul_rn(__dadd_rn(x, -lo), scale);
  y = fmin(fmax(y, -1.0), (double)kLutBuckets);
  // low word of 2^52 + round(y) is round(y) (two's complement for y = -1)
  const int q = __double2loint(__dadd_rn(y, 4503599627370496.0));
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

// Build the tables in shared memory; every thread of the block calls it.
// s_grid must already hold the D grids (loaded by the caller, so it can
// order the grid loads ahead of its own record loads) and be synchronised;
// s_lut holds D * kLutBuckets words.  Every thread derives lo / scale
// itself.  Three steps, no serial loops over buckets or grid values:
//   1. every bucket's entry := n (empty);
//   2. one thread per grid value: the first value of each occupied bucket
//      writes its index there (the values are sorted, so the first of a
//      bucket is the one whose predecessor lies in a lower bucket);
//   3. per model a block-wide suffix minimum turns "first index of this
//      bucket or n" into lb(q) = first index of the first occupied bucket
//      >= q = #{values in buckets < q}; the entry is lb(q) | (lb(q+1) -
//      lb(q)) << 16.
template <int D, int THREADS>
__device__ __forceinline__ BinTables<D> build_bin_tables(const int32_t* glen, double* s_grid,
                                                         uint32_t* s_lut) {
  static_assert(kLutBuckets % THREADS == 0, "bucket split");
  constexpr int per = kLutBuckets / THREADS;
  constexpr int nwarps = THREADS / 32;
  __shared__ uint32_t s_wmin[D][nwarps];
  BinTables<D> t;
  int n_grid = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    t.goff[j] = n_grid;
    n_grid += glen[j];
    const double* g = s_grid + t.goff[j];
    const int n = glen[j];
    t.lo[j] = g[0];
    t.scale[j] = n > 1 ? (double)kLutBuckets / (g[n - 1] - g[0]) : 0.0;
  }
  const int q0 = threadIdx.x * per;
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int q = 0; q < per; ++q) s_lut[j * kLutBuckets + q0 + q] = (uint32_t)glen[j];
  __syncthreads();
  for (int i = threadIdx.x; i < n_grid; i += THREADS) {
    int j = 0;
#pragma unroll
    for (int q = 1; q < D; ++q) j += i >= t.goff[q] ? 1 : 0;
    // register arrays indexed by a runtime j would go to local memory
    int goff = t.goff[0];
    double lo = t.lo[0], scale = t.scale[0];
#pragma unroll
    for (int q = 1; q < D; ++q)
      if (j == q) {
        goff = t.goff[q];
        lo = t.lo[q];
        scale = t.scale[q];
      }
    const int k = i - goff;
    const int qk = bucket_of(s_grid[i], lo, scale);
    if (k == 0 || bucket_of(s_grid[i - 1], lo, scale) != qk) s_lut[j * kLutBuckets + qk] = (uint32_t)k;
  }
  __syncthreads();
  // suffix minimum over buckets, per model: thread-local (per buckets), then
  // warp (shuffles), then across warps (shared memory)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v[D][per], tmin[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    uint32_t m = 0xffffffffu;
#pragma unroll
    for (int q = per - 1; q >= 0; --q) {
      m = min(m, s_lut[j * kLutBuckets + q0 + q]);
      v[j][q] = m;  // suffix min within the thread's buckets
    }
    uint32_t incl = m;  // suffix min over lanes >= lane
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_down_sync(0xffffffffu, incl, o);
      if (lane + o < 32) incl = min(incl, y);
    }
    if (lane == 0) s_wmin[j][warp] = incl;
    uint32_t after = __shfl_down_sync(0xffffffffu, incl, 1);  // lanes > lane
    tmin[j] = lane == 31 ? 0xffffffffu : after;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < D; ++j) {
    uint32_t after = tmin[j];
    for (int w = warp + 1; w < nwarps; ++w) after = min(after, s_wmin[j][w]);
    // lb(q) for the thread's buckets, lb of the bucket after the last
    uint32_t lb[per + 1];
    lb[per] = min(after, (uint32_t)glen[j]);
#pragma unroll
    for (int q = 0; q < per; ++q) lb[q] = min(v[j][q], after);
#pragma unroll
    for (int q = 0; q < per; ++q) s_lut[j * kLutBuckets + q0 + q] = lb[q] | ((lb[q + 1] - lb[q]) << 16);
  }
  __syncthreads();
  t.grid = s_grid;
  t.lut = s_lut;
  return t;
}

}  // namespace gs
