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
constexpr int kLutEntryBytes = 8;

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
// q(x) only has to be monotone non-decreasing (grid values and records go
// through the same function; values sharing a bucket are compared exactly
// in f64), so it is computed in f32: x rounded to f32 (monotone), minus the
// grid's low end, times kLutBuckets / range (each rounded step monotone),
// clamped to [0, kLutBuckets - 1] by fmaxf / fminf (NaN -> 0: NaN >= g is
// false for every g, so its bin 0 is exact; +-inf saturate), and rounded to
// an integer with the 2^23 magic-number add (exact below 2^22) instead of a
// conversion instruction.  An entry holds the bucket's first grid index and
// how many grid values it holds (usually 0 or 1), so a lookup is one LDS,
// one f64 LDS and one f64 compare.
__device__ __forceinline__ int bucket_of_f(float xf, float lo, float scale) {
  float y = __fmul_rn(__fsub_rn(xf, lo), scale);
  y = fminf(fmaxf(y, 0.f), (float)(kLutBuckets - 1));
  return __float_as_int(__fadd_rn(y, 8388608.f)) - 0x4B000000;
}
__device__ __forceinline__ int bucket_of(double x, float lo, float scale) {
  return bucket_of_f(__double2float_rn(x), lo, scale);
}

// An entry is {first grid index | count << 16, f32 of the bucket's first
// grid value}: with one value in the bucket (the usual case) the f32
// compare decides unless the two round to the same f32 (monotone rounding:
// xf > gf implies x > g, xf < gf implies x < g), and only then, or for NaN
// or several values, the exact f64 compare runs.
template <int D>
struct BinTables {
  const double* grid;  // smem, concatenated grids of models 0..D-1
  const uint2* lut;    // smem, [D][kLutBuckets]
  int goff[D];
  float lo[D], scale[D];

  __device__ __forceinline__ int bin(int j, double x) const {
    const float xf = __double2float_rn(x);
    const uint2 e = lut[j * kLutBuckets + bucket_of_f(xf, lo[j], scale[j])];
    const int lb = (int)(e.x & 0xffffu), c = (int)(e.x >> 16);
    const float gf = __uint_as_float(e.y);
    int b = lb + ((c != 0 && xf > gf) ? 1 : 0);
    if (c > 1 || (c == 1 && !(xf > gf) && !(xf < gf))) b = lb + upper_count(grid + goff[j] + lb, c, x);
    return b;
  }
};

// Build the tables in shared memory; every thread of the block calls it.
// s_grid must already hold the D grids (loaded by the caller, so it can
// order the grid loads ahead of its own record loads) and be synchronised;
// s_lut holds D * kLutBuckets 8-byte entries (kLutEntryBytes); the first
// half serves as 32-bit scratch until the entries are written.  Every thread derives lo / scale
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
                                                         void* s_lut_mem) {
  uint32_t* s_lut = static_cast<uint32_t*>(s_lut_mem);
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
    t.lo[j] = __double2float_rn(g[0]);
    const float range = __fsub_rn(__double2float_rn(g[n - 1]), t.lo[j]);
    t.scale[j] = range > 0.f ? __fdiv_rn((float)kLutBuckets, range) : 0.f;
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
    float lo = t.lo[0], scale = t.scale[0];
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
  // across warps: warp j turns model j's warp minima into "minimum over the
  // warps after this one" (a suffix minimum by shuffles, not a serial loop)
  if (warp < D) {
    const uint32_t m = lane < nwarps ? s_wmin[warp][lane] : 0xffffffffu;
    uint32_t incl = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_down_sync(0xffffffffu, incl, o);
      if (lane + o < 32) incl = min(incl, y);
    }
    const uint32_t after = __shfl_down_sync(0xffffffffu, incl, 1);
    __syncwarp();
    if (lane < nwarps) s_wmin[warp][lane] = lane == 31 ? 0xffffffffu : after;
  }
  __syncthreads();
  uint2 entry[D][per];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const uint32_t after = min(tmin[j], s_wmin[j][warp]);
    // lb(q) for the thread's buckets, lb of the bucket after the last
    uint32_t lb[per + 1];
    lb[per] = min(after, (uint32_t)glen[j]);
#pragma unroll
    for (int q = 0; q < per; ++q) lb[q] = min(v[j][q], after);
#pragma unroll
    for (int q = 0; q < per; ++q) {
      const uint32_t c = lb[q + 1] - lb[q];
      const float gf = c ? __double2float_rn(s_grid[t.goff[j] + lb[q]]) : 0.f;
      entry[j][q] = make_uint2(lb[q] | (c << 16), __float_as_uint(gf));
    }
  }
  __syncthreads();  // every scratch word is read: the entries overwrite them
  uint2* s_entry = static_cast<uint2*>(s_lut_mem);
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int q = 0; q < per; ++q) s_entry[j * kLutBuckets + q0 + q] = entry[j][q];
  __syncthreads();
  t.grid = s_grid;
  t.lut = s_entry;
  return t;
}

}  // namespace gs
