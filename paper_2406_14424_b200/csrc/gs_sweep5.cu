// gs_sweep5.cu — grid sweep, five-model path (BASELINE configs[3], variant
// 4b: a 5-stage cascade over 100-level grids).
//
// Same algorithm and outputs as the general path (gs_sweep.cu: dominance
// counting over the threshold bins, every config scored exactly like
// _evaluate_numba, /root/reference/pkg/src/gearserve/kernels.py:39-62); the
// difference is how the 4-D prefix table F over (b0, b1, b2, b3) is formed.
// The general path histograms every record into a dense 1.7 GB table (mostly
// zeros for 1e5 records), prefixes it in place along each dimension (a slab
// pass and two strided column passes) and then reads it back to score: ~20
// GB of traffic for 5.9 GB of outputs.  Here F is never materialised:
//
//   w5_bin      records -> bins, a 4-byte key {b1, b2, b3, c4, c3, c2} and
//               the (b0, b1) slab; per-slab counts; the side table of models
//               0 and 1 (c0, c1 per (b0, b1)).
//   w5_scan     one CTA: slab offsets (exclusive scan), the side table's
//               inclusive 2-D prefix P, counters re-zeroed for the next build.
//   w5_scatter  keys counting-sorted by slab.
//   w5_slab     a CTA per b0 walks b1 = 0..g1 keeping the (b2, b3) plane of
//               all records with this b0 and b1' <= b1, prefixed along b2 and
//               b3, in registers (each record adds to the cells dominating
//               it); after each b1 the plane is stored as T[b0][b1]: T is F
//               without the prefix along b0 (1.7 GB written once).
//   w5_walk     (gs_grid_eval) a CTA per (k1, block of k2 rows) walks k0 =
//               0..g0 adding T[k0][k1][rows] to running sums in registers,
//               which are then F(k0, k1, k2, *): each full-cascade config
//               (k0, k1, k2, k3) is scored there (95% of the configs) and the
//               face cells (some index at "any") are written out for the
//               regular eval, which scores every other structure from them.
// Traffic: T written and read once (3.3 GB) plus the outputs.
#include "gs_sweep5.cuh"

namespace gs {
namespace {

constexpr int kW5SlabThreads = 256;  // slab-pass CTA bound (rows x 32)
constexpr int kW5Seg = 4;              // plane cells per slab-pass thread: a warp per row, j = lane + 32 m
constexpr int kW5SlabChunk = 512;      // slab records ranked per round
constexpr int kW5SlabStage = 4096;     // keys of one b0 staged in shared memory
constexpr int kW5MaxD1 = 255;
constexpr int kW5WalkWarps = 8;
constexpr int kW5RowsPerWarp = 1;
constexpr int kW5Rows = kW5WalkWarps * kW5RowsPerWarp;  // k2 rows per walk CTA
constexpr int kW5U = 4;                 // d3 <= 32 * kW5U
constexpr uint64_t kF21m = (1ull << 21) - 1;

__device__ __forceinline__ uint4 unpack_cell(uint64_t q, uint32_t c2) {
  return make_uint4((uint32_t)(q & kF21m), (uint32_t)((q >> 21) & kF21m), (uint32_t)(q >> 42), c2);
}
__device__ __forceinline__ uint64_t pack_cell(const uint4& v) {
  return (uint64_t)v.x | ((uint64_t)v.y << 21) | ((uint64_t)v.z << 42);
}

// #{g[i] <= x} for strictly increasing g (n >= 1)
__device__ __forceinline__ int bin_of(const double* g, int n, double x) {
  int base = 0, len = n;
  while (len > 1) {
    const int half = len >> 1;
    base = (g[base + half - 1] <= x) ? base + half : base;
    len -= half;
  }
  return base + (g[base] <= x ? 1 : 0);
}

struct W5BinArgs {
  const double* cert;
  const uint8_t* corr;
  int64_t n_rec;
  const double* grids;
  int32_t goff[4], glen[4];
  int32_t d1;
  uint64_t* tmp;   // [n_rec] slab << 32 | key
  uint32_t* cnt;   // [cells2] records per slab (zero on entry)
  uint32_t* HP;    // [cells2][2] c0, c1 per slab (zero on entry)
};

__global__ void __launch_bounds__(256) w5_bin_kernel(const __grid_constant__ W5BinArgs a) {
  __shared__ double s_g[4 * 256];
  const int ng = a.goff[3] + a.glen[3];
  for (int i = threadIdx.x; i < ng; i += blockDim.x) s_g[i] = a.grids[i];
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.n_rec;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double* x = a.cert + r * 5;
    const uint8_t* k = a.corr + r * 5;
    const int b0 = bin_of(s_g + a.goff[0], a.glen[0], __ldg(x + 0));
    const int b1 = bin_of(s_g + a.goff[1], a.glen[1], __ldg(x + 1));
    const int b2 = bin_of(s_g + a.goff[2], a.glen[2], __ldg(x + 2));
    const int b3 = bin_of(s_g + a.goff[3], a.glen[3], __ldg(x + 3));
    const uint32_t key = (uint32_t)b1 | ((uint32_t)b2 << 8) | ((uint32_t)b3 << 16) |
                         ((__ldg(k + 4) != 0) ? 1u << 24 : 0u) | ((__ldg(k + 3) != 0) ? 1u << 25 : 0u) |
                         ((__ldg(k + 2) != 0) ? 1u << 26 : 0u);
    const uint32_t slab = (uint32_t)b0 * (uint32_t)a.d1 + (uint32_t)b1;
    a.tmp[r] = ((uint64_t)slab << 32) | key;
    atomicAdd(a.cnt + slab, 1u);
    if (__ldg(k + 0)) atomicAdd(a.HP + 2 * slab, 1u);
    if (__ldg(k + 1)) atomicAdd(a.HP + 2 * slab + 1, 1u);
  }
}

// One CTA: exclusive scan of the slab counts (offsets and scatter cursors),
// the side table's inclusive prefix over (b0, b1), counters re-zeroed.
__global__ void __launch_bounds__(1024) w5_scan_kernel(uint32_t* cnt, uint32_t* off, uint32_t* cur,
                                                        uint32_t* HP, uint4* P, int d0, int d1) {
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const int cells = d0 * d1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int b = 0; b < cells; b += 1024) {
    const int i = b + threadIdx.x;
    const uint32_t v = i < cells ? cnt[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_w[lane] = w;
    }
    __syncthreads();
    const uint32_t excl = s_carry + (warp ? s_w[warp - 1] : 0u) + x - v;
    if (i < cells) {
      off[i] = excl;
      cur[i] = excl;
      cnt[i] = 0u;
    }
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[cells] = s_carry;
  // side table: inclusive prefix along b1 (a warp per row, shuffle scans)
  // then along b0 (a warp per column), in shared memory
  extern __shared__ uint32_t s_side[];  // [2][cells]: c0, c1
  uint32_t* s0 = s_side;
  uint32_t* s1 = s_side + cells;
  for (int i = threadIdx.x; i < cells; i += 1024) {
    s0[i] = HP[2 * i];
    s1[i] = HP[2 * i + 1];
    HP[2 * i] = 0u;
    HP[2 * i + 1] = 0u;
  }
  __syncthreads();
  for (int r = warp; r < d0; r += 32) {
    uint32_t a0 = 0, a1 = 0;
    for (int c = lane; c - lane < d1; c += 32) {
      uint32_t x0 = c < d1 ? s0[r * d1 + c] : 0u, x1 = c < d1 ? s1[r * d1 + c] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
        if (lane >= o) {
          x0 += y0;
          x1 += y1;
        }
      }
      x0 += a0;
      x1 += a1;
      if (c < d1) {
        s0[r * d1 + c] = x0;
        s1[r * d1 + c] = x1;
      }
      a0 = __shfl_sync(0xffffffffu, x0, 31);
      a1 = __shfl_sync(0xffffffffu, x1, 31);
    }
  }
  __syncthreads();
  for (int c = warp; c < d1; c += 32) {
    uint32_t a0 = 0, a1 = 0;
    for (int r = lane; r - lane < d0; r += 32) {
      uint32_t x0 = r < d0 ? s0[r * d1 + c] : 0u, x1 = r < d0 ? s1[r * d1 + c] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
        if (lane >= o) {
          x0 += y0;
          x1 += y1;
        }
      }
      x0 += a0;
      x1 += a1;
      if (r < d0) P[r * d1 + c] = make_uint4(x0, x1, 0u, 0u);
      a0 = __shfl_sync(0xffffffffu, x0, 31);
      a1 = __shfl_sync(0xffffffffu, x1, 31);
    }
  }
}

__global__ void __launch_bounds__(256) w5_scatter_kernel(const uint64_t* tmp, int64_t n_rec, uint32_t* cur,
                                                         uint32_t* keys) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rec;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t t = tmp[r];
    keys[atomicAdd(cur + (uint32_t)(t >> 32), 1u)] = (uint32_t)t;
  }
}

// A CTA per (b0, block of b2 rows): the running (b2, b3) plane of records
// with this b0 and b1' <= b1, prefixed along b2 and b3, in registers: warp i
// of the block owns row i, lane s the cells j = s + 32 m (every store of a
// warp is 32 consecutive cells, 512 B; strided per-thread segments measured
// 0.75 ms against 0.48 ms for this layout).  A record (p2, p3) adds to every
// cell with i >= p2 and j >= p3, i.e. to this lane's cells m >= m0 =
// ceil((p3 - s) / 32) when p2 <= i: each record is one add into a per-lane
// difference array over m (shared memory), and one running sum over m then
// gives every cell its gain -- O(cells + records) per lane and step instead
// of O(cells x records).  The row blocks of a plane are independent (each
// sees all of the slab's records), so the CTAs spread over every SM.  After
// each b1 step the block's rows are stored as T[b0][b1].
// NARROW: the b0 slab holds < 2^16 records, so a cell's four counts pack
// into 16-bit fields of one u64 (no field can carry); else 21-bit fields
// {cnt, c4, c3} plus c2 apart.  Both variants are launched; each CTA runs
// in the one that fits its slab and returns at once from the other.
template <bool NARROW>
__global__ void __launch_bounds__(kW5SlabThreads) w5_slab_kernel(const uint32_t* __restrict__ keys,
                                                                    const uint32_t* __restrict__ off,
                                                                    uint4* __restrict__ T, int d1, int d2,
                                                                    int d3, int rows_per_blk) {
  __shared__ uint32_t s_in[kW5SlabChunk];   // the slab's keys as read
  __shared__ uint32_t s_all[kW5SlabStage];  // every key of this b0 (when they fit)
  __shared__ uint32_t s_off[kW5MaxD1 + 1];  // this b0's slab offsets
  __shared__ uint64_t s_d[(kW5Seg + 1) * kW5SlabThreads];    // difference arrays
  __shared__ uint32_t s_d2[NARROW ? 1 : (kW5Seg + 1) * kW5SlabThreads];
  const int nblk = (d2 + rows_per_blk - 1) / rows_per_blk;
  const int b0 = blockIdx.x / nblk, blk = blockIdx.x % nblk;
  const uint32_t base = off[b0 * d1];
  if ((off[(b0 + 1) * d1] - base < 65536u) != NARROW) return;
  // this b0's offsets, and its keys when they fit, staged once: the b1 loop
  // then never waits on global memory
  for (int t = threadIdx.x; t <= d1; t += blockDim.x) s_off[t] = off[b0 * d1 + t] - base;
  __syncthreads();
  const bool staged = s_off[d1] <= (uint32_t)kW5SlabStage;
  if (staged)
    for (uint32_t t = threadIdx.x; t < s_off[d1]; t += blockDim.x) s_all[t] = keys[base + t];
  // warp i of the block owns row i, lane s the cells j = s + 32 m: every
  // store of the warp writes 32 consecutive cells (512 B)
  const int segs = 32;
  const int i = blk * rows_per_blk + (int)threadIdx.x / segs, j0 = threadIdx.x % segs;
  const bool live = (int)threadIdx.x / segs < rows_per_blk && i < d2;
  const int cells = d2 * d3;
  uint64_t q[kW5Seg];
  uint32_t q2[NARROW ? 1 : kW5Seg];
#pragma unroll
  for (int m = 0; m < kW5Seg; ++m) {
    q[m] = 0;
    if (!NARROW) q2[m] = 0;
  }
  uint4* out = T + (int64_t)b0 * d1 * cells;
  for (int b1 = 0; b1 < d1; ++b1) {
    const uint32_t kb = s_off[b1], ke = s_off[b1 + 1];
    for (uint32_t c0 = kb; c0 < ke; c0 += kW5SlabChunk) {
      const int nk = (int)min((uint32_t)kW5SlabChunk, ke - c0);
      __syncthreads();
      for (int t = threadIdx.x; t < nk; t += blockDim.x) s_in[t] = staged ? s_all[c0 + t] : keys[base + c0 + t];
      __syncthreads();
      __syncthreads();
      if (!live) continue;
      // a record (p2 <= i) reaches this thread's cells m >= m0 = ceil((p3 - s) / segs):
      // a difference array over m (shared memory, this thread's column), then
      // one running sum over m adds each cell's gain
      for (int m = 0; m <= kW5Seg; ++m) {
        s_d[m * blockDim.x + threadIdx.x] = 0ull;
        if (!NARROW) s_d2[m * blockDim.x + threadIdx.x] = 0u;
      }
      for (int e = 0; e < nk; ++e) {
        const uint32_t k = s_in[e];
        if (((k >> 8) & 255u) > (uint32_t)i) continue;
        const int p3 = (int)((k >> 16) & 255u);
        const int m0 = p3 <= j0 ? 0 : min(kW5Seg, (p3 - j0 + segs - 1) / segs);
        const uint64_t k4 = (k >> 24) & 1u, k3 = (k >> 25) & 1u, k2 = (k >> 26) & 1u;
        s_d[m0 * blockDim.x + threadIdx.x] += NARROW ? (1ull | (k4 << 16) | (k3 << 32) | (k2 << 48))
                                                     : (1ull | (k4 << 21) | (k3 << 42));
        if (!NARROW) s_d2[m0 * blockDim.x + threadIdx.x] += (uint32_t)k2;
      }
      uint64_t run = 0;
      uint32_t run2 = 0;
#pragma unroll
      for (int m = 0; m < kW5Seg; ++m) {
        run += s_d[m * blockDim.x + threadIdx.x];
        q[m] += run;
        if (!NARROW) {
          run2 += s_d2[m * blockDim.x + threadIdx.x];
          q2[m] += run2;
        }
      }
    }
    if (!live) continue;
    uint4* dst = out + (int64_t)b1 * cells + (int64_t)i * d3;
#pragma unroll
    for (int m = 0; m < kW5Seg; ++m) {
      const int j = j0 + segs * m;
      if (j >= d3) break;
      dst[j] = NARROW ? make_uint4((uint32_t)(q[m] & 0xffffu), (uint32_t)((q[m] >> 16) & 0xffffu),
                                   (uint32_t)((q[m] >> 32) & 0xffffu), (uint32_t)(q[m] >> 48))
                      : unpack_cell(q[m], q2[m]);
    }
  }
}

struct W5WalkArgs {
  int32_t g0, g1, g2, g3, d1, d2, d3, nblk;
  int64_t sF0, sF1, sF2;   // F strides of dims 0..2 (dim 3 contiguous)
  int64_t sb;              // first config of the full cascade
  int64_t cfg_begin, cfg_count;
  int64_t n_rec;
  double rcp_n;
  const double* cost1;
  const uint4* T;          // [b0][b1][b2][b3] prefixed along b1, b2, b3
  const uint4* P;          // side table [b0][b1] {c0, c1} fully prefixed
  uint4* faces;            // F layout, face cells only
  double* acc;
  double* cost;
  double* frac;
  uint32_t* n_correct;
};

// A CTA per (k1, block of kW5Rows k2 rows); a warp owns kW5RowsPerWarp rows,
// lane l the cells k3 = l + 32u.  For k0 = 0..g0 the running sums become
// F(k0, k1, k2, k3); the row's last cell (k3 = g3) and the CTA's corner
// cells F(k0, k1, g, g), F(k0, g, g, g) give the row-shared terms.
__global__ void __launch_bounds__(kW5WalkWarps * 32) w5_walk_kernel(const __grid_constant__ W5WalkArgs a) {
  __shared__ double s_frac[kW5WalkWarps][32 * kW5U * 5];
  const int k1 = blockIdx.x / a.nblk, blk = blockIdx.x % a.nblk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g0 = a.g0, g1 = a.g1, g2 = a.g2, g3 = a.g3, d3 = a.d3;
  const double n = (double)a.n_rec, rcp = a.rcp_n;
  const double one = div_count(n, n, rcp);
  const double c0 = __ldg(a.cost1), c1 = __ldg(a.cost1 + 1), c2 = __ldg(a.cost1 + 2),
               c3 = __ldg(a.cost1 + 3), c4 = __ldg(a.cost1 + 4);
  uint64_t q[kW5RowsPerWarp][kW5U];
  uint32_t q2[kW5RowsPerWarp][kW5U];
  int rows[kW5RowsPerWarp];
#pragma unroll
  for (int r = 0; r < kW5RowsPerWarp; ++r) {
    rows[r] = blk * kW5Rows + warp * kW5RowsPerWarp + r;
#pragma unroll
    for (int u = 0; u < kW5U; ++u) {
      q[r][u] = 0;
      q2[r][u] = 0;
    }
  }
  uint64_t A = 0, B = 0;       // running corner cells (k1, g, g) and (g, g, g)
  uint32_t A2 = 0;
  const uint4 Pgg = __ldg(a.P + (int64_t)g0 * a.d1 + g1);
  double* buf = s_frac[warp];
  const bool full_range_cta = true;
  (void)full_range_cta;
  for (int k0 = 0; k0 <= g0; ++k0) {
    const uint4* plane = a.T + (int64_t)k0 * a.sF0 + (int64_t)k1 * a.sF1;
    {
      const uint4 ca = __ldg(plane + (int64_t)g2 * a.sF2 + g3);
      const uint4 cb = __ldg(a.T + (int64_t)k0 * a.sF0 + (int64_t)g1 * a.sF1 + (int64_t)g2 * a.sF2 + g3);
      A += pack_cell(ca);
      A2 += ca.w;
      B += pack_cell(cb);
    }
#pragma unroll
    for (int r = 0; r < kW5RowsPerWarp; ++r) {
      if (rows[r] >= a.d2) continue;
      const uint4* row = plane + (int64_t)rows[r] * a.sF2;
#pragma unroll
      for (int u = 0; u < kW5U; ++u) {
        const int k3 = lane + 32 * u;
        if (k3 < d3) {
          const uint4 t = __ldg(row + k3);
          q[r][u] += pack_cell(t);
          q2[r][u] += t.w;
        }
      }
    }
    // face cells: some index at "any"
#pragma unroll
    for (int r = 0; r < kW5RowsPerWarp; ++r) {
      const int k2 = rows[r];
      if (k2 >= a.d2) continue;
      const bool all = k0 == g0 || k1 == g1 || k2 == g2;
      uint4* frow = a.faces + (int64_t)k0 * a.sF0 + (int64_t)k1 * a.sF1 + (int64_t)k2 * a.sF2;
#pragma unroll
      for (int u = 0; u < kW5U; ++u) {
        const int k3 = lane + 32 * u;
        if (k3 < d3 && (all || k3 == g3)) frow[k3] = unpack_cell(q[r][u], q2[r][u]);
      }
    }
    if (k1 == g1 || k0 == g0) continue;  // no full-cascade config here
    const uint4 Fk0 = unpack_cell(B, 0u);
    const uint4 Fk01 = unpack_cell(A, A2);
    const uint4 Pk0 = __ldg(a.P + (int64_t)k0 * a.d1 + g1);
    const uint4 Pk01 = __ldg(a.P + (int64_t)k0 * a.d1 + k1);
    const double fr1 = div_count((double)Fk0.x, n, rcp);
    const double fr2 = div_count((double)Fk01.x, n, rcp);
    const double m2 = dadd(dadd(dadd(0.0, dmul(one, c0)), dmul(fr1, c1)), dmul(fr2, c2));
    const uint32_t base = (Pgg.x - Pk0.x) + (Pk0.y - Pk01.y) + Fk01.w;
#pragma unroll
    for (int r = 0; r < kW5RowsPerWarp; ++r) {
      const int k2 = rows[r];
      if (k2 >= g2) continue;  // rows past the table or the "any" row
      // (k0, k1, k2, g): the row's last cell, from the lane holding k3 = g3
      uint64_t rq = 0;
      uint32_t rq2 = 0;
#pragma unroll
      for (int u = 0; u < kW5U; ++u) {
        const uint64_t tq = __shfl_sync(0xffffffffu, q[r][u], g3 & 31);
        const uint32_t tq2 = __shfl_sync(0xffffffffu, q2[r][u], g3 & 31);
        if (u == (g3 >> 5)) {
          rq = tq;
          rq2 = tq2;
        }
      }
      const uint4 rc = unpack_cell(rq, rq2);
      const double fr3 = div_count((double)rc.x, n, rcp);
      const double m3 = dadd(m2, dmul(fr3, c3));
      const uint32_t cr = base - rc.w + rc.z;
      const int64_t cfg0 = a.sb + (((int64_t)k0 * g1 + k1) * g2 + k2) * g3;  // k3 = 0
      const int64_t i0 = cfg0 - a.cfg_begin;
      const bool full = i0 >= 0 && i0 + g3 <= a.cfg_count;
      if (!full && (i0 + g3 <= 0 || i0 >= a.cfg_count)) continue;
#pragma unroll
      for (int u = 0; u < kW5U; ++u) {
        const int k3 = lane + 32 * u;
        if (k3 < g3) {
          const uint4 c = unpack_cell(q[r][u], q2[r][u]);
          const double fr4 = div_count((double)c.x, n, rcp);
          const double mean = dadd(m3, dmul(fr4, c4));
          const uint32_t correct = cr - c.z + c.y;
          const int64_t i = i0 + k3;
          if (full || (i >= 0 && i < a.cfg_count)) {
            if (a.cost) a.cost[i] = mean;
            if (a.acc) a.acc[i] = div_count((double)correct, n, rcp);
            if (a.n_correct) a.n_correct[i] = correct;
          }
          double* f = buf + k3 * 5;
          f[0] = one;
          f[1] = fr1;
          f[2] = fr2;
          f[3] = fr3;
          f[4] = fr4;
        }
      }
      __syncwarp();
      if (a.frac) {
        double* dst = a.frac + i0 * 5;
        const int ne = g3 * 5;
        if (full) {  // 16-byte stores from the first 16-byte boundary of the row
          const int head = (reinterpret_cast<uintptr_t>(dst) & 15u) ? 1 : 0;
          if (head && lane == 0) dst[0] = buf[0];
          const int npair = (ne - head) / 2;
          for (int p = lane; p < npair; p += 32) {
            const int e = head + 2 * p;
            *reinterpret_cast<double2*>(dst + e) = make_double2(buf[e], buf[e + 1]);
          }
          if (((ne - head) & 1) && lane == 0) dst[ne - 1] = buf[ne - 1];
        } else {
          for (int e = lane; e < ne; e += 32) {
            const int64_t i = i0 + e / 5;
            if (i >= 0 && i < a.cfg_count) dst[e] = buf[e];
          }
        }
      }
      __syncwarp();
    }
  }
}

}  // namespace

bool w5_supported(int64_t n_rec, int32_t M, const int32_t* glen) {
  if (M != 5 || n_rec < 1 || n_rec >= (1ll << 21)) return false;
  for (int j = 0; j < 4; ++j)
    if (glen[j] < 1 || glen[j] > 254) return false;
  const int64_t d3 = glen[3] + 1;
  return d3 <= 32 * kW5Seg && d3 <= 32 * kW5U &&
         (int64_t)(glen[0] + 1) * (glen[1] + 1) <= 26 * 1024;  // side table scanned in smem
}

W5Layout w5_layout(const int32_t* glen, int64_t n_rec) {
  W5Layout L{};
  L.d0 = glen[0] + 1;
  L.d1 = glen[1] + 1;
  L.d2 = glen[2] + 1;
  L.d3 = glen[3] + 1;
  L.cells2 = (int64_t)L.d0 * L.d1;
  L.cellsF = L.cells2 * L.d2 * L.d3;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += round_up(bytes, 256);
    return at;
  };
  L.offTmp = take((size_t)std::max<int64_t>(n_rec, 1) * 8);
  L.offKeys = take((size_t)std::max<int64_t>(n_rec, 1) * 4);
  L.offCnt = take((size_t)L.cells2 * 4);
  L.offHP = take((size_t)L.cells2 * 8);
  L.offOff = take((size_t)(L.cells2 + 1) * 4);
  L.offCur = take((size_t)L.cells2 * 4);
  L.offP = take((size_t)L.cells2 * 16);
  L.offT = take((size_t)L.cellsF * 16);
  L.offFaces = take((size_t)L.cellsF * 16);
  L.bytes = o;
  return L;
}

cudaError_t w5_build(const double* cert, const uint8_t* corr, int64_t n_rec, const double* grids,
                     const int32_t* glen, uint8_t* ws, bool dirty, cudaStream_t st) {
  const W5Layout L = w5_layout(glen, n_rec);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ws + L.offCnt);
  uint32_t* HP = reinterpret_cast<uint32_t*>(ws + L.offHP);
  cudaError_t e;
  if (dirty) {  // counts and the side histogram are left zero by every build
    if ((e = cudaMemsetAsync(cnt, 0, (size_t)L.cells2 * 4, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(HP, 0, (size_t)L.cells2 * 8, st)) != cudaSuccess) return e;
  }
  W5BinArgs b{};
  b.cert = cert;
  b.corr = corr;
  b.n_rec = n_rec;
  b.grids = grids;
  int og = 0;
  for (int j = 0; j < 4; ++j) {
    b.goff[j] = og;
    b.glen[j] = glen[j];
    og += glen[j];
  }
  b.d1 = L.d1;
  b.tmp = reinterpret_cast<uint64_t*>(ws + L.offTmp);
  b.cnt = cnt;
  b.HP = HP;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n_rec + 255) / 256, (int64_t)sm_count() * 8));
  w5_bin_kernel<<<(unsigned)blocks, 256, 0, st>>>(b);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  uint32_t* off = reinterpret_cast<uint32_t*>(ws + L.offOff);
  uint32_t* cur = reinterpret_cast<uint32_t*>(ws + L.offCur);
  static SmemAttr scan_attr;
  const size_t scan_smem = (size_t)L.cells2 * 8;
  if ((e = ensure_smem(w5_scan_kernel, scan_attr, scan_smem)) != cudaSuccess) return e;
  w5_scan_kernel<<<1, 1024, scan_smem, st>>>(cnt, off, cur, HP, reinterpret_cast<uint4*>(ws + L.offP),
                                            L.d0, L.d1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  w5_scatter_kernel<<<(unsigned)blocks, 256, 0, st>>>(b.tmp, n_rec, cur,
                                                      reinterpret_cast<uint32_t*>(ws + L.offKeys));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const uint32_t* keys = reinterpret_cast<const uint32_t*>(ws + L.offKeys);
  uint4* T = reinterpret_cast<uint4*>(ws + L.offT);
  // a CTA per (b0, block of b2 rows): the row blocks of a plane are
  // independent (every block sees all of the slab's records), so the planes'
  // stores spread over every SM
  const int segs = 32;  // a warp per row
  int nblk = std::max(1, std::min(L.d2, (8 * sm_count() + L.d0 - 1) / L.d0));
  int rows = (L.d2 + nblk - 1) / nblk;
  if (rows * segs > kW5SlabThreads) rows = kW5SlabThreads / segs;
  const int nb = (L.d2 + rows - 1) / rows;
  const int threads = (rows * segs + 31) / 32 * 32;
  w5_slab_kernel<true><<<(unsigned)(L.d0 * nb), threads, 0, st>>>(keys, off, T, L.d1, L.d2, L.d3, rows);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  w5_slab_kernel<false><<<(unsigned)(L.d0 * nb), threads, 0, st>>>(keys, off, T, L.d1, L.d2, L.d3, rows);
  return cudaGetLastError();
}

cudaError_t w5_walk(int64_t n_rec, const int32_t* glen, int64_t sb, const double* cost1, int64_t cfg_begin,
                    int64_t cfg_count, double* acc, double* cost, double* frac, uint32_t* n_correct,
                    const uint8_t* ws, cudaStream_t st) {
  const W5Layout L = w5_layout(glen, n_rec);
  W5WalkArgs a{};
  a.g0 = glen[0];
  a.g1 = glen[1];
  a.g2 = glen[2];
  a.g3 = glen[3];
  a.d1 = L.d1;
  a.d2 = L.d2;
  a.d3 = L.d3;
  a.nblk = (L.d2 + kW5Rows - 1) / kW5Rows;
  a.sF2 = L.d3;
  a.sF1 = (int64_t)L.d2 * L.d3;
  a.sF0 = (int64_t)L.d1 * a.sF1;
  a.sb = sb;
  a.cfg_begin = cfg_begin;
  a.cfg_count = cfg_count;
  a.n_rec = n_rec;
  a.rcp_n = 1.0 / (double)n_rec;
  a.cost1 = cost1;
  a.T = reinterpret_cast<const uint4*>(ws + L.offT);
  a.P = reinterpret_cast<const uint4*>(ws + L.offP);
  a.faces = reinterpret_cast<uint4*>(const_cast<uint8_t*>(ws) + L.offFaces);
  a.acc = acc;
  a.cost = cost;
  a.frac = frac;
  a.n_correct = n_correct;
  w5_walk_kernel<<<(unsigned)(L.d1 * a.nblk), kW5WalkWarps * 32, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace gs
