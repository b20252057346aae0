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

constexpr int kW5SlabThreads = 640;
constexpr int kW5SlabCells = 16;       // plane cells per thread (d2 * d3 <= 10240)
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
  // side table: prefix along b1 per row, then along b0 per column
  for (int r = threadIdx.x; r < d0; r += 1024) {
    uint32_t c0 = 0, c1 = 0;
    for (int c = 0; c < d1; ++c) {
      const int i = r * d1 + c;
      c0 += HP[2 * i];
      c1 += HP[2 * i + 1];
      HP[2 * i] = 0u;
      HP[2 * i + 1] = 0u;
      P[i] = make_uint4(c0, c1, 0u, 0u);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d1; c += 1024) {
    uint32_t c0 = 0, c1 = 0;
    for (int r = 0; r < d0; ++r) {
      uint4 v = P[r * d1 + c];
      c0 += v.x;
      c1 += v.y;
      v.x = c0;
      v.y = c1;
      P[r * d1 + c] = v;
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

// A CTA per b0: the running (b2, b3) plane of records with this b0 and
// b1' <= b1, prefixed along b2 and b3, one set of cells per thread in
// registers; a record adds to every cell (i, j) with i >= b2, j >= b3.
// Dominance is one subtraction: cell word X = 1 << 24 | i << 16 | 1 << 8 | j,
// record word y = b2 << 16 | b3 (all fields < 256): bit 8 of X - y survives
// iff j >= b3 and bit 24 iff i >= b2 (each field's guard bit absorbs its own
// borrow and the low field never borrows from the high one).  Cells past the
// plane accumulate garbage and are never stored.
// NARROW: the b0 slab holds < 2^16 records, so the four counts of a cell
// pack into 16-bit fields of one u64 (no field can carry); else 21-bit
// fields {cnt, c4, c3} plus c2 apart.  Both variants are launched; each CTA
// runs in the one that fits its slab and returns at once from the other.
template <bool NARROW>
__global__ void __launch_bounds__(kW5SlabThreads, 1) w5_slab_kernel(const uint32_t* __restrict__ keys,
                                                                    const uint32_t* __restrict__ off,
                                                                    uint4* __restrict__ T, int d1, int d2,
                                                                    int d3) {
  __shared__ uint32_t s_k[kW5SlabThreads];
  const int b0 = blockIdx.x;
  if ((off[(b0 + 1) * d1] - off[b0 * d1] < 65536u) != NARROW) return;
  const int cells = d2 * d3;
  uint32_t X[kW5SlabCells];
  uint64_t q[kW5SlabCells];
  uint32_t q2[NARROW ? 1 : kW5SlabCells];
#pragma unroll
  for (int m = 0; m < kW5SlabCells; ++m) {
    const int c = threadIdx.x + m * kW5SlabThreads;
    X[m] = c < cells ? (1u << 24) | ((uint32_t)(c / d3) << 16) | (1u << 8) | (uint32_t)(c % d3) : 0u;
    q[m] = 0;
    if (!NARROW) q2[m] = 0;
  }
  uint4* out = T + (int64_t)b0 * d1 * cells;
  for (int b1 = 0; b1 < d1; ++b1) {
    const uint32_t kb = off[b0 * d1 + b1], ke = off[b0 * d1 + b1 + 1];
    for (uint32_t c0 = kb; c0 < ke; c0 += kW5SlabThreads) {
      const uint32_t nk = min((uint32_t)kW5SlabThreads, ke - c0);
      __syncthreads();
      if (threadIdx.x < nk) s_k[threadIdx.x] = keys[c0 + threadIdx.x];
      __syncthreads();
      for (uint32_t e = 0; e < nk; ++e) {
        const uint32_t key = s_k[e];
        const uint32_t y = (((key >> 8) & 255u) << 16) | ((key >> 16) & 255u);  // b2 << 16 | b3
        const uint64_t k4 = (key >> 24) & 1u, k3 = (key >> 25) & 1u, k2 = (key >> 26) & 1u;
        const uint64_t inc = NARROW ? (1ull | (k4 << 16) | (k3 << 32) | (k2 << 48))
                                    : (1ull | (k4 << 21) | (k3 << 42));
#pragma unroll
        for (int m = 0; m < kW5SlabCells; ++m) {
          const bool dom = ((X[m] - y) & 0x01000100u) == 0x01000100u;
          q[m] += dom ? inc : 0ull;
          if (!NARROW) q2[m] += dom ? (uint32_t)k2 : 0u;
        }
      }
    }
    uint4* dst = out + (int64_t)b1 * cells;
#pragma unroll
    for (int m = 0; m < kW5SlabCells; ++m) {
      const int c = threadIdx.x + m * kW5SlabThreads;
      if (c >= cells) continue;
      dst[c] = NARROW ? make_uint4((uint32_t)(q[m] & 0xffffu), (uint32_t)((q[m] >> 16) & 0xffffu),
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
  const int64_t d2 = glen[2] + 1, d3 = glen[3] + 1;
  return d2 * d3 <= (int64_t)kW5SlabThreads * kW5SlabCells && d3 <= 32 * kW5U &&
         (int64_t)(glen[0] + 1) * (glen[1] + 1) <= 65536;
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
  w5_scan_kernel<<<1, 1024, 0, st>>>(cnt, off, cur, HP, reinterpret_cast<uint4*>(ws + L.offP), L.d0, L.d1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  w5_scatter_kernel<<<(unsigned)blocks, 256, 0, st>>>(b.tmp, n_rec, cur,
                                                      reinterpret_cast<uint32_t*>(ws + L.offKeys));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const uint32_t* keys = reinterpret_cast<const uint32_t*>(ws + L.offKeys);
  uint4* T = reinterpret_cast<uint4*>(ws + L.offT);
  w5_slab_kernel<true><<<(unsigned)L.d0, kW5SlabThreads, 0, st>>>(keys, off, T, L.d1, L.d2, L.d3);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  w5_slab_kernel<false><<<(unsigned)L.d0, kW5SlabThreads, 0, st>>>(keys, off, T, L.d1, L.d2, L.d3);
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
