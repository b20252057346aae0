// gs_grid.cu — grid path: the full cascade x per-stage-threshold product.
//
// Reference semantics: every config is an encoded cascade scored exactly as
// _evaluate_numba scores it (/root/reference/pkg/src/gearserve/kernels.py:
// 39-62); thresholds come from per-model grids (cascades.ThresholdGrid,
// src/cascades.py:132-163); structures are model subsets walked cheap to
// expensive like sample_cascades builds them (src/cascades.py:181-185).
//
// Algorithm: dominance counting instead of walking every record through
// every config.  With grid G_j of model j let b_j(r) = #{g in G_j : g <=
// cert[r, j]}.  cert >= G_j[k] <=> b_j > k, so record r is forwarded past a
// stage of model j with threshold index k iff b_j(r) <= k.  Models are in
// cost order and subsets are walked in that order, so model M-1 never
// forwards: one (M-1)-dimensional table over (b_0 .. b_{M-2}) answers every
// structure.  After an inclusive prefix sum along every dimension, a cell
// counts the records whose bins it dominates; a dimension at its maximum
// index g_j means "any".  With pos holding the thresholds of the stages
// walked so far:
//   reach(stage t+1) = cnt[pos after setting k_t]
//   correct          = sum_t (c_{m_t}[pos before k_t] - c_{m_t}[pos after])
//                      + c_{m_K}[final pos]
// which is the per-record walk's count, exactly.
//
// Table layout (HBM / L2): the main table F holds, per cell, one 16-byte
// vector of four counts {cnt, c_{M-1}, c_{M-2}, c_{M-3}}.  A correct count
// c_j is only ever read at positions whose dimensions > j are at "any", so
// models j <= M-4 live in a smaller side table S over dims 0..M-4 (for the
// 4-model cascade: one row of 101 cells, privatised in shared memory).
// The histogram adds each record with ONE red.global.add.v4.f32 (integer
// counts are exact in f32 below 2^24), so the histogram costs one L2 vector
// atomic per record.  The prefix sums convert to u32.
//
// Random-scatter L2 atomics bound the histogram, so the main table is first
// accumulated with ONE 64-bit atomic add per record: four 16-bit counts per
// cell.  A field can only carry if some cell holds >= 2^16 records; the
// thread that moves a count off 0xFFFF raises a flag and a second, normally
// empty, pass redoes the main table with f32 vector reductions (exact below
// 2^24), all on the device.  Histogram and prefix tables are separate
// buffers: the first scan pass reads the histogram, writes the u32 prefix and
// re-zeroes the histogram, so no memset runs per build (the caller zeroes the
// workspace once).
//
// Kernels: grid_hist (one pass over the records, vector loads, binary search
// in shared-memory grids), rowscan (contiguous last dim, warp-shuffle scan),
// colscan (strided dims: [len x 32]-cell tiles staged in shared memory with
// cp.async, one round trip per 128 rows), grid_eval (R consecutive configs per thread; everything that
// depends only on the leading thresholds is computed once per "row" of
// configs; f64 epilogue in the reference's order, no FMA contraction).
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "gs_common.cuh"
#include "gs_grid4.cuh"
#include "gs_grid_lut.cuh"

#include "gs_sweep5.cuh"

namespace gs {
namespace {

constexpr int kMaxM = GS_MAX_MODELS;
constexpr int64_t kMaxExactF32 = 1ll << 24;  // f32 fallback histogram exact below
constexpr int64_t kMaxRec = 1ll << 30;        // 32-bit record indices (with grid-stride headroom) and counts
constexpr int64_t kMaxRcp = 1ll << 26;        // div_count's range (gs_common.cuh)

// count / n, correctly rounded: div_count's three FP64 ops below 2^26
// records (the host passes rcp = 1/n), IEEE division above (rcp = 0)
__device__ __forceinline__ double div_n(double x, double n, double rcp) {
  return rcp != 0.0 ? div_count(x, n, rcp) : __ddiv_rn(x, n);
}
inline double rcp_of(int64_t n) { return n < kMaxRcp ? 1.0 / (double)n : 0.0; }
constexpr int kHistThreads = 512;
constexpr size_t kSidePrivMax = 16 * 1024;
constexpr size_t kSlabSmemMax = 200 * 1024;

struct Plan {
  int M = 0, D = 0, DP = 0, NVP = 0, n_struct = 0;
  int glen[kMaxM] = {};
  int64_t dims[kMaxM] = {};
  int64_t strideF[kMaxM] = {};
  int64_t strideP[kMaxM] = {};
  int64_t cellsF = 1, cellsP = 0;
  int64_t n_configs = 0;
  int64_t struct_begin[256 + 1] = {};
  uint32_t struct_mask[256] = {};
  size_t offH16 = 0, offHF = 0, offF = 0, offHP = 0, offP = 0, offFlag = 0, bytes = 0;
  bool g4 = false;    // M == 4 fast path (gs_grid4.cu)
  bool walk = false;  // M == 4: fused b_0 prefix + full-structure scoring
  bool w5 = false;    // M == 5: slab-sorted build + b_0 walk (gs_sweep5.cu)
  size_t offFaces = 0;
};

int make_plan(int64_t n_rec, int32_t M, const int32_t* grid_len, Plan* p) {
  if (M < 1 || !grid_len || n_rec < 1) return GS_EINVAL;
  if (M > kMaxM || n_rec >= kMaxRec) return GS_EUNSUPPORTED;
  p->M = M;
  p->D = M - 1;
  p->DP = M >= 4 ? M - 3 : 0;
  p->NVP = M >= 4 ? (M - 3 + 3) / 4 : 0;
  for (int j = 0; j < M; ++j) {
    if (grid_len[j] < 1 || grid_len[j] > 65535) return GS_EINVAL;
    p->glen[j] = grid_len[j];
  }
  double cells = 1.0;
  for (int j = 0; j < p->D; ++j) {
    p->dims[j] = (int64_t)p->glen[j] + 1;
    cells *= (double)p->dims[j];
  }
  if (cells * 16.0 > 1.4e11) return GS_EUNSUPPORTED;
  int64_t s = 1;
  for (int j = p->D - 1; j >= 0; --j) {
    p->strideF[j] = s;
    s *= p->dims[j];
  }
  p->cellsF = s;
  s = 1;
  for (int j = p->DP - 1; j >= 0; --j) {
    p->strideP[j] = s;
    s *= p->dims[j];
  }
  p->cellsP = p->DP > 0 ? s : 0;
  // structures: size ascending, then lexicographic (itertools.combinations)
  int ns = 0;
  int64_t off = 0;
  double total = 0.0;
  for (int K = 1; K <= M; ++K) {
    int idx[kMaxM];
    for (int i = 0; i < K; ++i) idx[i] = i;
    while (true) {
      uint32_t mask = 0;
      double cnt = 1.0;
      int64_t icnt = 1;
      for (int i = 0; i < K; ++i) mask |= 1u << idx[i];
      for (int i = 0; i + 1 < K; ++i) {
        cnt *= p->glen[idx[i]];
        icnt *= p->glen[idx[i]];
      }
      p->struct_mask[ns] = mask;
      p->struct_begin[ns] = off;
      off += icnt;
      total += cnt;
      ++ns;
      int i = K - 1;
      while (i >= 0 && idx[i] == M - K + i) --i;
      if (i < 0) break;
      ++idx[i];
      for (int q = i + 1; q < K; ++q) idx[q] = idx[q - 1] + 1;
    }
  }
  if (total > 9.0e18) return GS_EUNSUPPORTED;
  p->n_struct = ns;
  p->struct_begin[ns] = off;
  p->n_configs = off;
  const size_t bF = round_up((size_t)p->cellsF * 16, 256);
  const size_t bP = round_up((size_t)p->cellsP * p->NVP * 16, 256);
  const size_t b16 = round_up((size_t)p->cellsF * 8, 256);
  p->offH16 = 0;
  p->offHF = b16;
  p->offF = b16 + bF;
  p->offHP = b16 + 2 * bF;
  p->offP = b16 + 2 * bF + bP;
  p->offFlag = b16 + 2 * bF + 2 * bP;
  p->bytes = p->offFlag + 256;
  // GS_GRID_GENERAL=1 (tests only): the general path for every shape, so the
  // fast paths can be checked against it over a whole enumeration
  const char* general = std::getenv("GS_GRID_GENERAL");
  const bool special = !(general && general[0] == '1');
  p->g4 = special && grid4_supported(n_rec, M, p->glen);
  if (p->g4) {
    p->bytes = grid4_layout(p->glen, n_rec).bytes;
    return GS_OK;
  }
  p->w5 = special && w5_supported(n_rec, M, p->glen);
  if (p->w5) {
    const W5Layout L = w5_layout(p->glen, n_rec);
    p->bytes = L.bytes;
    p->offFaces = L.offFaces;
    p->offP = L.offP;
    return GS_OK;
  }
  p->walk = M == 4 && p->dims[0] <= 160 &&
            (size_t)p->dims[1] * p->dims[2] * 16 <= 200 * 1024 &&
            (size_t)p->dims[0] * 36 * 16 <= 92 * 1024;
  if (p->walk) {
    p->offFaces = p->bytes;
    p->bytes += bF;
  }
  return GS_OK;
}

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size,
// so later calls (e.g. inside a CUDA-graph capture) issue no attribute calls.

// ------------------------------------------------------------------ hist --
struct HistArgs {
  const double* cert;
  const uint8_t* corr;
  int64_t n_rec;
  const double* grids;
  int32_t goff[kMaxM];
  int32_t glen[kMaxM];
  int64_t strideF[kMaxM];
  int64_t strideP[kMaxM];
  int64_t cellsP;
  int32_t grid_doubles;  // grids of models 0..D-1 staged in smem
  int32_t vec_ok;
  int32_t priv;          // side table privatised in shared memory
  float* F;                // f32 fallback main histogram
  uint32_t* P;             // side histogram (u32 counts)
  unsigned long long* H16; // packed main histogram: 4 x 16-bit counts per cell
  uint32_t* flag;          // set when a cell count reaches 2^16 (fallback needed)
  int32_t f_u32;           // fallback histogram in u32 words (n_rec >= 2^24: f32 would round)
};

// MODE 0: main table as ONE 64-bit atomic add per record (fields {cnt,
// c_{M-1}, c_{M-2}, c_{M-3}} of 16 bits; every other field of a cell is <= its
// count, so no field can carry unless some cell's count passes 0xFFFF, and the
// thread that moves a count from 0xFFFF sees it in the returned old value and
// raises the flag).  MODE 1: exits at once unless the flag is up; then redoes
// the main table with f32 vector reductions (exact below 2^24), or with u32
// atomics for larger record sets (f_u32).
// Bin lookup: gs_grid_lut.cuh.
template <int M, typename Cell, int MODE>
__global__ void __launch_bounds__(kHistThreads) grid_hist_kernel(const __grid_constant__ HistArgs a) {
  if (MODE == 1 && *reinterpret_cast<volatile uint32_t*>(a.flag) == 0) return;
  constexpr int D = M - 1;
  constexpr int DP = M >= 4 ? M - 3 : 0;
  constexpr int NVP = M >= 4 ? (M - 3 + 3) / 4 : 0;
  extern __shared__ __align__(16) double s_grid[];
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(s_grid + a.grid_doubles);  // [D][buckets]: lb | ub << 16
  uint32_t* s_side = s_lut + D * kLutBuckets;
  __shared__ double s_lo[kMaxM], s_hi[kMaxM], s_scale[kMaxM];
  for (int i = threadIdx.x; i < a.grid_doubles; i += blockDim.x) s_grid[i] = a.grids[i];
  for (int i = threadIdx.x; i < D * kLutBuckets; i += blockDim.x) s_lut[i] = 0u;
  if (MODE == 0 && DP > 0 && a.priv)
    for (int64_t i = threadIdx.x; i < a.cellsP * NVP * 4; i += blockDim.x) s_side[i] = 0u;
  __syncthreads();
  if ((int)threadIdx.x < D) {
    const int j = threadIdx.x;
    const double* g = s_grid + a.goff[j];
    const int n = a.glen[j];
    s_lo[j] = g[0];
    s_hi[j] = g[n - 1];
    s_scale[j] = n > 1 ? (double)kLutBuckets / (g[n - 1] - g[0]) : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < D; ++j)
    for (int i = threadIdx.x; i < a.glen[j]; i += blockDim.x)
      atomicAdd(s_lut + j * kLutBuckets + lut_bucket(s_grid[a.goff[j] + i], s_lo[j], s_hi[j], s_scale[j]), 1u);
  __syncthreads();
  // per model: exclusive scan of the bucket counts -> (lb, ub), whole block
  // (kLutBuckets / kHistThreads consecutive buckets per thread)
  {
    __shared__ uint32_t s_wsum[kHistThreads / 32];
    constexpr int per = kLutBuckets / kHistThreads;
    const int warp = threadIdx.x >> 5, lane = (int)lane_id();
    for (int j = 0; j < D; ++j) {
      uint32_t* L = s_lut + j * kLutBuckets + threadIdx.x * per;
      uint32_t c[per], tot = 0;
#pragma unroll
      for (int q = 0; q < per; ++q) {
        c[q] = L[q];
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
#pragma unroll
      for (int q = 0; q < per; ++q) {
        L[q] = run | ((run + c[q]) << 16);
        run += c[q];
      }
      __syncthreads();
    }
  }

  // n_rec < 2^30: record indices fit 32 bits (offsets are taken in 64)
  const int n_rec = (int)a.n_rec;
  const int step = gridDim.x * blockDim.x;
  // the overflow test on each atomic's old value is made one iteration late,
  // so the loop never waits for an atomic's round trip
  unsigned long long prev_old = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rec; r += step) {
    double x[M];
    uint32_t k[M];
    const double* row = a.cert + (int64_t)r * M;
    if (M % 2 == 0 && a.vec_ok) {
#pragma unroll
      for (int j = 0; j < (M / 2) * 2; j += 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(row) + j / 2);
        x[j] = v.x;
        x[j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < M; ++j) x[j] = __ldg(row + j);
    }
    if (M == 4 && a.vec_ok) {
      const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(a.corr) + r);
#pragma unroll
      for (int j = 0; j < M; ++j) k[j] = ((w >> (8 * j)) & 0xffu) != 0;
    } else {
#pragma unroll
      for (int j = 0; j < M; ++j) k[j] = __ldg(a.corr + (int64_t)r * M + j) != 0;
    }
    Cell cellF = 0, cellP = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const uint32_t e = s_lut[j * kLutBuckets + lut_bucket(x[j], s_lo[j], s_hi[j], s_scale[j])];
      const int lb = (int)(e & 0xffffu), ub = (int)(e >> 16);
      const int b = lb + (ub > lb ? upper_count(s_grid + a.goff[j] + lb, ub - lb, x[j]) : 0);
      cellF += (Cell)b * (Cell)a.strideF[j];
      if (j < DP) cellP += (Cell)b * (Cell)a.strideP[j];
    }
    // main table: {cnt, c_{M-1}, c_{M-2}, c_{M-3}}
    uint32_t v[4] = {1u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (M - 1 - i >= 0) v[1 + i] = k[M - 1 - i];
    if (MODE == 1) {
      if (a.f_u32) {
        uint32_t* w = reinterpret_cast<uint32_t*>(a.F) + cellF * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (v[i]) atomicAdd(w + i, v[i]);
      } else {
        red_add_v4(a.F + cellF * 4, 1.f, (float)v[1], (float)v[2], (float)v[3]);
      }
      continue;
    }
    const unsigned long long inc = 1ull | ((unsigned long long)v[1] << 16) |
                                   ((unsigned long long)v[2] << 32) | ((unsigned long long)v[3] << 48);
    if ((prev_old & 0xffffull) == 0xffffull) *reinterpret_cast<volatile uint32_t*>(a.flag) = 1u;
    prev_old = atomicAdd(a.H16 + cellF, inc);
    // side table: c_j for j <= M-4 at (b_0..b_{M-4}); integer counts
    if constexpr (DP > 0) {
#pragma unroll
      for (int j = 0; j < DP; ++j) {
        const Cell e = (cellP * NVP + j / 4) * 4 + (j % 4);
        if (a.priv) {
          if (k[j]) atomicAdd(s_side + e, 1u);
        } else if (k[j]) {
          atomicAdd(a.P + e, 1u);
        }
      }
    }
  }
  if (MODE == 0 && (prev_old & 0xffffull) == 0xffffull) *reinterpret_cast<volatile uint32_t*>(a.flag) = 1u;
  if (MODE == 0 && DP > 0 && a.priv) {
    __syncthreads();
    for (int64_t i = threadIdx.x; i < a.cellsP * NVP * 4; i += blockDim.x) {
      const uint32_t c = s_side[i];
      if (c) atomicAdd(a.P + i, c);
    }
  }
}

// ----------------------------------------------------------------- scans --
__device__ __forceinline__ uint4 to_u4(float4 f) {
  return make_uint4(__float2uint_rn(f.x), __float2uint_rn(f.y), __float2uint_rn(f.z),
                    __float2uint_rn(f.w));
}
__device__ __forceinline__ uint4 add4(uint4 a, uint4 b) {
  return make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ uint4 shfl_up4(uint4 v, int o) {
  return make_uint4(__shfl_up_sync(0xffffffffu, v.x, o), __shfl_up_sync(0xffffffffu, v.y, o),
                    __shfl_up_sync(0xffffffffu, v.z, o), __shfl_up_sync(0xffffffffu, v.w, o));
}
__device__ __forceinline__ uint4 shfl4(uint4 v, int src) {
  return make_uint4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                    __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}

// Inclusive prefix along the contiguous last dimension: one warp per row of
// `len` uint4 cells, four consecutive cells per lane, warp-shuffle scan, one
// load round trip per 128 cells.  from_f32 converts the f32 histogram.
__global__ void __launch_bounds__(256) rowscan_kernel(uint4* src, uint4* T, int64_t n_rows, int len,
                                                      int from_f32) {
  const int lane = (int)lane_id();
  const bool zero = src != T;  // first pass: read the histogram and re-zero it
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += nw) {
    uint4* in = src + r * len;
    uint4* row = T + r * len;
    uint4 carry = make_uint4(0, 0, 0, 0);
    for (int base = 0; base < len; base += 128) {
      uint4 e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = base + lane * 4 + u;
        e[u] = c < len ? in[c] : make_uint4(0, 0, 0, 0);
        if (from_f32) e[u] = to_u4(*reinterpret_cast<float4*>(&e[u]));
      }
      if (zero) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = base + lane * 4 + u;
          if (c < len) in[c] = make_uint4(0, 0, 0, 0);
        }
      }
      uint4 tot = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        tot = add4(tot, e[u]);
        e[u] = tot;
      }
      uint4 incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint4 y = shfl_up4(incl, o);
        if (lane >= o) incl = add4(incl, y);
      }
      const uint4 excl = add4(carry, make_uint4(incl.x - tot.x, incl.y - tot.y, incl.z - tot.z,
                                                incl.w - tot.w));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = base + lane * 4 + u;
        if (c < len) row[c] = add4(e[u], excl);
      }
      carry = add4(carry, shfl4(incl, 31));
    }
  }
}

// First prefix pass of the main table (contiguous last dim): reads the packed
// 16-bit histogram, or the f32 fallback histogram when the overflow flag is
// up, re-zeroes what it read, and writes the u32 prefix.
__global__ void __launch_bounds__(256) rowscan_first_kernel(unsigned long long* H16, uint4* HF,
                                                            const uint32_t* flag, uint4* T,
                                                            int64_t n_rows, int len, int hf_u32) {
  const int lane = (int)lane_id();
  const bool fb = *flag != 0u;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += nw) {
    unsigned long long* in16 = H16 + r * len;
    uint4* inF = HF + r * len;
    uint4* row = T + r * len;
    uint4 carry = make_uint4(0, 0, 0, 0);
    for (int base = 0; base < len; base += 128) {
      uint4 e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = base + lane * 4 + u;
        e[u] = make_uint4(0, 0, 0, 0);
        if (c < len) {
          if (fb) {
            uint4 f = inF[c];
            e[u] = hf_u32 ? f : to_u4(*reinterpret_cast<float4*>(&f));
          } else {
            const unsigned long long w = in16[c];
            e[u] = make_uint4((uint32_t)(w & 0xffff), (uint32_t)((w >> 16) & 0xffff),
                              (uint32_t)((w >> 32) & 0xffff), (uint32_t)(w >> 48));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = base + lane * 4 + u;
        if (c < len) {
          in16[c] = 0ull;
          if (fb) inF[c] = make_uint4(0, 0, 0, 0);
        }
      }
      uint4 tot = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        tot = add4(tot, e[u]);
        e[u] = tot;
      }
      uint4 incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint4 y = shfl_up4(incl, o);
        if (lane >= o) incl = add4(incl, y);
      }
      const uint4 excl = add4(carry, make_uint4(incl.x - tot.x, incl.y - tot.y, incl.z - tot.z,
                                                incl.w - tot.w));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = base + lane * 4 + u;
        if (c < len) row[c] = add4(e[u], excl);
      }
      carry = add4(carry, shfl4(incl, 31));
    }
  }
}

// First prefix pass of the main table when its last two dims form a slab
// that fits in shared memory: one CTA per slab reads the packed histogram
// (or the f32 fallback), row-scans it in registers (a warp per row), writes
// the expanded u32 counts into a shared-memory slab, column-scans there and
// stores the slab once — one global read and one write for two dimensions.
__global__ void __launch_bounds__(1024) slab_first_kernel(unsigned long long* H16, uint4* HF,
                                                          const uint32_t* flag, uint4* T,
                                                          int64_t n_slabs, int rows, int cols,
                                                          uint4* sideH, uint4* sideT, int side_len,
                                                          int parts, int zero, int hf_u32) {
  // a slab may be split into `parts` column ranges, one CTA each: every CTA
  // reads whole rows (for the row prefix) but keeps, scans and stores only
  // its own columns, so twice the CTAs share the work
  extern __shared__ __align__(16) uint4 s_slab[];
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const bool fb = *flag != 0u;
  const int n = rows * cols;
  if (blockIdx.x == 0 && warp == nwarps - 1 && side_len > 0) {
    // a one-dimensional side table (4-model sweeps): scan it here too
    uint4 carry = make_uint4(0, 0, 0, 0);
    for (int b = 0; b < side_len; b += 32) {
      const int c = b + lane;
      uint4 v = c < side_len ? sideH[c] : make_uint4(0, 0, 0, 0);
      if (c < side_len) sideH[c] = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint4 y = shfl_up4(v, o);
        if (lane >= o) v = add4(v, y);
      }
      v = add4(v, carry);
      if (c < side_len) sideT[c] = v;
      carry = shfl4(v, 31);
    }
  }
  // fast path: every row load of a warp issued before any is consumed
  const bool pre = !fb && cols <= 128 && rows <= 4 * nwarps;
  const int hc = (cols + parts - 1) / parts;
  for (int64_t item = blockIdx.x; item < n_slabs * parts; item += gridDim.x) {
    const int64_t slab = item / parts;
    const int cb = (int)(item - slab * parts) * hc;
    const int ce = min(cols, cb + hc), wc = ce - cb;
    const int64_t base = slab * (int64_t)n;
    if (pre) {
      unsigned long long pv[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = warp + i * nwarps;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = lane * 4 + u;
          pv[i][u] = (r < rows && c < cols) ? H16[base + (int64_t)r * cols + c] : 0ull;
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = warp + i * nwarps;
        if (r >= rows) break;  // uniform across the warp
        uint4 e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = lane * 4 + u;
          const unsigned long long w = pv[i][u];
          e[u] = make_uint4((uint32_t)(w & 0xffff), (uint32_t)((w >> 16) & 0xffff),
                            (uint32_t)((w >> 32) & 0xffff), (uint32_t)(w >> 48));
          if (zero && c >= cb && c < ce) H16[base + (int64_t)r * cols + c] = 0ull;
        }
        uint4 tot = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          tot = add4(tot, e[u]);
          e[u] = tot;
        }
        uint4 incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint4 y = shfl_up4(incl, o);
          if (lane >= o) incl = add4(incl, y);
        }
        const uint4 excl = make_uint4(incl.x - tot.x, incl.y - tot.y, incl.z - tot.z, incl.w - tot.w);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = lane * 4 + u;
          if (c >= cb && c < ce) s_slab[r * wc + (c - cb)] = add4(e[u], excl);
        }
      }
    }
    for (int r = pre ? rows : warp; r < rows; r += nwarps) {
      unsigned long long* in16 = H16 + base + (int64_t)r * cols;
      uint4* inF = HF + base + (int64_t)r * cols;
      uint4* out = s_slab + r * wc - cb;
      uint4 carry = make_uint4(0, 0, 0, 0);
      for (int c0 = 0; c0 < cols; c0 += 128) {
        uint4 e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + lane * 4 + u;
          e[u] = make_uint4(0, 0, 0, 0);
          if (c < cols) {
            if (fb) {
              uint4 f = inF[c];
              e[u] = hf_u32 ? f : to_u4(*reinterpret_cast<float4*>(&f));
            } else {
              const unsigned long long w = in16[c];
              e[u] = make_uint4((uint32_t)(w & 0xffff), (uint32_t)((w >> 16) & 0xffff),
                                (uint32_t)((w >> 32) & 0xffff), (uint32_t)(w >> 48));
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + lane * 4 + u;
          if (zero && c >= cb && c < ce) {
            in16[c] = 0ull;
            if (fb) inF[c] = make_uint4(0, 0, 0, 0);
          }
        }
        uint4 tot = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          tot = add4(tot, e[u]);
          e[u] = tot;
        }
        uint4 incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint4 y = shfl_up4(incl, o);
          if (lane >= o) incl = add4(incl, y);
        }
        const uint4 excl = add4(carry, make_uint4(incl.x - tot.x, incl.y - tot.y, incl.z - tot.z,
                                                  incl.w - tot.w));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + lane * 4 + u;
          if (c >= cb && c < ce) out[c] = add4(e[u], excl);
        }
        carry = add4(carry, shfl4(incl, 31));
      }
    }
    __syncthreads();
    // columns: thread (cell, lane) walks the rows; consecutive threads touch
    // consecutive 32-bit words, so the walk is bank-conflict free
    uint32_t* w32 = reinterpret_cast<uint32_t*>(s_slab);
    const int rw = wc * 4;  // 32-bit words per smem row
    for (int t = threadIdx.x; t < rw; t += blockDim.x) {
      uint32_t acc = 0;
      int r = 0;
      for (; r + 4 <= rows; r += 4) {
        const uint32_t v0 = w32[(r + 0) * rw + t], v1 = w32[(r + 1) * rw + t];
        const uint32_t v2 = w32[(r + 2) * rw + t], v3 = w32[(r + 3) * rw + t];
        acc += v0;
        w32[(r + 0) * rw + t] = acc;
        acc += v1;
        w32[(r + 1) * rw + t] = acc;
        acc += v2;
        w32[(r + 2) * rw + t] = acc;
        acc += v3;
        w32[(r + 3) * rw + t] = acc;
      }
      for (; r < rows; ++r) {
        acc += w32[r * rw + t];
        w32[r * rw + t] = acc;
      }
    }
    __syncthreads();
    uint4* dst = T + base + cb;
    for (int i = threadIdx.x; i < rows * wc; i += blockDim.x) {
      const int r = i / wc, j = i - r * wc;
      dst[(int64_t)r * cols + j] = s_slab[i];
    }
    __syncthreads();
  }
}

// re-zero the f32 fallback histogram, only if the overflow flag is up
__global__ void zero_if_flag_kernel(uint4* HF, int64_t cells, const uint32_t* flag) {
  if (*reinterpret_cast<const volatile uint32_t*>(flag) == 0u) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cells;
       i += (int64_t)gridDim.x * blockDim.x)
    HF[i] = make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

constexpr int kColTile = 32;    // consecutive inner cells per CTA
constexpr int kColChunk = 128;  // rows of the scanned dimension per smem pass

// Inclusive prefix along a strided dimension of a table of uint4 cells viewed
// as [outer][len][inner].  A CTA owns kColTile consecutive inner cells of one
// outer index: it stages the [len x kColTile] tile in shared memory with
// cp.async (one round trip per 128 rows), scans each (cell, lane) column in
// shared memory, and writes the tile back coalesced.
__global__ void __launch_bounds__(256) colscan_kernel(uint4* src, uint4* T, int64_t outer, int64_t len,
                                                      int64_t inner, int from_f32) {
  extern __shared__ __align__(16) uint4 s[];  // [kColChunk][kColTile]
  const int64_t tiles_per_outer = (inner + kColTile - 1) / kColTile;
  const int64_t n_tiles = outer * tiles_per_outer;
  const int t = threadIdx.x;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t o = tile / tiles_per_outer;
    const int64_t i0 = (tile - o * tiles_per_outer) * kColTile;
    const int w = (int)min((int64_t)kColTile, inner - i0);
    uint4* base = T + o * len * inner + i0;
    uint4* in = src + o * len * inner + i0;
    const bool zero = src != T;
    // scanning threads: (cell c, lane q) = (t / 4, t % 4) for t < 4 * w
    uint32_t carry = 0;
    for (int64_t r0 = 0; r0 < len; r0 += kColChunk) {
      const int rows = (int)min((int64_t)kColChunk, len - r0);
      for (int e = t; e < rows * w; e += blockDim.x) {
        const int rr = e / w, cc = e - (e / w) * w;
        cp_async16(s + rr * kColTile + cc, in + (r0 + rr) * inner + cc);
      }
      cp_async_wait_all();
      __syncthreads();
      if (zero)
        for (int e = t; e < rows * w; e += blockDim.x) {
          const int rr = e / w, cc = e - (e / w) * w;
          in[(r0 + rr) * inner + cc] = make_uint4(0, 0, 0, 0);
        }
      if (t < 4 * w) {
        uint32_t* col = reinterpret_cast<uint32_t*>(s) + (t >> 2) * 4 + (t & 3);
        uint32_t acc = carry;
        int r = 0;
        for (; r + 4 <= rows; r += 4) {
          uint32_t v0 = col[(r + 0) * kColTile * 4], v1 = col[(r + 1) * kColTile * 4];
          uint32_t v2 = col[(r + 2) * kColTile * 4], v3 = col[(r + 3) * kColTile * 4];
          if (from_f32) {
            v0 = __float2uint_rn(__uint_as_float(v0));
            v1 = __float2uint_rn(__uint_as_float(v1));
            v2 = __float2uint_rn(__uint_as_float(v2));
            v3 = __float2uint_rn(__uint_as_float(v3));
          }
          acc += v0;
          col[(r + 0) * kColTile * 4] = acc;
          acc += v1;
          col[(r + 1) * kColTile * 4] = acc;
          acc += v2;
          col[(r + 2) * kColTile * 4] = acc;
          acc += v3;
          col[(r + 3) * kColTile * 4] = acc;
        }
        for (; r < rows; ++r) {
          uint32_t v = col[r * kColTile * 4];
          if (from_f32) v = __float2uint_rn(__uint_as_float(v));
          acc += v;
          col[r * kColTile * 4] = acc;
        }
        carry = acc;
      }
      __syncthreads();
      for (int e = t; e < rows * w; e += blockDim.x) {
        const int rr = e / w, cc = e - (e / w) * w;
        base[(r0 + rr) * inner + cc] = s[rr * kColTile + cc];
      }
      __syncthreads();
    }
  }
}

// -------------------------------------------------------------- epilogue --
// Configs are processed in "rows": the configs of one structure that share
// every threshold except the last forwarding stage's (consecutive in the
// enumeration).  One warp owns a row: the row-shared part of the walk (cells
// of the leading stages, their forward fractions and the partial mean cost)
// is computed once per warp from broadcast loads, then each lane finishes
// configs kl = lane, lane+32, ... with one 16-byte cell load, two f64
// divisions and coalesced stores.
struct EvalGridArgs {
  int32_t M, n_struct, NVP, DP;
  int32_t glen[kMaxM];
  int64_t strideF[kMaxM];
  int64_t strideP[kMaxM];
  int64_t n_rec, cellsF, cellsP;
  double rcp_n;  // RN(1 / n_rec), computed on the host
  int64_t cfg_begin, cfg_count;
  int64_t row_lo, row_hi;
  int64_t struct_begin[256 + 1];
  int64_t row_begin[256 + 1];
  uint32_t struct_mask[256];
  const uint4* F;
  const uint4* P;
  const double* cost1;
  double* acc;
  double* cost;
  double* frac;
  uint32_t* n_correct;
};

__device__ __forceinline__ uint32_t lane4(const uint4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

// correct count of model m at the current position
template <int M>
__device__ __forceinline__ uint32_t chan(const uint4& vF, const uint4* vP, int m) {
  if (m >= M - 3) return lane4(vF, 1 + (M - 1 - m));
  return lane4(vP[m / 4], m % 4);
}

template <int M>
__device__ __forceinline__ void store_config(const EvalGridArgs& a, int64_t i, const double* fr,
                                             int K, double frK, double mean, uint32_t correct,
                                             double n, double rcp) {
  if (a.frac) {
    double o[M];
#pragma unroll
    for (int t = 0; t < M; ++t) o[t] = t < K - 1 ? fr[t] : (t == K - 1 ? frK : 0.0);
    double* row = a.frac + i * M;
    if constexpr (M % 2 == 0) {
#pragma unroll
      for (int t = 0; t < M; t += 2) reinterpret_cast<double2*>(row)[t / 2] = make_double2(o[t], o[t + 1]);
    } else {
#pragma unroll
      for (int t = 0; t < M; ++t) row[t] = o[t];
    }
  }
  if (a.cost) a.cost[i] = mean;
  if (a.acc) a.acc[i] = div_n((double)correct, n, rcp);
  if (a.n_correct) a.n_correct[i] = correct;
}

template <int M>
__global__ void __launch_bounds__(256) grid_eval_kernel(const __grid_constant__ EvalGridArgs a) {
  __shared__ double s_frac[8 * 32 * M];  // per-warp staging of forward_frac rows
  constexpr int NVP = M >= 4 ? (M - 3 + 3) / 4 : 0;
  constexpr int NVPX = NVP > 0 ? NVP : 1;
  const int lane = (int)lane_id();
  const double n = (double)a.n_rec;
  const double rcp = a.rcp_n;
  const double one = div_n(n, n, rcp);  // first-stage fraction: n / n
  const uint4 totF = __ldg(a.F + a.cellsF - 1);
  uint4 totP[NVPX];
#pragma unroll
  for (int v = 0; v < NVPX; ++v)
    totP[v] = NVP > 0 ? __ldg(a.P + (a.cellsP - 1) * NVP + v) : make_uint4(0, 0, 0, 0);

  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t rg = a.row_lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
       rg < a.row_hi; rg += nw) {
    int s = 0;
    {
      int lo = 0, hi = a.n_struct - 1;  // last s with row_begin[s] <= rg
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.row_begin[mid] <= rg)
          lo = mid;
        else
          hi = mid - 1;
      }
      s = lo;
    }
    const uint32_t mask = a.struct_mask[s];
    int K = 0;
    uint32_t mdl = 0;  // stage models, 4 bits each, stage 0 lowest
#pragma unroll
    for (int j = 0; j < M; ++j)
      if ((mask >> j) & 1u) {
        mdl |= (uint32_t)j << (4 * K);
        ++K;
      }
    const int64_t row = rg - a.row_begin[s];
    const int64_t s_begin = a.struct_begin[s];
    const int mK = (mdl >> (4 * (K - 1))) & 15u;
    double fr[M];
#pragma unroll
    for (int t = 0; t < M; ++t) fr[t] = 0.0;
    if (K == 1) {
      const int64_t i = s_begin - a.cfg_begin;
      if (lane == 0 && i >= 0 && i < a.cfg_count) {
        const double mean = dadd(0.0, dmul(one, __ldg(a.cost1 + mK)));
        store_config<M>(a, i, fr, 1, one, mean, chan<M>(totF, totP, mK), n, rcp);
      }
      continue;
    }
    const int mL = (mdl >> (4 * (K - 2))) & 15u;
    const int gL = a.glen[mL];
    // leading thresholds k_0 .. k_{K-3} from the row index
    int kk[M];
    int64_t rem = row;
#pragma unroll
    for (int t = M - 1; t >= 0; --t) {
      kk[t] = 0;
      if (t <= K - 3) {
        const int g = a.glen[(mdl >> (4 * t)) & 15u];
        if (rem < 0x7fffffffLL) {  // 32-bit division in the common case
          const int r32 = (int)rem;
          kk[t] = r32 % g;
          rem = r32 / g;
        } else {
          kk[t] = (int)(rem % g);
          rem /= g;
        }
      }
    }
    int64_t cF = a.cellsF - 1, cP = a.cellsP - 1;
    uint4 vF = totF;
    uint4 vP[NVPX];
#pragma unroll
    for (int v = 0; v < NVPX; ++v) vP[v] = totP[v];
    uint32_t cp = 0;
    fr[0] = one;
    double mp = dadd(0.0, dmul(one, __ldg(a.cost1 + (mdl & 15u))));
#pragma unroll
    for (int t = 0; t < M - 2; ++t) {
      if (t <= K - 3) {
        const int m = (mdl >> (4 * t)) & 15u;
        const uint32_t A = chan<M>(vF, vP, m);
        const int64_t dk = (int64_t)(a.glen[m] - kk[t]);
        cF -= dk * a.strideF[m];
        vF = __ldg(a.F + cF);
        if (NVP > 0 && m < a.DP) {
          cP -= dk * a.strideP[m];
#pragma unroll
          for (int v = 0; v < NVPX; ++v) vP[v] = __ldg(a.P + cP * NVP + v);
        }
        cp += A - chan<M>(vF, vP, m);
        fr[t + 1] = div_n((double)vF.x, n, rcp);
        mp = dadd(mp, dmul(fr[t + 1], __ldg(a.cost1 + ((mdl >> (4 * (t + 1))) & 15u))));
      }
    }
    const uint32_t a_last = chan<M>(vF, vP, mL);
    const double costK = __ldg(a.cost1 + mK);
    const bool needP = NVP > 0 && (mL < a.DP || mK < a.DP);
    const int64_t c_row = s_begin + row * gL - a.cfg_begin;
    // cell of threshold index kl: rowF + kl * sL (kl = gL would be "any")
    const int64_t sL = a.strideF[mL];
    const uint4* rowF = a.F + (cF - (int64_t)gL * sL);
    const int64_t sPL = (NVP > 0 && mL < a.DP) ? a.strideP[mL] : 0;
    const int64_t rowP = cP - (int64_t)gL * sPL;
    constexpr int U = 4;  // configs per lane per pass, loads issued together
    for (int base = 0; base < gL; base += 32 * U) {
      uint4 wF[U];
      uint4 wP[U][NVPX];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kl = base + lane + 32 * u;
        wF[u] = kl < gL ? __ldg(rowF + (int64_t)kl * sL) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int v = 0; v < NVPX; ++v)
          wP[u][v] = (needP && kl < gL) ? __ldg(a.P + (rowP + (int64_t)kl * sPL) * NVP + v)
                                        : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kl = base + lane + 32 * u;
        const int64_t i = c_row + kl;
        const bool ok = kl < gL && i >= 0 && i < a.cfg_count;
        const uint32_t correct =
            cp + a_last - chan<M>(wF[u], wP[u], mL) + chan<M>(wF[u], wP[u], mK);
        const double frK = div_n((double)wF[u].x, n, rcp);
        const double mean = dadd(mp, dmul(frK, costK));
        if (ok) {
          if (a.cost) a.cost[i] = mean;
          if (a.acc) a.acc[i] = div_n((double)correct, n, rcp);
          if (a.n_correct) a.n_correct[i] = correct;
        }
        // forward_frac: the warp's 32 consecutive [M]-rows go through a
        // per-warp shared buffer and leave as M fully coalesced stores
        // (strided per-lane rows cost M partial-line writes per row)
        if (a.frac) {
          double* buf = s_frac + (threadIdx.x >> 5) * (32 * M);
#pragma unroll
          for (int t = 0; t < M; ++t) buf[lane * M + t] = t < K - 1 ? fr[t] : (t == K - 1 ? frK : 0.0);
          __syncwarp();
          const int64_t i0 = c_row + base + 32 * u;  // config of lane 0
#pragma unroll
          for (int j = 0; j < M; ++j) {
            const int e = j * 32 + lane, src = e / M;
            const int64_t is = i0 + src;
            if (base + 32 * u + src < gL && is >= 0 && is < a.cfg_count) a.frac[i0 * M + e] = buf[e];
          }
          __syncwarp();
        }
      }
    }
  }
}

// ------------------------------------------------ full cascade (M = 5) --
// For five models the full cascade (0,1,2,3,4) holds g0 g1 g2 g3 of the
// configs (95% at 100-level grids) and its config (k0, k1, k2, k3) reads the
// table at (k0,g,g,g), (k0,k1,g,g), (k0,k1,k2,g) and (k0,k1,k2,k3).  A CTA
// owns one (k0, k1) pair: its row-shared terms (two fractions, the partial
// mean through stage 2, the correct counts of models 0-2) once per CTA; a
// warp per k2 row loads the row's d3 cells (contiguous, the last one being
// (k0,k1,k2,g)) and scores its g3 configs, which are consecutive in the
// enumeration; forward_frac rows (40 B, not vector aligned) go through a
// per-warp shared buffer and the row's block leaves as coalesced 16-byte
// stores.  The regular
// eval scores the other structures.
constexpr int kFull5Threads = 256;
constexpr int kFull5MaxRow = 128;  // g3 bound (per-warp frac buffer: 40 KB static)

struct Full5Args {
  int32_t g0, g1, g2, g3, d1;
  int64_t sF0, sF1, sF2;  // F strides of dims 0..2 (dim 3 contiguous)
  int64_t sb;             // first config of the full cascade
  int64_t cfg_begin, cfg_count;
  int64_t n_rec;
  double rcp_n;
  const double* cost1;
  const uint4* F;  // {cnt, c4, c3, c2} fully prefixed
  const uint4* P;  // side table over (b0, b1): {c0, c1, -, -}
  double* acc;
  double* cost;
  double* frac;
  uint32_t* n_correct;
};

__global__ void __launch_bounds__(kFull5Threads) full5_eval_kernel(const __grid_constant__ Full5Args a) {
  __shared__ double s_frac[kFull5Threads / 32][kFull5MaxRow * 5];  // the warp's row of frac rows
  const int k0 = blockIdx.x / a.g1, k1 = blockIdx.x % a.g1;
  const int g1 = a.g1, g2 = a.g2, g3 = a.g3;
  const int64_t cta_first = a.sb + ((int64_t)k0 * g1 + k1) * g2 * g3;
  const int64_t cta_end = cta_first + (int64_t)g2 * g3;
  if (cta_end <= a.cfg_begin || cta_first >= a.cfg_begin + a.cfg_count) return;
  const bool full = cta_first >= a.cfg_begin && cta_end <= a.cfg_begin + a.cfg_count;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double n = (double)a.n_rec, rcp = a.rcp_n;
  const double one = div_n(n, n, rcp);
  const double c0 = __ldg(a.cost1), c1 = __ldg(a.cost1 + 1), c2 = __ldg(a.cost1 + 2),
               c3 = __ldg(a.cost1 + 3), c4 = __ldg(a.cost1 + 4);
  const uint4 Fk0 = __ldg(a.F + k0 * a.sF0 + (int64_t)g1 * a.sF1 + (int64_t)g2 * a.sF2 + g3);
  const uint4 Fk01 = __ldg(a.F + k0 * a.sF0 + (int64_t)k1 * a.sF1 + (int64_t)g2 * a.sF2 + g3);
  const uint4 Pgg = __ldg(a.P + (int64_t)a.g0 * a.d1 + g1);
  const uint4 Pk0 = __ldg(a.P + (int64_t)k0 * a.d1 + g1);
  const uint4 Pk01 = __ldg(a.P + (int64_t)k0 * a.d1 + k1);
  const double fr1 = div_n((double)Fk0.x, n, rcp);
  const double fr2 = div_n((double)Fk01.x, n, rcp);
  const double m2 = dadd(dadd(dadd(0.0, dmul(one, c0)), dmul(fr1, c1)), dmul(fr2, c2));
  // models 0, 1 complete between their positions; model 2's count before k2
  const uint32_t base = (Pgg.x - Pk0.x) + (Pk0.y - Pk01.y) + Fk01.w;
  double* buf = s_frac[warp];
  constexpr int U = (kFull5MaxRow + 32) / 32;  // cells per lane (d3 = g3 + 1 <= 32 U)
  for (int k2 = warp; k2 < g2; k2 += kFull5Threads / 32) {
    const uint4* row = a.F + k0 * a.sF0 + (int64_t)k1 * a.sF1 + (int64_t)k2 * a.sF2;
    uint4 cell[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k3 = lane + 32 * u;
      cell[u] = k3 <= g3 ? __ldg(row + k3) : make_uint4(0, 0, 0, 0);
    }
    uint4 rc = make_uint4(0, 0, 0, 0);  // (k0, k1, k2, g): the row's last cell
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4 t = make_uint4(__shfl_sync(0xffffffffu, cell[u].x, g3 & 31),
                                 __shfl_sync(0xffffffffu, cell[u].y, g3 & 31),
                                 __shfl_sync(0xffffffffu, cell[u].z, g3 & 31),
                                 __shfl_sync(0xffffffffu, cell[u].w, g3 & 31));
      if (u == (g3 >> 5)) rc = t;
    }
    const double fr3 = div_n((double)rc.x, n, rcp);
    const double m3 = dadd(m2, dmul(fr3, c3));
    const uint32_t cr = base - rc.w + rc.z;  // through model 2, plus model 3's count before k3
    const int64_t i0 = cta_first + (int64_t)k2 * g3 - a.cfg_begin;  // config of k3 = 0
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k3 = lane + 32 * u;
      if (k3 < g3) {
        const uint4 c = cell[u];
        const double fr4 = div_n((double)c.x, n, rcp);
        const double mean = dadd(m3, dmul(fr4, c4));
        const uint32_t correct = cr - c.z + c.y;
        const int64_t i = i0 + k3;
        if (full || (i >= 0 && i < a.cfg_count)) {
          if (a.cost) a.cost[i] = mean;
          if (a.acc) a.acc[i] = div_n((double)correct, n, rcp);
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
      if (full) {
        // 16-byte stores from the first 16-byte boundary of the block
        const int head = (reinterpret_cast<uintptr_t>(dst) & 15u) ? 1 : 0;
        if (head && lane == 0) dst[0] = buf[0];
        const int npair = (ne - head) / 2;
        for (int q = lane; q < npair; q += 32) {
          const int e = head + 2 * q;
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

// -------------------------------------------------------- fused walk (M=4) --
// For four models the dominant structure is the full cascade (0,1,2,3): its
// g0*g1*g2 configs are 96% of the enumeration and map one-to-one onto table
// cells (k0, k1, k2).  walk_eval fuses the last prefix pass (along b_0) with
// their scoring: a CTA owns a tile of kWalkTile consecutive cells of the
// (b_1, b_2) plane, stages that tile for every k0 with 1-D TMA bulk copies
// (one mbarrier), scans it along k0 in shared memory (threads = cell x step
// group, two-level), and for each (k0, cell) writes the config's outputs
// directly.  The row-shared cells the walk needs, (k0, k1, g2) and
// (k0, g1, g2), are three extra running columns per CTA.  Only the "face"
// cells (some index at its maximum) are written back: they are all the
// smaller structures read, which the regular eval then scores.
constexpr int kWalkTile = 36;    // max cells per tile (<= d2, so a tile spans <= 2 rows)
constexpr int kWalkGroups = 14;  // step groups: 36 x 14 = 504 threads
constexpr int kWalkMaxSteps = 160;

struct WalkArgs {
  int32_t d0, d1, d2;
  int32_t tile;  // cells per CTA (<= kWalkTile and <= d2)
  int64_t sb;    // first config of the full structure
  int64_t cfg_begin, cfg_count;
  int64_t n_rec;
  double rcp_n;
  const double* cost1;
  const uint4* S;      // slab-prefixed table [d0][d1 * d2]
  uint4* faces;        // full prefix, face cells only
  const uint4* Pside;  // finished side table [d0] (c_0 in .x)
  double* acc;
  double* cost;
  double* frac;
  uint32_t* n_correct;
};

__global__ void __launch_bounds__(512) walk_eval_kernel(const __grid_constant__ WalkArgs a) {
  extern __shared__ __align__(16) uint4 s_tile[];  // [d0][tile]
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint4 s_grp[kWalkGroups][kWalkTile];
  __shared__ uint4 s_ext[3][kWalkMaxSteps];  // running (k0, ra, g2), (k0, rb, g2), (k0, g1, g2)
  __shared__ uint32_t s_side[kWalkMaxSteps];
  const int d0 = a.d0, d1 = a.d1, d2 = a.d2;
  const int g0 = d0 - 1, g1 = d1 - 1, g2 = d2 - 1;
  const int plane = d1 * d2;
  const int T = a.tile;
  const int c0 = blockIdx.x * T;
  const int w = min(T, plane - c0);
  const int ra = c0 / d2, rb = (c0 + w - 1) / d2;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar, (uint32_t)(d0 * w * sizeof(uint4)));
    for (int k0 = 0; k0 < d0; ++k0)
      bulk_g2s(s_tile + k0 * T, a.S + (int64_t)k0 * plane + c0, (uint32_t)(w * sizeof(uint4)), &bar);
  }
  for (int i = tid; i < 3 * d0; i += blockDim.x) {
    const int col = i / d0, k0 = i - col * d0;
    const int row = col == 0 ? ra : (col == 1 ? rb : g1);
    s_ext[col][k0] = a.S[(int64_t)k0 * plane + row * d2 + g2];
  }
  for (int k0 = tid; k0 < d0; k0 += blockDim.x) s_side[k0] = a.Pside[k0].x;
  __syncthreads();
  // prefix of the three extra columns along k0 (one warp per column)
  for (int col = tid >> 5; col < 3; col += blockDim.x >> 5) {
    const int lane = tid & 31;
    uint4 carry = make_uint4(0, 0, 0, 0);
    for (int base = 0; base < d0; base += 32) {
      const int k0 = base + lane;
      uint4 v = k0 < d0 ? s_ext[col][k0] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint4 y = shfl_up4(v, o);
        if (lane >= o) v = add4(v, y);
      }
      v = add4(v, carry);
      if (k0 < d0) s_ext[col][k0] = v;
      carry = shfl4(v, 31);
    }
  }
  mbar_wait(&bar, 0);
  // two-level scan of the tile along k0: thread = (cell ci, step group q)
  const int ci = tid % T, q = tid / T;  // threads past T * kWalkGroups only pad the warp
  const int L = (d0 + kWalkGroups - 1) / kWalkGroups;
  const int s0 = q * L, s1 = min(d0, s0 + L);
  uint4 run = make_uint4(0, 0, 0, 0);
  if (ci < w && q < kWalkGroups)
    for (int k0 = s0; k0 < s1; ++k0) run = add4(run, s_tile[k0 * T + ci]);
  if (q < kWalkGroups) s_grp[q][ci] = run;
  __syncthreads();
  if (ci >= w || q >= kWalkGroups) return;
  uint4 P = make_uint4(0, 0, 0, 0);
  for (int qq = 0; qq < q; ++qq) P = add4(P, s_grp[qq][ci]);
  const int cell = c0 + ci;
  const int k1 = cell / d2, k2 = cell - k1 * d2;
  const int xcol = k1 == ra ? 0 : 1;
  const double n = (double)a.n_rec, rcp = a.rcp_n;
  const double one = div_n(n, n, rcp);
  const double cA = __ldg(a.cost1 + 0), cB = __ldg(a.cost1 + 1), cC = __ldg(a.cost1 + 2),
               cD = __ldg(a.cost1 + 3);
  const double m0 = dadd(0.0, dmul(one, cA));
  const uint32_t side_tot = s_side[g0];
  const bool face_cell = k1 == g1 || k2 == g2;
  const bool cfg_cell = k1 < g1 && k2 < g2;
  for (int k0 = s0; k0 < s1; ++k0) {
    P = add4(P, s_tile[k0 * T + ci]);  // full prefix P[k0][k1][k2]
    if (face_cell || k0 == g0) a.faces[(int64_t)k0 * plane + cell] = P;
    if (!cfg_cell || k0 == g0) continue;
    const int64_t i = a.sb + ((int64_t)k0 * g1 + k1) * g2 + k2 - a.cfg_begin;
    if (i < 0 || i >= a.cfg_count) continue;
    const uint4 X0 = s_ext[2][k0];     // (k0, g1, g2): after stage 0
    const uint4 X1 = s_ext[xcol][k0];  // (k0, k1, g2): after stage 1
    // channels {cnt, c3, c2, c1}; c0 from the side table
    const uint32_t correct = (side_tot - s_side[k0]) + (X0.w - X1.w) + (X1.z - P.z) + P.y;
    const double f1 = div_n((double)X0.x, n, rcp);
    const double f2 = div_n((double)X1.x, n, rcp);
    const double f3 = div_n((double)P.x, n, rcp);
    const double mean = dadd(dadd(dadd(m0, dmul(f1, cB)), dmul(f2, cC)), dmul(f3, cD));
    if (a.frac) {
      double2* row = reinterpret_cast<double2*>(a.frac + i * 4);
      row[0] = make_double2(one, f1);
      row[1] = make_double2(f2, f3);
    }
    if (a.cost) a.cost[i] = mean;
    if (a.acc) a.acc[i] = div_n((double)correct, n, rcp);
    if (a.n_correct) a.n_correct[i] = correct;
  }
}

// ---------------------------------------------------------------- decode --
struct DecodeArgs {
  int32_t M, n_struct;
  int32_t glen[kMaxM];
  int32_t goff[kMaxM];
  int64_t struct_begin[256 + 1];
  uint32_t struct_mask[256];
  const double* grids;
  const int64_t* idx;
  int64_t count;
  int32_t* stage_model;
  double* thr;
  int32_t* n_stages;
};

__global__ void grid_decode_kernel(const __grid_constant__ DecodeArgs a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = a.idx[i];
    int lo = 0, hi = a.n_struct - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.struct_begin[mid] <= c)
        lo = mid;
      else
        hi = mid - 1;
    }
    const uint32_t mask = a.struct_mask[lo];
    int mdl[kMaxM];
    int K = 0;
    for (int j = 0; j < a.M; ++j)
      if ((mask >> j) & 1u) mdl[K++] = j;
    int64_t local = c - a.struct_begin[lo];
    int kidx[kMaxM];
    for (int t = K - 2; t >= 0; --t) {
      const int g = a.glen[mdl[t]];
      kidx[t] = (int)(local % g);
      local /= g;
    }
    for (int t = 0; t < a.M; ++t) {
      a.stage_model[i * a.M + t] = t < K ? mdl[t] : -1;
      a.thr[i * a.M + t] = (t < K - 1) ? a.grids[a.goff[mdl[t]] + kidx[t]] : 0.0;
    }
    a.n_stages[i] = K;
  }
}

// configs per row of structure s (the last forwarding stage's grid size)
int64_t row_len(const Plan& p, int s) {
  const uint32_t mask = p.struct_mask[s];
  int prev = -1, last = -1;
  for (int j = 0; j < p.M; ++j)
    if ((mask >> j) & 1u) {
      prev = last;
      last = j;
    }
  return prev < 0 ? 1 : p.glen[prev];
}

int64_t global_row(const Plan& p, const int64_t* row_begin, int64_t c) {
  int s = 0;
  while (s + 1 < p.n_struct && p.struct_begin[s + 1] <= c) ++s;
  return row_begin[s] + (c - p.struct_begin[s]) / row_len(p, s);
}

template <int M, typename Cell>
cudaError_t launch_hist_t(const HistArgs& h, int64_t n_rec, size_t smem, cudaStream_t st) {
  // persistent grid: the bin lookup tables are built once per CTA
  int64_t blocks = (n_rec + kHistThreads - 1) / kHistThreads;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 4));
  {
    auto k = grid_hist_kernel<M, Cell, 0>;
    static SmemAttr smem_set;
    cudaError_t e = ensure_smem(k, smem_set, smem);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)blocks, kHistThreads, smem, st>>>(h);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (n_rec < 65536) return cudaSuccess;  // no cell can reach 2^16 records
  auto k = grid_hist_kernel<M, Cell, 1>;  // no-op unless a cell passed 0xFFFF records
  static SmemAttr smem_set;
  cudaError_t e = ensure_smem(k, smem_set, smem);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)std::min<int64_t>(blocks, sm_count()), kHistThreads, smem, st>>>(h);
  return cudaGetLastError();
}

// 32-bit cell arithmetic whenever every table index fits
template <int M>
cudaError_t launch_hist(const HistArgs& h, int64_t n_rec, size_t smem, int64_t max_index,
                        cudaStream_t st) {
  return max_index < ((int64_t)1 << 32) ? launch_hist_t<M, uint32_t>(h, n_rec, smem, st)
                                        : launch_hist_t<M, int64_t>(h, n_rec, smem, st);
}

template <int M>
cudaError_t launch_grid_eval(const EvalGridArgs& a, cudaStream_t st) {
  const int64_t rows = a.row_hi - a.row_lo;
  int64_t blocks = (rows * 32 + 255) / 256;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 32));
  grid_eval_kernel<M><<<(unsigned)blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// Inclusive prefix over every dimension of a table of uint4 elements
// (`vec` elements per cell).  The first pass reads the f32 histogram H (and
// re-zeroes it) and writes T; later passes run in place on T.
cudaError_t prefix_table(uint4* H, uint4* T, int ndim, const int64_t* dims, int64_t cells, int vec,
                         cudaStream_t st, unsigned long long* H16 = nullptr,
                         const uint32_t* flag = nullptr, bool h_f32 = true, int skip_leading = 0,
                         uint4* sideH = nullptr, uint4* sideT = nullptr, int side_len = 0,
                         bool hf_u32 = false) {
  int fused = 0;  // trailing dims already scanned by the first pass
  if (H16 && ndim >= 2 &&
      (size_t)dims[ndim - 1] * dims[ndim - 2] * sizeof(uint4) <= kSlabSmemMax) {
    const int rows = (int)dims[ndim - 2], cols = (int)dims[ndim - 1];
    const int64_t n_slabs = cells / ((int64_t)rows * cols);
    // split a slab across two CTAs when there are too few slabs to fill the GPU
    const int parts = (cols >= 64 && n_slabs < 2 * sm_count()) ? 2 : 1;
    const size_t smem = (size_t)rows * ((cols + parts - 1) / parts) * sizeof(uint4);
    static SmemAttr smem_set;
    cudaError_t e = ensure_smem(slab_first_kernel, smem_set, (size_t)kSlabSmemMax);
    if (e != cudaSuccess) return e;
    const int64_t blocks = std::min<int64_t>(n_slabs * parts, (int64_t)sm_count() * 4);
    // with two CTAs per slab each reads whole rows, so neither may re-zero
    // the histogram in place (the other may not have read it yet): re-zero
    // after the pass instead
    slab_first_kernel<<<(unsigned)blocks, 1024, smem, st>>>(H16, H, flag, T, n_slabs, rows, cols,
                                                            sideH, sideT, side_len, parts,
                                                            parts == 1 ? 1 : 0, hf_u32 ? 1 : 0);
    e = cudaGetLastError();
    if (e == cudaSuccess && parts > 1) {
      e = cudaMemsetAsync(H16, 0, (size_t)cells * 8, st);
      if (e == cudaSuccess) {
        const int64_t zb = std::max<int64_t>(1, std::min<int64_t>((cells + 255) / 256, (int64_t)sm_count() * 8));
        zero_if_flag_kernel<<<(unsigned)zb, 256, 0, st>>>(H, cells, flag);
        e = cudaGetLastError();
      }
    }
    if (e != cudaSuccess || ndim - skip_leading == 2) return e;
    fused = 2;
  } else if (H16) {  // main table: packed first pass along the last dim (vec == 1)
    const int64_t len = ndim == 0 ? 1 : dims[ndim - 1];
    const int64_t rows = cells / len;
    int64_t blocks = (rows * 32 + 255) / 256;
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 16));
    rowscan_first_kernel<<<(unsigned)blocks, 256, 0, st>>>(H16, H, flag, T, rows, (int)len, hf_u32 ? 1 : 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || ndim <= 1) return e;
    fused = 1;
  } else if (ndim == 0) {  // a single cell: convert, copy and re-zero
    rowscan_kernel<<<1, 32, 0, st>>>(H, T, vec, 1, h_f32 ? 1 : 0);
    return cudaGetLastError();
  }
  int64_t inner = vec;
  uint4* src = H;
  for (int q = 0; q < fused; ++q) inner *= dims[ndim - 1 - q];
  if (fused) src = T;
  for (int d = ndim - 1 - fused; d >= skip_leading; --d) {
    const int64_t len = dims[d];
    const int64_t outer = cells * vec / (len * inner);
    const int from_f32 = (src == H && h_f32) ? 1 : 0;
    if (inner == 1) {
      int64_t blocks = (outer * 32 + 255) / 256;
      blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 16));
      rowscan_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, T, outer, (int)len, from_f32);
    } else {
      const size_t smem = (size_t)kColChunk * kColTile * sizeof(uint4);
      static SmemAttr smem_set;
      cudaError_t e = ensure_smem(colscan_kernel, smem_set, smem);
      if (e != cudaSuccess) return e;
      const int64_t tiles = outer * ((inner + kColTile - 1) / kColTile);
      const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count() * 8));
      colscan_kernel<<<(unsigned)blocks, 256, smem, st>>>(src, T, outer, len, inner, from_f32);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    src = T;
    inner *= len;
  }
  return cudaSuccess;
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" int gs_grid_plan(int64_t n_rec, int32_t n_models, const int32_t* grid_len,
                            gs_grid_info* info) {
  if (!info) return GS_EINVAL;
  Plan p;
  int rc = make_plan(n_rec, n_models, grid_len, &p);
  if (rc != GS_OK) return rc;
  info->n_configs = p.n_configs;
  info->n_cells = p.cellsF;
  info->side_cells = p.cellsP;
  info->n_structures = p.n_struct;
  info->max_len = p.M;
  info->workspace_bytes = p.bytes;
  info->fast_path = p.g4 ? (grid4_layout(p.glen, n_rec).sorted ? 2 : 1) : 0;
  if (p.g4) {
    info->build_launches = 2;  // g4_sort + g4_gather (one-shot) or g4_hist + g4_plane
    info->eval_launches = 1;   // g4_eval
  } else if (p.w5) {
    info->build_launches = 5;  // w5_bin, w5_scan, w5_scatter, w5_slab (two variants)
    info->eval_launches = 2;   // w5_walk + the regular eval
  } else {
    // mirrors gs_grid_build / prefix_table / gs_grid_eval below
    int b = 1 + (n_rec >= 65536 ? 1 : 0);
    const bool slab = p.D >= 2 && (size_t)p.dims[p.D - 1] * p.dims[p.D - 2] * sizeof(uint4) <= kSlabSmemMax;
    const int skip = p.walk ? 1 : 0;
    if (p.D == 0) b += 1;
    else if (slab) {
      const int64_t n_slabs = p.cellsF / (p.dims[p.D - 1] * p.dims[p.D - 2]);
      const bool two = p.dims[p.D - 1] >= 64 && n_slabs < 2 * sm_count();
      b += 1 + (two ? 1 : 0) + std::max(0, p.D - 2 - skip);  // + zero_if_flag after a split pass
    }
    else b += 1 + std::max(0, p.D - 1 - skip);
    const bool fold_side = p.DP == 1 && p.NVP == 1 && slab;
    if (p.DP > 0 && !fold_side) b += std::max(1, p.DP);
    info->build_launches = b;
    info->eval_launches = (p.walk || (p.M == 5 && p.glen[3] <= kFull5MaxRow)) ? 2 : 1;
  }
  return GS_OK;
}

extern "C" int gs_grid_build(const double* certainty, const uint8_t* correct, int64_t n_rec,
                             int32_t n_models, const double* grids, const int32_t* grid_len,
                             void* workspace, size_t workspace_bytes, int32_t flags,
                             void* stream) {
  Plan p;
  int rc = make_plan(n_rec, n_models, grid_len, &p);
  if (rc != GS_OK) return rc;
  GS_REQUIRE(certainty && correct && grids);
  if (!workspace || workspace_bytes < p.bytes) return GS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const int passes = (flags & (GS_GRID_BUILD_RECORDS_PASS | GS_GRID_BUILD_TABLES_PASS)) == 0
                         ? 3
                         : ((flags & GS_GRID_BUILD_RECORDS_PASS) ? 1 : 0) |
                               ((flags & GS_GRID_BUILD_TABLES_PASS) ? 2 : 0);
  if (p.g4) {
    GS_CUDA_TRY(grid4_build(certainty, correct, n_rec, grids, p.glen, ws,
                            (flags & GS_GRID_WORKSPACE_DIRTY) != 0, passes, st));
    return GS_OK;
  }
  if (passes != 3) return GS_EUNSUPPORTED;
  if (p.w5) {
    GS_CUDA_TRY(w5_build(certainty, correct, n_rec, grids, p.glen, ws,
                         (flags & GS_GRID_WORKSPACE_DIRTY) != 0, st));
    return GS_OK;
  }
  float* F = reinterpret_cast<float*>(ws + p.offHF);
  uint32_t* P = reinterpret_cast<uint32_t*>(ws + p.offHP);
  auto* H16 = reinterpret_cast<unsigned long long*>(ws + p.offH16);
  auto* flag = reinterpret_cast<uint32_t*>(ws + p.offFlag);
  GS_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(uint32_t), st));
  if (flags & GS_GRID_WORKSPACE_DIRTY) {
    GS_CUDA_TRY(cudaMemsetAsync(H16, 0, (size_t)p.cellsF * 8, st));
    GS_CUDA_TRY(cudaMemsetAsync(F, 0, (size_t)p.cellsF * 16, st));
    if (p.cellsP) GS_CUDA_TRY(cudaMemsetAsync(P, 0, (size_t)p.cellsP * p.NVP * 16, st));
  }

  HistArgs h{};
  h.cert = certainty;
  h.corr = correct;
  h.n_rec = n_rec;
  h.grids = grids;
  int off = 0;
  for (int j = 0; j < n_models; ++j) {
    h.goff[j] = off;
    h.glen[j] = p.glen[j];
    off += p.glen[j];
  }
  for (int j = 0; j < p.D; ++j) h.strideF[j] = p.strideF[j];
  for (int j = 0; j < p.DP; ++j) h.strideP[j] = p.strideP[j];
  h.cellsP = p.cellsP;
  h.grid_doubles = p.D > 0 ? h.goff[p.D - 1] + h.glen[p.D - 1] : 0;
  h.vec_ok = aligned16(certainty) && ((reinterpret_cast<uintptr_t>(correct) & 3u) == 0);
  const size_t side_bytes = (size_t)p.cellsP * p.NVP * 16;
  h.priv = p.DP > 0 && side_bytes <= kSidePrivMax;
  h.F = F;
  h.P = P;
  h.H16 = H16;
  h.flag = flag;
  h.f_u32 = n_rec >= kMaxExactF32 ? 1 : 0;
  const size_t smem = (size_t)h.grid_doubles * sizeof(double) + (size_t)p.D * kLutBuckets * 4 +
                      (h.priv ? side_bytes : 0) + 16;
  if (smem > 200 * 1024) return GS_EUNSUPPORTED;
  const int64_t imax = std::max<int64_t>(p.cellsF * 4, p.cellsP * p.NVP * 4);
  cudaError_t e = cudaSuccess;
  switch (n_models) {
    case 1: e = launch_hist<1>(h, n_rec, smem, imax, st); break;
    case 2: e = launch_hist<2>(h, n_rec, smem, imax, st); break;
    case 3: e = launch_hist<3>(h, n_rec, smem, imax, st); break;
    case 4: e = launch_hist<4>(h, n_rec, smem, imax, st); break;
    case 5: e = launch_hist<5>(h, n_rec, smem, imax, st); break;
    case 6: e = launch_hist<6>(h, n_rec, smem, imax, st); break;
    case 7: e = launch_hist<7>(h, n_rec, smem, imax, st); break;
    case 8: e = launch_hist<8>(h, n_rec, smem, imax, st); break;
    default: return GS_EUNSUPPORTED;
  }
  GS_CUDA_TRY(e);
  // with the fused walk the b_0 prefix is taken inside gs_grid_eval
  // a 1-D side table (4 models) is scanned inside the slab pass
  const bool fold_side = p.DP == 1 && p.NVP == 1 && p.D >= 2 &&
                         (size_t)p.dims[p.D - 1] * p.dims[p.D - 2] * sizeof(uint4) <= kSlabSmemMax;
  GS_CUDA_TRY(prefix_table(reinterpret_cast<uint4*>(F), reinterpret_cast<uint4*>(ws + p.offF), p.D,
                           p.dims, p.cellsF, 1, st, H16, flag, true, p.walk ? 1 : 0,
                           fold_side ? reinterpret_cast<uint4*>(P) : nullptr,
                           fold_side ? reinterpret_cast<uint4*>(ws + p.offP) : nullptr,
                           fold_side ? (int)p.cellsP : 0, n_rec >= kMaxExactF32));
  if (p.DP > 0 && !fold_side)
    GS_CUDA_TRY(prefix_table(reinterpret_cast<uint4*>(P), reinterpret_cast<uint4*>(ws + p.offP), p.DP,
                             p.dims, p.cellsP, p.NVP, st, nullptr, nullptr, false));
  return GS_OK;
}

extern "C" int gs_grid_accumulate(const double* certainty, const uint8_t* correct, int64_t n_chunk,
                                  int64_t n_rec, int32_t n_models, const double* grids,
                                  const int32_t* grid_len, void* workspace, size_t workspace_bytes,
                                  int32_t flags, void* stream) {
  Plan p;
  int rc = make_plan(n_rec, n_models, grid_len, &p);
  if (rc != GS_OK) return rc;
  if (!p.g4) return GS_EUNSUPPORTED;
  GS_REQUIRE(n_chunk >= 0 && n_chunk <= n_rec && grids && (n_chunk == 0 || (certainty && correct)));
  if (!workspace || workspace_bytes < p.bytes) return GS_EWORKSPACE;
  GS_CUDA_TRY(grid4_accumulate(certainty, correct, n_chunk, grids, p.glen,
                               static_cast<uint8_t*>(workspace),
                               (flags & GS_GRID_WORKSPACE_DIRTY) != 0,
                               static_cast<cudaStream_t>(stream)));
  return GS_OK;
}

extern "C" int gs_grid_finish(int64_t n_rec, int32_t n_models, const int32_t* grid_len,
                              void* workspace, size_t workspace_bytes, void* stream) {
  Plan p;
  int rc = make_plan(n_rec, n_models, grid_len, &p);
  if (rc != GS_OK) return rc;
  if (!p.g4) return GS_EUNSUPPORTED;
  if (!workspace || workspace_bytes < p.bytes) return GS_EWORKSPACE;
  GS_CUDA_TRY(grid4_finish(p.glen, static_cast<uint8_t*>(workspace),
                           static_cast<cudaStream_t>(stream)));
  return GS_OK;
}

extern "C" int gs_grid_eval(int64_t n_rec, int32_t n_models, const int32_t* grid_len,
                            const double* cost1, int64_t config_begin, int64_t config_count,
                            double* accuracy, double* mean_cost, double* forward_frac,
                            uint32_t* n_correct, const void* workspace, size_t workspace_bytes,
                            void* stream) {
  Plan p;
  int rc = make_plan(n_rec, n_models, grid_len, &p);
  if (rc != GS_OK) return rc;
  GS_REQUIRE(cost1 && config_begin >= 0 && config_count >= 0 &&
             config_begin + config_count <= p.n_configs);
  if (config_count == 0) return GS_OK;
  if (!workspace || workspace_bytes < p.bytes) return GS_EWORKSPACE;
  // vector stores need 16-byte aligned outputs
  if ((accuracy && !aligned16(accuracy)) || (mean_cost && !aligned16(mean_cost)) ||
      (n_correct && !aligned16(n_correct)) || (forward_frac && !aligned16(forward_frac)))
    return GS_EINVAL;
  if (p.g4) {
    GS_CUDA_TRY(grid4_eval(n_rec, p.glen, p.struct_begin, p.struct_mask, p.n_struct, cost1,
                           config_begin, config_count, accuracy, mean_cost, forward_frac, n_correct,
                           static_cast<const uint8_t*>(workspace), static_cast<cudaStream_t>(stream)));
    return GS_OK;
  }
  EvalGridArgs a{};
  a.M = p.M;
  a.n_struct = p.n_struct;
  a.NVP = p.NVP;
  a.DP = p.DP;
  for (int j = 0; j < p.M; ++j) a.glen[j] = p.glen[j];
  for (int j = 0; j < p.D; ++j) a.strideF[j] = p.strideF[j];
  for (int j = 0; j < p.DP; ++j) a.strideP[j] = p.strideP[j];
  a.n_rec = n_rec;
  a.rcp_n = rcp_of(n_rec);
  a.cellsF = p.cellsF;
  a.cellsP = p.cellsP;
  a.cfg_begin = config_begin;
  a.cfg_count = config_count;
  for (int s = 0; s <= p.n_struct; ++s) a.struct_begin[s] = p.struct_begin[s];
  for (int s = 0; s < p.n_struct; ++s) a.struct_mask[s] = p.struct_mask[s];
  // rows: configs sharing all thresholds but the last forwarding stage's
  int64_t rows = 0;
  for (int s = 0; s < p.n_struct; ++s) {
    a.row_begin[s] = rows;
    rows += (p.struct_begin[s + 1] - p.struct_begin[s]) / row_len(p, s);
  }
  a.row_begin[p.n_struct] = rows;
  const uint8_t* ws = static_cast<const uint8_t*>(workspace);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t reg_end = config_begin + config_count;  // regular eval covers [config_begin, reg_end)
  if (p.walk) {
    WalkArgs w{};
    w.d0 = (int32_t)p.dims[0];
    w.d1 = (int32_t)p.dims[1];
    w.d2 = (int32_t)p.dims[2];
    w.sb = p.struct_begin[p.n_struct - 1];
    w.cfg_begin = config_begin;
    w.cfg_count = config_count;
    w.n_rec = n_rec;
    w.rcp_n = rcp_of(n_rec);
    w.cost1 = cost1;
    w.S = reinterpret_cast<const uint4*>(ws + p.offF);
    w.faces = reinterpret_cast<uint4*>(const_cast<uint8_t*>(ws) + p.offFaces);
    w.Pside = reinterpret_cast<const uint4*>(ws + p.offP);
    w.acc = accuracy;
    w.cost = mean_cost;
    w.frac = forward_frac;
    w.n_correct = n_correct;
    w.tile = std::min(kWalkTile, w.d2);
    const size_t smem = (size_t)w.d0 * w.tile * sizeof(uint4);
    static SmemAttr smem_set;
    GS_CUDA_TRY(ensure_smem(walk_eval_kernel, smem_set, (size_t)kWalkMaxSteps * kWalkTile * sizeof(uint4)));
    const int plane = w.d1 * w.d2;
    const int threads = (w.tile * kWalkGroups + 31) / 32 * 32;
    walk_eval_kernel<<<(plane + w.tile - 1) / w.tile, threads, smem, st>>>(w);
    GS_LAUNCH_CHECK();
    reg_end = std::min<int64_t>(reg_end, w.sb);
    if (reg_end <= config_begin) return GS_OK;
  }
  if (p.w5) {
    // the b_0 walk scores the full cascade and leaves the face cells the
    // regular eval reads (it runs even when the range holds no full-cascade
    // config)
    const int64_t sb = p.struct_begin[p.n_struct - 1];
    GS_CUDA_TRY(w5_walk(n_rec, p.glen, sb, cost1, config_begin, config_count, accuracy, mean_cost,
                        forward_frac, n_correct, ws, st));
    reg_end = std::min<int64_t>(reg_end, sb);
    if (reg_end <= config_begin) return GS_OK;
  } else if (p.M == 5 && p.glen[3] <= kFull5MaxRow && p.cellsP > 0) {
    // the full cascade (the last structure): full5_eval_kernel
    Full5Args f{};
    f.g0 = p.glen[0];
    f.g1 = p.glen[1];
    f.g2 = p.glen[2];
    f.g3 = p.glen[3];
    f.d1 = (int32_t)p.dims[1];
    f.sF0 = p.strideF[0];
    f.sF1 = p.strideF[1];
    f.sF2 = p.strideF[2];
    f.sb = p.struct_begin[p.n_struct - 1];
    f.cfg_begin = config_begin;
    f.cfg_count = config_count;
    f.n_rec = n_rec;
    f.rcp_n = rcp_of(n_rec);
    f.cost1 = cost1;
    f.F = reinterpret_cast<const uint4*>(ws + p.offF);
    f.P = reinterpret_cast<const uint4*>(ws + p.offP);
    f.acc = accuracy;
    f.cost = mean_cost;
    f.frac = forward_frac;
    f.n_correct = n_correct;
    if (config_begin + config_count > f.sb) {
      full5_eval_kernel<<<(unsigned)((int64_t)f.g0 * f.g1), kFull5Threads, 0, st>>>(f);
      GS_LAUNCH_CHECK();
    }
    reg_end = std::min<int64_t>(reg_end, f.sb);
    if (reg_end <= config_begin) return GS_OK;
  }
  a.cfg_count = reg_end - config_begin;
  a.row_lo = global_row(p, a.row_begin, config_begin);
  a.row_hi = global_row(p, a.row_begin, reg_end - 1) + 1;
  a.F = reinterpret_cast<const uint4*>(ws + ((p.walk || p.w5) ? p.offFaces : p.offF));
  a.P = reinterpret_cast<const uint4*>(ws + p.offP);
  a.cost1 = cost1;
  a.acc = accuracy;
  a.cost = mean_cost;
  a.frac = forward_frac;
  a.n_correct = n_correct;
  cudaError_t e = cudaSuccess;
  switch (n_models) {
    case 1: e = launch_grid_eval<1>(a, st); break;
    case 2: e = launch_grid_eval<2>(a, st); break;
    case 3: e = launch_grid_eval<3>(a, st); break;
    case 4: e = launch_grid_eval<4>(a, st); break;
    case 5: e = launch_grid_eval<5>(a, st); break;
    case 6: e = launch_grid_eval<6>(a, st); break;
    case 7: e = launch_grid_eval<7>(a, st); break;
    case 8: e = launch_grid_eval<8>(a, st); break;
    default: return GS_EUNSUPPORTED;
  }
  GS_CUDA_TRY(e);
  return GS_OK;
}

extern "C" int gs_grid_decode(int32_t n_models, const int32_t* grid_len, const double* grids,
                              const int64_t* config_idx, int64_t count, int32_t* stage_model,
                              double* thresholds, int32_t* n_stages, void* stream) {
  Plan p;
  int rc = make_plan(1, n_models, grid_len, &p);
  if (rc != GS_OK) return rc;
  if (count == 0) return GS_OK;
  GS_REQUIRE(count > 0 && grids && config_idx && stage_model && thresholds && n_stages);
  DecodeArgs a{};
  a.M = p.M;
  a.n_struct = p.n_struct;
  int off = 0;
  for (int j = 0; j < p.M; ++j) {
    a.glen[j] = p.glen[j];
    a.goff[j] = off;
    off += p.glen[j];
  }
  for (int s = 0; s <= p.n_struct; ++s) a.struct_begin[s] = p.struct_begin[s];
  for (int s = 0; s < p.n_struct; ++s) a.struct_mask[s] = p.struct_mask[s];
  a.grids = grids;
  a.idx = config_idx;
  a.count = count;
  a.stage_model = stage_model;
  a.thr = thresholds;
  a.n_stages = n_stages;
  int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, (int64_t)sm_count() * 16));
  grid_decode_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  GS_LAUNCH_CHECK();
  return GS_OK;
}
