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
// Table layout.  A correct count c_j is only ever read at positions whose
// dimensions > j are at "any", so:
//   main table F over dims 0..M-2, channels {cnt, c_{M-1}, c_{M-2}};
//   side table S over dims 0..M-3, channels {c_0 .. c_{M-3}}.
// Channels are packed as fields of B = bitlen(n_rec) bits into u64 words
// (three per word while n_rec < 2^21).  Every count — histogram or prefix —
// is <= n_rec < 2^B, so packed words add without carries: the histogram is
// one 64-bit L2 atomic per record per table, and the prefix sums add whole
// words.  (Random-scatter L2 atomic throughput bounds the histogram, so
// packing three counts into one op matters more than anything else there.)
// Histogram and prefix live in separate buffers: the first scan pass reads
// the histogram, writes the prefix and re-zeroes the histogram, so no
// memset runs per build (the caller zeroes the workspace once).
//
// Kernels: grid_hist (one pass over the records), rowscan (contiguous last
// dim, warp-shuffle scan), colscan (strided dims: [128 x 32]-element tiles in
// shared memory, two-level scan), grid_eval (one warp per "row" of configs
// sharing every threshold but the last forwarding one; f64 epilogue in the
// reference's order with non-contracted multiply/add).
#include <algorithm>
#include <atomic>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kMaxM = GS_MAX_MODELS;
constexpr int64_t kMaxRec = 1ll << 24;
constexpr int kHistThreads = 512;
constexpr size_t kSidePrivMax = 32 * 1024;
constexpr int kMaxWF = 2;  // words per main-table cell
constexpr int kMaxWS = 3;  // words per side-table cell

struct Plan {
  int M = 0, D = 0, DS = 0, n_struct = 0;
  int B = 0, F = 0, WF = 0, WS = 0;
  int glen[kMaxM] = {};
  int64_t dims[kMaxM] = {};
  int64_t strideF[kMaxM] = {};
  int64_t strideS[kMaxM] = {};
  int64_t cellsF = 1, cellsS = 0;
  int64_t n_configs = 0;
  int64_t struct_begin[256 + 1] = {};
  uint32_t struct_mask[256] = {};
  size_t offHF = 0, offF = 0, offHS = 0, offS = 0, bytes = 0;
  // bucketed build: records grouped by b_0, one CTA per b_0 slab
  bool bucket = false;
  int64_t d0 = 0, slab_cells = 0, side_slab = 0, cap = 0;
  size_t offBk = 0, offCur = 0;
};

constexpr size_t kSlabSmemMax = 160 * 1024;
constexpr double kBucketBytesMax = 4.0e9;

int make_plan(int64_t n_rec, int32_t M, const int32_t* grid_len, Plan* p) {
  if (M < 1 || !grid_len || n_rec < 1) return GS_EINVAL;
  if (M > kMaxM || n_rec >= kMaxRec) return GS_EUNSUPPORTED;
  p->M = M;
  p->D = M - 1;
  p->DS = M >= 3 ? M - 2 : 0;
  for (int j = 0; j < M; ++j) {
    if (grid_len[j] < 1 || grid_len[j] > (1 << 20)) return GS_EINVAL;
    p->glen[j] = grid_len[j];
  }
  // field width: 21 bits (three fields per word) while every count fits
  p->B = n_rec < ((int64_t)1 << 21) ? 21 : 32;
  p->F = 64 / p->B;
  p->WF = (3 + p->F - 1) / p->F;
  p->WS = p->DS > 0 ? (M - 2 + p->F - 1) / p->F : 0;
  if (p->WF > kMaxWF || p->WS > kMaxWS) return GS_EUNSUPPORTED;
  double cells = 1.0;
  for (int j = 0; j < p->D; ++j) {
    p->dims[j] = (int64_t)p->glen[j] + 1;
    cells *= (double)p->dims[j];
  }
  if (cells * 16.0 * p->WF > 1.4e11) return GS_EUNSUPPORTED;
  int64_t s = 1;
  for (int j = p->D - 1; j >= 0; --j) {
    p->strideF[j] = s;
    s *= p->dims[j];
  }
  p->cellsF = s;
  s = 1;
  for (int j = p->DS - 1; j >= 0; --j) {
    p->strideS[j] = s;
    s *= p->dims[j];
  }
  p->cellsS = p->DS > 0 ? s : 0;
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
  const size_t bF = round_up((size_t)p->cellsF * p->WF * 8, 256);
  const size_t bS = round_up((size_t)p->cellsS * p->WS * 8, 256);
  // bucketed build when a b_0 slab (dims 1..M-2, at most two of them) and its
  // side-table row fit in shared memory
  if (p->D >= 2 && p->D <= 3) {
    p->d0 = p->dims[0];
    p->slab_cells = p->cellsF / p->d0;
    p->side_slab = p->DS > 0 ? p->cellsS / p->d0 : 0;
    p->cap = n_rec;
    const size_t smem = (size_t)(p->slab_cells * p->WF + p->side_slab * p->WS) * 8;
    p->bucket = smem <= kSlabSmemMax && p->slab_cells < (1 << 24) &&
                (double)p->d0 * (double)p->cap * 4.0 <= kBucketBytesMax;
  }
  if (p->bucket) {
    p->offF = 0;
    p->offS = bF;
    p->offBk = bF + bS;
    p->offCur = p->offBk + round_up((size_t)p->d0 * p->cap * 4, 256);
    p->bytes = p->offCur + round_up((size_t)p->d0 * 4, 256);
    p->offHF = p->offHS = 0;  // unused
  } else {
    p->offHF = 0;
    p->offF = bF;
    p->offHS = 2 * bF;
    p->offS = 2 * bF + bS;
    p->bytes = 2 * bF + 2 * bS;
  }
  return GS_OK;
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

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size,
// so later calls (e.g. inside a CUDA-graph capture) issue no attribute calls.
template <typename Kernel>
cudaError_t ensure_smem(Kernel k, std::atomic<int>& done, size_t bytes) {
  if ((int)bytes <= done.load(std::memory_order_acquire)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.store((int)bytes, std::memory_order_release);
  return e;
}

// ------------------------------------------------------------------ hist --
struct HistArgs {
  const double* cert;
  const uint8_t* corr;
  int32_t n_rec;
  const double* grids;
  int32_t glen[kMaxM];
  int64_t strideF[kMaxM];
  int64_t strideS[kMaxM];
  int64_t cellsS;
  int32_t B, F, WF, WS;
  int32_t grid_doubles;  // grids of models 0..M-2 staged in smem
  int32_t vec_ok;
  int32_t priv;          // side table privatised in shared memory
  unsigned long long* HF;
  unsigned long long* HS;
};

template <int M, int PB, typename Cell>
__global__ void __launch_bounds__(kHistThreads) grid_hist_kernel(const __grid_constant__ HistArgs a) {
  constexpr int PF = 64 / PB;  // packed fields per word
  constexpr int D = M - 1;
  constexpr int DS = M >= 3 ? M - 2 : 0;
  extern __shared__ __align__(16) double s_grid[];
  unsigned long long* s_side = reinterpret_cast<unsigned long long*>(s_grid + a.grid_doubles);
  for (int i = threadIdx.x; i < a.grid_doubles; i += blockDim.x) s_grid[i] = a.grids[i];
  if (DS > 0 && a.priv)
    for (int64_t i = threadIdx.x; i < a.cellsS * a.WS; i += blockDim.x) s_side[i] = 0ull;
  __syncthreads();

  const int step = gridDim.x * blockDim.x;  // n_rec < 2^24, M <= 8: 32-bit offsets
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n_rec; r += step) {
    double x[M];
    uint32_t k[M];
    const double* row = a.cert + r * M;
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
      for (int j = 0; j < M; ++j) k[j] = (w >> (8 * j)) & 0xffu;
    } else {
#pragma unroll
      for (int j = 0; j < M; ++j) k[j] = __ldg(a.corr + r * M + j) != 0;
    }
#pragma unroll
    for (int j = 0; j < M; ++j) k[j] = k[j] != 0;
    Cell cellF = 0, cellS = 0;
    int off = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int b = upper_count(s_grid + off, a.glen[j], x[j]);
      off += a.glen[j];
      cellF += (Cell)b * (Cell)a.strideF[j];
      if (j < DS) cellS += (Cell)b * (Cell)a.strideS[j];
    }
    // main table: fields {cnt, c_{M-1}, c_{M-2}}
    unsigned long long wf[kMaxWF] = {0ull, 0ull};
    {
      const uint32_t f[3] = {1u, k[M - 1], M >= 2 ? k[M >= 2 ? M - 2 : 0] : 0u};
#pragma unroll
      for (int c = 0; c < 3; ++c) wf[c / PF] += (unsigned long long)f[c] << ((c % PF) * PB);
    }
#pragma unroll
    for (int w = 0; w < kMaxWF; ++w)
      if (w < a.WF && wf[w]) atomicAdd(a.HF + (Cell)cellF * a.WF + w, wf[w]);
    // side table: fields {c_0 .. c_{M-3}}
    if constexpr (DS > 0) {
      unsigned long long ws[kMaxWS] = {0ull, 0ull, 0ull};
#pragma unroll
      for (int j = 0; j < DS; ++j) ws[j / PF] += (unsigned long long)k[j] << ((j % PF) * PB);
#pragma unroll
      for (int w = 0; w < kMaxWS; ++w) {
        if (w >= a.WS || !ws[w]) continue;
        if (a.priv)
          atomicAdd(s_side + (Cell)cellS * a.WS + w, ws[w]);
        else
          atomicAdd(a.HS + (Cell)cellS * a.WS + w, ws[w]);
      }
    }
  }
  if (DS > 0 && a.priv) {
    __syncthreads();
    for (int64_t i = threadIdx.x; i < a.cellsS * a.WS; i += blockDim.x) {
      const unsigned long long c = s_side[i];
      if (c) atomicAdd(a.HS + i, c);
    }
  }
}

// ------------------------------------------------------- bucketed build --
// Pass 1 (bucket_scatter): bin every record and append a 32-bit payload
// (cell inside its b_0 slab | correct bits << 24) to bucket b_0.  A CTA ranks
// its chunk per bucket with shared-memory counters and reserves each
// bucket's range with ONE global atomic per (chunk, bucket); order inside a
// bucket is irrelevant (counts are order-free).
// Pass 2 (slab_hist): one CTA per b_0 slab accumulates the slab's main-table
// cells and side-table row with shared-memory atomics, takes the prefix over
// the slab's own dimensions in shared memory and writes both out.  The only
// remaining global pass is the prefix along b_0 (colscan).
struct BucketArgs {
  const double* cert;
  const uint8_t* corr;
  int32_t n_rec;
  const double* grids;
  int32_t glen[kMaxM];
  int64_t strideF[kMaxM];
  int32_t d0;
  int64_t cap;
  int32_t grid_doubles;
  int32_t vec_ok;
  uint32_t* buckets;
  uint32_t* cursor;
};

constexpr int kScatterThreads = 512;
constexpr int kScatterR = 4;  // records per thread per chunk

template <int M>
__global__ void __launch_bounds__(kScatterThreads) bucket_scatter_kernel(const __grid_constant__ BucketArgs a) {
  constexpr int D = M - 1;
  extern __shared__ __align__(16) double s_grid[];
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_grid + a.grid_doubles);
  uint32_t* s_base = s_cnt + a.d0;
  for (int i = threadIdx.x; i < a.grid_doubles; i += blockDim.x) s_grid[i] = a.grids[i];
  for (int i = threadIdx.x; i < a.d0; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int chunk = blockDim.x * kScatterR;
  for (int c0 = blockIdx.x * chunk; c0 < a.n_rec; c0 += gridDim.x * chunk) {
    uint32_t pay[kScatterR], rank[kScatterR];
    int b0[kScatterR];
#pragma unroll
    for (int u = 0; u < kScatterR; ++u) {
      const int r = c0 + u * blockDim.x + threadIdx.x;
      b0[u] = -1;
      if (r >= a.n_rec) continue;
      double x[M];
      uint32_t k[M];
      const double* row = a.cert + r * M;
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
        for (int j = 0; j < M; ++j) k[j] = __ldg(a.corr + r * M + j) != 0;
      }
      uint32_t cell = 0, bits = 0;
      int off = 0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const int b = upper_count(s_grid + off, a.glen[j], x[j]);
        off += a.glen[j];
        if (j == 0)
          b0[u] = b;
        else
          cell += (uint32_t)b * (uint32_t)a.strideF[j];
      }
#pragma unroll
      for (int j = 0; j < M; ++j) bits |= k[j] << j;
      pay[u] = cell | (bits << 24);
      rank[u] = atomicAdd(s_cnt + b0[u], 1u);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < a.d0; t += blockDim.x) {
      const uint32_t c = s_cnt[t];
      if (c) {
        s_base[t] = atomicAdd(a.cursor + t, c);
        s_cnt[t] = 0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kScatterR; ++u)
      if (b0[u] >= 0) a.buckets[(int64_t)b0[u] * a.cap + s_base[b0[u]] + rank[u]] = pay[u];
    __syncthreads();
  }
}

struct SlabArgs {
  int32_t d0, rows, cols;       // slab = [rows][cols] cells (rows = 1 for a 1-D slab)
  int32_t side_cells, side_div;  // side row cells; slab cell / side_div = side cell
  int64_t cap;
  const uint32_t* buckets;
  uint32_t* cursor;
  unsigned long long* Ft;
  unsigned long long* St;
};

// inclusive prefix of `len` u64 elements (stride `step`) by one warp
__device__ __forceinline__ void warp_scan_line(unsigned long long* p, int len, int step) {
  const int lane = (int)lane_id();
  unsigned long long carry = 0;
  for (int base = 0; base < len; base += 128) {
    unsigned long long e[4], tot = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = base + lane * 4 + u;
      e[u] = c < len ? p[c * step] : 0ull;
      tot += e[u];
      e[u] = tot;
    }
    unsigned long long incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned long long excl = carry + incl - tot;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = base + lane * 4 + u;
      if (c < len) p[c * step] = e[u] + excl;
    }
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
}

template <int M, int PB>
__global__ void __launch_bounds__(1024) slab_hist_kernel(const __grid_constant__ SlabArgs a) {
  constexpr int PF = 64 / PB;
  constexpr int WF = (3 + PF - 1) / PF;
  constexpr int DS = M >= 3 ? M - 2 : 0;
  constexpr int WS = DS > 0 ? (DS + PF - 1) / PF : 0;
  extern __shared__ __align__(16) unsigned long long s_slab[];
  const int slab_words = a.rows * a.cols * WF;
  unsigned long long* s_side = s_slab + slab_words;
  const int side_words = a.side_cells * WS;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int b0 = blockIdx.x; b0 < a.d0; b0 += gridDim.x) {
    for (int i = threadIdx.x; i < slab_words + side_words; i += blockDim.x) s_slab[i] = 0ull;
    __syncthreads();
    const uint32_t n = a.cursor[b0];
    const uint32_t* src = a.buckets + (int64_t)b0 * a.cap;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t p = __ldg(src + i);
      const uint32_t cell = p & 0xffffffu, bits = p >> 24;
      unsigned long long wf[WF];
#pragma unroll
      for (int w = 0; w < WF; ++w) wf[w] = 0ull;
      const uint32_t f[3] = {1u, (bits >> (M - 1)) & 1u, M >= 2 ? (bits >> (M >= 2 ? M - 2 : 0)) & 1u : 0u};
#pragma unroll
      for (int c = 0; c < 3; ++c) wf[c / PF] += (unsigned long long)f[c] << ((c % PF) * PB);
#pragma unroll
      for (int w = 0; w < WF; ++w)
        if (wf[w]) atomicAdd(s_slab + cell * WF + w, wf[w]);
      if constexpr (DS > 0) {
        unsigned long long ws[WS > 0 ? WS : 1];
#pragma unroll
        for (int w = 0; w < WS; ++w) ws[w] = 0ull;
#pragma unroll
        for (int j = 0; j < DS; ++j) ws[j / PF] += (unsigned long long)((bits >> j) & 1u) << ((j % PF) * PB);
        const uint32_t sc = cell / (uint32_t)a.side_div;
#pragma unroll
        for (int w = 0; w < WS; ++w)
          if (ws[w]) atomicAdd(s_side + sc * WS + w, ws[w]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) a.cursor[b0] = 0;  // leave the cursors zero for the next build
    // prefix along cols (each row, each word), then along rows (each col, each word)
    for (int t = warp; t < a.rows * WF; t += nwarps)
      warp_scan_line(s_slab + (t / WF) * a.cols * WF + (t % WF), a.cols, WF);
    __syncthreads();
    if (a.rows > 1) {
      for (int t = threadIdx.x; t < a.cols * WF; t += blockDim.x) {
        unsigned long long acc = 0;
        unsigned long long* p = s_slab + t;
        for (int r = 0; r < a.rows; ++r) {
          acc += p[(int64_t)r * a.cols * WF];
          p[(int64_t)r * a.cols * WF] = acc;
        }
      }
    }
    if (DS > 0 && a.side_cells > 1)
      for (int t = warp; t < WS; t += nwarps) warp_scan_line(s_side + t, a.side_cells, WS);
    __syncthreads();
    unsigned long long* dF = a.Ft + (int64_t)b0 * slab_words;
    for (int i = threadIdx.x; i < slab_words; i += blockDim.x) dF[i] = s_slab[i];
    if (DS > 0) {
      unsigned long long* dS = a.St + (int64_t)b0 * side_words;
      for (int i = threadIdx.x; i < side_words; i += blockDim.x) dS[i] = s_side[i];
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------- scans --
// Inclusive prefix along the contiguous last dimension (rows of `len` u64
// words): one warp per row, four consecutive words per lane, warp-shuffle
// scan.  When src != dst the source (the histogram) is zeroed after reading.
__global__ void __launch_bounds__(256) rowscan_kernel(unsigned long long* src,
                                                      unsigned long long* dst, int64_t n_rows,
                                                      int len) {
  const int lane = (int)lane_id();
  const bool zero = src != dst;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rows; r += nw) {
    unsigned long long* in = src + r * len;
    unsigned long long* out = dst + r * len;
    unsigned long long carry = 0;
    for (int base = 0; base < len; base += 128) {
      unsigned long long e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = base + lane * 4 + u;
        e[u] = c < len ? in[c] : 0ull;
      }
      if (zero) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = base + lane * 4 + u;
          if (c < len) in[c] = 0ull;
        }
      }
      unsigned long long tot = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        tot += e[u];
        e[u] = tot;
      }
      unsigned long long incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned long long excl = carry + incl - tot;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = base + lane * 4 + u;
        if (c < len) out[c] = e[u] + excl;
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

constexpr int kColTile = 32;    // consecutive inner elements per CTA
constexpr int kColChunk = 128;  // rows of the scanned dimension per smem pass
constexpr int kColSeg = 16;     // rows per scanning thread (8 segments x 32 columns)

// Inclusive prefix along a strided dimension of a u64 table viewed as
// [outer][len][inner].  A CTA owns kColTile consecutive inner elements of one
// outer index: it loads a [128 x 32] tile (16 independent loads per thread,
// one round trip), scans it in shared memory (each thread a 16-row segment
// of one column, then segment offsets), and writes it back coalesced.
__global__ void __launch_bounds__(256) colscan_kernel(unsigned long long* src,
                                                      unsigned long long* dst, int64_t outer,
                                                      int64_t len, int64_t inner) {
  __shared__ unsigned long long s[kColChunk][kColTile + 1];
  __shared__ unsigned long long s_seg[kColChunk / kColSeg][kColTile];
  const bool zero = src != dst;
  const int64_t tiles_per_outer = (inner + kColTile - 1) / kColTile;
  const int64_t n_tiles = outer * tiles_per_outer;
  const int t = threadIdx.x;
  const int col = t & (kColTile - 1);
  const int seg = t >> 5;  // 0..7
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t o = tile / tiles_per_outer;
    const int64_t i0 = (tile - o * tiles_per_outer) * kColTile;
    const int w = (int)min((int64_t)kColTile, inner - i0);
    unsigned long long* in = src + o * len * inner + i0;
    unsigned long long* out = dst + o * len * inner + i0;
    unsigned long long carry = 0;  // per column, kept by segment-7 threads' view via smem
    for (int64_t r0 = 0; r0 < len; r0 += kColChunk) {
      const int rows = (int)min((int64_t)kColChunk, len - r0);
      // load: thread (seg, col) loads rows seg, seg+8, ... of column col
      unsigned long long v[kColChunk / 8];
#pragma unroll
      for (int u = 0; u < kColChunk / 8; ++u) {
        const int rr = seg + 8 * u;
        v[u] = (rr < rows && col < w) ? in[(r0 + rr) * inner + col] : 0ull;
      }
      if (zero) {
#pragma unroll
        for (int u = 0; u < kColChunk / 8; ++u) {
          const int rr = seg + 8 * u;
          if (rr < rows && col < w) in[(r0 + rr) * inner + col] = 0ull;
        }
      }
#pragma unroll
      for (int u = 0; u < kColChunk / 8; ++u) s[seg + 8 * u][col] = v[u];
      __syncthreads();
      // segment scan: thread (seg, col) scans rows [seg*16, seg*16+16)
      unsigned long long acc = 0;
#pragma unroll
      for (int q = 0; q < kColSeg; ++q) {
        acc += s[seg * kColSeg + q][col];
        s[seg * kColSeg + q][col] = acc;
      }
      s_seg[seg][col] = acc;
      __syncthreads();
      unsigned long long total = carry;
#pragma unroll
      for (int q = 0; q < kColChunk / kColSeg; ++q) total += s_seg[q][col];
#pragma unroll
      for (int u = 0; u < kColChunk / 8; ++u) {
        const int rr = seg + 8 * u;
        if (rr < rows && col < w) {
          // rows of segment rr/16 get that segment's offset
          unsigned long long base = carry;
          for (int q = 0; q < rr / kColSeg; ++q) base += s_seg[q][col];
          out[(r0 + rr) * inner + col] = s[rr][col] + base;
        }
      }
      carry = total;
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
// configs kl = lane, lane+32, ... (four loads in flight) with one cell load,
// two f64 divisions and coalesced stores.
struct EvalGridArgs {
  int32_t M, n_struct, B, F, WF, WS, DS;
  int32_t glen[kMaxM];
  int64_t strideF[kMaxM];
  int64_t strideS[kMaxM];
  int64_t n_rec, cellsF, cellsS;
  int64_t cfg_begin, cfg_count;
  int64_t row_lo, row_hi;
  int64_t struct_begin[256 + 1];
  int64_t row_begin[256 + 1];
  uint32_t struct_mask[256];
  const unsigned long long* Ft;
  const unsigned long long* St;
  const double* cost1;
  double* acc;
  double* cost;
  double* frac;
  uint32_t* n_correct;
};

struct CellF {
  unsigned long long w[kMaxWF];
};
struct CellS {
  unsigned long long w[kMaxWS];
};

// field c of a packed cell (word chosen with selects, never a dynamic
// register-array index, so cells stay in registers)
template <int W>
__device__ __forceinline__ uint32_t fieldw(const unsigned long long (&w)[W], int c, int F, int B) {
  const int q = c / F;
  unsigned long long word = w[0];
#pragma unroll
  for (int i = 1; i < W; ++i) word = q == i ? w[i] : word;
  return (uint32_t)((word >> ((c - q * F) * B)) & ((1ull << B) - 1));
}

__device__ __forceinline__ CellF loadF(const EvalGridArgs& a, int64_t cell) {
  CellF v;
#pragma unroll
  for (int q = 0; q < kMaxWF; ++q) v.w[q] = q < a.WF ? __ldg(a.Ft + cell * a.WF + q) : 0ull;
  return v;
}
__device__ __forceinline__ CellS loadS(const EvalGridArgs& a, int64_t cell) {
  CellS v;
#pragma unroll
  for (int q = 0; q < kMaxWS; ++q) v.w[q] = q < a.WS ? __ldg(a.St + cell * a.WS + q) : 0ull;
  return v;
}

// correct count of model m at the current position
template <int M, int PB>
__device__ __forceinline__ uint32_t chan(const EvalGridArgs& a, const CellF& f, const CellS& s, int m) {
  constexpr int PF = 64 / PB;
  if (m == M - 1) return fieldw(f.w, 1, PF, PB);
  if (m == M - 2) return fieldw(f.w, 2, PF, PB);
  return fieldw(s.w, m, PF, PB);
}

template <int M>
__device__ __forceinline__ void store_config(const EvalGridArgs& a, int64_t i, const double* fr,
                                             int K, double frK, double mean, uint32_t correct,
                                             double n) {
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
  if (a.acc) a.acc[i] = ddiv((double)correct, n);
  if (a.n_correct) a.n_correct[i] = correct;
}

template <int M, int PB>
__global__ void __launch_bounds__(256) grid_eval_kernel(const __grid_constant__ EvalGridArgs a) {
  constexpr int PF = 64 / PB;
  const int lane = (int)lane_id();
  const double n = (double)a.n_rec;
  const double one = ddiv(n, n);  // first-stage fraction, as the reference computes it
  const CellF totF = loadF(a, a.cellsF - 1);
  CellS totS;
#pragma unroll
  for (int q = 0; q < kMaxWS; ++q) totS.w[q] = 0ull;
  if (a.DS > 0) totS = loadS(a, a.cellsS - 1);

  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t rg = a.row_lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
       rg < a.row_hi; rg += nw) {
    int s;
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
        store_config<M>(a, i, fr, 1, one, mean, chan<M, PB>(a, totF, totS, mK), n);
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
    int64_t cF = a.cellsF - 1, cS = a.cellsS - 1;
    CellF vF = totF;
    CellS vS = totS;
    uint32_t cp = 0;
    fr[0] = one;
    double mp = dadd(0.0, dmul(one, __ldg(a.cost1 + (mdl & 15u))));
#pragma unroll
    for (int t = 0; t < M - 2; ++t) {
      if (t <= K - 3) {
        const int m = (mdl >> (4 * t)) & 15u;
        const uint32_t A = chan<M, PB>(a, vF, vS, m);
        const int64_t dk = (int64_t)(a.glen[m] - kk[t]);
        cF -= dk * a.strideF[m];
        vF = loadF(a, cF);
        if (m < a.DS) {
          cS -= dk * a.strideS[m];
          vS = loadS(a, cS);
        }
        cp += A - chan<M, PB>(a, vF, vS, m);
        fr[t + 1] = ddiv((double)fieldw(vF.w, 0, PF, PB), n);
        mp = dadd(mp, dmul(fr[t + 1], __ldg(a.cost1 + ((mdl >> (4 * (t + 1))) & 15u))));
      }
    }
    const uint32_t a_last = chan<M, PB>(a, vF, vS, mL);
    const double costK = __ldg(a.cost1 + mK);
    const bool needS = mL < a.DS || mK < a.DS;
    const int64_t c_row = s_begin + row * gL - a.cfg_begin;
    // cell of threshold index kl = base cell + kl * stride (kl = gL is "any")
    const int64_t sFL = a.strideF[mL];
    const int64_t rowF = cF - (int64_t)gL * sFL;
    const int64_t sSL = mL < a.DS ? a.strideS[mL] : 0;
    const int64_t rowS = cS - (int64_t)gL * sSL;
    constexpr int U = 4;  // configs per lane per pass, loads issued together
    for (int base = 0; base < gL; base += 32 * U) {
      CellF wF[U];
      CellS wS[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kl = base + lane + 32 * u;
#pragma unroll
        for (int q = 0; q < kMaxWF; ++q) wF[u].w[q] = 0ull;
#pragma unroll
        for (int q = 0; q < kMaxWS; ++q) wS[u].w[q] = 0ull;
        if (kl < gL) {
          wF[u] = loadF(a, rowF + (int64_t)kl * sFL);
          if (needS) wS[u] = loadS(a, rowS + (int64_t)kl * sSL);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kl = base + lane + 32 * u;
        const int64_t i = c_row + kl;
        if (kl >= gL || i < 0 || i >= a.cfg_count) continue;
        CellS sv;
#pragma unroll
        for (int q = 0; q < kMaxWS; ++q) sv.w[q] = needS ? wS[u].w[q] : vS.w[q];
        const uint32_t correct = cp + a_last - chan<M, PB>(a, wF[u], sv, mL) + chan<M, PB>(a, wF[u], sv, mK);
        const double frK = ddiv((double)fieldw(wF[u].w, 0, PF, PB), n);
        const double mean = dadd(mp, dmul(frK, costK));
        store_config<M>(a, i, fr, K, frK, mean, correct, n);
      }
    }
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

template <int M, int PB, typename Cell>
cudaError_t launch_hist_t(const HistArgs& h, int64_t n_rec, size_t smem, cudaStream_t st) {
  auto k = grid_hist_kernel<M, PB, Cell>;
  static std::atomic<int> smem_set{0};
  cudaError_t e = ensure_smem(k, smem_set, smem);
  if (e != cudaSuccess) return e;
  int64_t blocks = (n_rec + kHistThreads - 1) / kHistThreads;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 4));
  k<<<(unsigned)blocks, kHistThreads, smem, st>>>(h);
  return cudaGetLastError();
}

// compile-time field width; 32-bit cell arithmetic whenever every index fits
template <int M>
cudaError_t launch_hist(const HistArgs& h, int64_t n_rec, size_t smem, int64_t max_index,
                        cudaStream_t st) {
  const bool narrow = max_index < ((int64_t)1 << 32);
  if (h.B == 21)
    return narrow ? launch_hist_t<M, 21, uint32_t>(h, n_rec, smem, st)
                  : launch_hist_t<M, 21, int64_t>(h, n_rec, smem, st);
  return narrow ? launch_hist_t<M, 32, uint32_t>(h, n_rec, smem, st)
                : launch_hist_t<M, 32, int64_t>(h, n_rec, smem, st);
}

template <int M>
cudaError_t launch_grid_eval(const EvalGridArgs& a, cudaStream_t st) {
  const int64_t rows = a.row_hi - a.row_lo;
  int64_t blocks = (rows * 32 + 255) / 256;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 32));
  if (a.B == 21)
    grid_eval_kernel<M, 21><<<(unsigned)blocks, 256, 0, st>>>(a);
  else
    grid_eval_kernel<M, 32><<<(unsigned)blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// Inclusive prefix over every dimension of a u64 table with `vec` words per
// cell.  The first pass reads the histogram `H` (and re-zeroes it), writes
// `T`; later passes run in place on `T`.
cudaError_t prefix_table(unsigned long long* H, unsigned long long* T, int ndim,
                         const int64_t* dims, int64_t cells, int vec, cudaStream_t st) {
  int64_t inner = vec;
  unsigned long long* src = H;
  if (ndim == 0) {  // one cell of `vec` words: copy-and-zero as a 1 x vec "scan"
    for (int q = 0; q < vec; ++q) {
      rowscan_kernel<<<1, 32, 0, st>>>(H + q, T + q, 1, 1);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  for (int d = ndim - 1; d >= 0; --d) {
    const int64_t len = dims[d];
    const int64_t outer = cells * vec / (len * inner);
    if (inner == 1) {
      int64_t blocks = (outer * 32 + 255) / 256;
      blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 16));
      rowscan_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, T, outer, (int)len);
    } else {
      const int64_t tiles = outer * ((inner + kColTile - 1) / kColTile);
      const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count() * 8));
      colscan_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, T, outer, len, inner);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    src = T;
    inner *= len;
  }
  return cudaSuccess;
}

template <int M, int PB>
cudaError_t bucket_build_t(const Plan& p, const double* cert, const uint8_t* corr,
                           const double* grids, uint8_t* ws, int flags, cudaStream_t st) {
  auto* Ft = reinterpret_cast<unsigned long long*>(ws + p.offF);
  auto* St = reinterpret_cast<unsigned long long*>(ws + p.offS);
  auto* bk = reinterpret_cast<uint32_t*>(ws + p.offBk);
  auto* cur = reinterpret_cast<uint32_t*>(ws + p.offCur);
  cudaError_t e;
  if (flags & GS_GRID_WORKSPACE_DIRTY) {
    e = cudaMemsetAsync(cur, 0, (size_t)p.d0 * 4, st);
    if (e != cudaSuccess) return e;
  }
  BucketArgs b{};
  b.cert = cert;
  b.corr = corr;
  b.n_rec = (int32_t)p.cap;
  b.grids = grids;
  int gd = 0;
  for (int j = 0; j < p.M; ++j) {
    b.glen[j] = p.glen[j];
    if (j < p.D) gd += p.glen[j];
  }
  for (int j = 0; j < p.D; ++j) b.strideF[j] = p.strideF[j];
  b.d0 = (int32_t)p.d0;
  b.cap = p.cap;
  b.grid_doubles = gd;
  b.vec_ok = aligned16(cert) && ((reinterpret_cast<uintptr_t>(corr) & 3u) == 0);
  b.buckets = bk;
  b.cursor = cur;
  const size_t smem1 = round_up((size_t)gd * 8, 16) + (size_t)p.d0 * 8;
  static std::atomic<int> smem1_set{0};
  e = ensure_smem(bucket_scatter_kernel<M>, smem1_set, smem1);
  if (e != cudaSuccess) return e;
  int64_t blocks = (p.cap + kScatterThreads * kScatterR - 1) / (kScatterThreads * kScatterR);
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 2));
  bucket_scatter_kernel<M><<<(unsigned)blocks, kScatterThreads, smem1, st>>>(b);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  SlabArgs s{};
  s.d0 = (int32_t)p.d0;
  s.rows = p.D == 3 ? (int32_t)p.dims[1] : 1;
  s.cols = (int32_t)p.dims[p.D - 1];
  s.side_cells = (int32_t)std::max<int64_t>(p.side_slab, 1);
  int64_t div = 1;
  for (int j = p.DS; j < p.D; ++j) div *= p.dims[j];
  s.side_div = (int32_t)div;
  s.cap = p.cap;
  s.buckets = bk;
  s.cursor = cur;
  s.Ft = Ft;
  s.St = St;
  const size_t smem2 = (size_t)(p.slab_cells * p.WF + p.side_slab * p.WS) * 8 + 16;
  static std::atomic<int> smem2_set{0};
  e = ensure_smem(slab_hist_kernel<M, PB>, smem2_set, smem2);
  if (e != cudaSuccess) return e;
  slab_hist_kernel<M, PB><<<(unsigned)p.d0, 1024, smem2, st>>>(s);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // prefix along b_0
  const int64_t innerF = p.slab_cells * p.WF;
  int64_t nb = std::max<int64_t>(1, std::min<int64_t>((innerF + kColTile - 1) / kColTile, (int64_t)sm_count() * 8));
  colscan_kernel<<<(unsigned)nb, 256, 0, st>>>(Ft, Ft, 1, p.d0, innerF);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.DS > 0) {
    const int64_t innerS = p.side_slab * p.WS;
    nb = std::max<int64_t>(1, std::min<int64_t>((innerS + kColTile - 1) / kColTile, (int64_t)sm_count() * 8));
    colscan_kernel<<<(unsigned)nb, 256, 0, st>>>(St, St, 1, p.d0, innerS);
    e = cudaGetLastError();
  }
  return e;
}

cudaError_t bucket_build(const Plan& p, const double* cert, const uint8_t* corr,
                         const double* grids, uint8_t* ws, int flags, cudaStream_t st) {
  if (p.M == 3)
    return p.B == 21 ? bucket_build_t<3, 21>(p, cert, corr, grids, ws, flags, st)
                     : bucket_build_t<3, 32>(p, cert, corr, grids, ws, flags, st);
  return p.B == 21 ? bucket_build_t<4, 21>(p, cert, corr, grids, ws, flags, st)
                   : bucket_build_t<4, 32>(p, cert, corr, grids, ws, flags, st);
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
  info->side_cells = p.cellsS;
  info->n_structures = p.n_struct;
  info->max_len = p.M;
  info->workspace_bytes = p.bytes;
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
  auto* HF = reinterpret_cast<unsigned long long*>(ws + p.offHF);
  auto* Ft = reinterpret_cast<unsigned long long*>(ws + p.offF);
  auto* HS = reinterpret_cast<unsigned long long*>(ws + p.offHS);
  auto* St = reinterpret_cast<unsigned long long*>(ws + p.offS);
  if (p.bucket) {
    GS_CUDA_TRY(bucket_build(p, certainty, correct, grids, ws, flags, st));
    return GS_OK;
  }
  if (flags & GS_GRID_WORKSPACE_DIRTY) {
    GS_CUDA_TRY(cudaMemsetAsync(HF, 0, (size_t)p.cellsF * p.WF * 8, st));
    if (p.cellsS) GS_CUDA_TRY(cudaMemsetAsync(HS, 0, (size_t)p.cellsS * p.WS * 8, st));
  }

  HistArgs h{};
  h.cert = certainty;
  h.corr = correct;
  h.n_rec = (int32_t)n_rec;
  h.grids = grids;
  int off = 0;
  for (int j = 0; j < n_models; ++j) {
    h.glen[j] = p.glen[j];
    if (j < p.D) off += p.glen[j];
  }
  for (int j = 0; j < p.D; ++j) h.strideF[j] = p.strideF[j];
  for (int j = 0; j < p.DS; ++j) h.strideS[j] = p.strideS[j];
  h.cellsS = p.cellsS;
  h.B = p.B;
  h.F = p.F;
  h.WF = p.WF;
  h.WS = p.WS;
  h.grid_doubles = off;
  h.vec_ok = aligned16(certainty) && ((reinterpret_cast<uintptr_t>(correct) & 3u) == 0);
  const size_t side_bytes = (size_t)p.cellsS * p.WS * 8;
  h.priv = p.DS > 0 && side_bytes <= kSidePrivMax;
  h.HF = HF;
  h.HS = HS;
  const size_t smem = round_up((size_t)h.grid_doubles * sizeof(double), 16) +
                      (h.priv ? side_bytes : 0) + 16;
  if (smem > 200 * 1024) return GS_EUNSUPPORTED;
  const int64_t imax = std::max<int64_t>(p.cellsF * p.WF, p.cellsS * p.WS);
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
  GS_CUDA_TRY(prefix_table(HF, Ft, p.D, p.dims, p.cellsF, p.WF, st));
  if (p.DS > 0) GS_CUDA_TRY(prefix_table(HS, St, p.DS, p.dims, p.cellsS, p.WS, st));
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
  if (forward_frac && n_models % 2 == 0 && !aligned16(forward_frac)) return GS_EINVAL;
  EvalGridArgs a{};
  a.M = p.M;
  a.n_struct = p.n_struct;
  a.B = p.B;
  a.F = p.F;
  a.WF = p.WF;
  a.WS = p.WS;
  a.DS = p.DS;
  for (int j = 0; j < p.M; ++j) a.glen[j] = p.glen[j];
  for (int j = 0; j < p.D; ++j) a.strideF[j] = p.strideF[j];
  for (int j = 0; j < p.DS; ++j) a.strideS[j] = p.strideS[j];
  a.n_rec = n_rec;
  a.cellsF = p.cellsF;
  a.cellsS = p.cellsS;
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
  a.row_lo = global_row(p, a.row_begin, config_begin);
  a.row_hi = global_row(p, a.row_begin, config_begin + config_count - 1) + 1;
  const uint8_t* ws = static_cast<const uint8_t*>(workspace);
  a.Ft = reinterpret_cast<const unsigned long long*>(ws + p.offF);
  a.St = reinterpret_cast<const unsigned long long*>(ws + p.offS);
  a.cost1 = cost1;
  a.acc = accuracy;
  a.cost = mean_cost;
  a.frac = forward_frac;
  a.n_correct = n_correct;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
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
