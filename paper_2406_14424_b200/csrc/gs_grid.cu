// gs_grid.cu — grid path: the full cascade x per-stage-threshold product.
//
// Reference semantics: every config is an encoded cascade scored exactly as
// _evaluate_numba scores it (/root/reference/pkg/src/gearserve/kernels.py:
// 39-62); thresholds come from per-model grids (cascades.ThresholdGrid,
// src/cascades.py:132-163), structures are model subsets ordered cheap to
// expensive like sample_cascades builds them (src/cascades.py:181-185).
//
// Algorithm (dominance counting instead of walking every record through
// every config).  With grid G_j of model j, let b_j(r) = #{g in G_j :
// g <= cert[r, j]}.  For threshold index k, cert >= G_j[k]  <=>  b_j > k, so
// a record is forwarded past stage s iff b_{m_s}(r) <= k_s.  Models are in
// cost order and a subset is walked in that order, so the last model M-1 is
// never a forwarding stage: one (M-1)-dimensional table indexed by
// (b_0 .. b_{M-2}) answers every structure.  Each cell holds M+1 integer
// channels — the record count and the correct count of each model — packed
// into u64 words (fields of ceil(log2(n_rec+1)) bits; every prefix sum is
// <= n_rec, so packed words add without carries).  After an inclusive
// prefix sum along every dimension, P[pos] counts records whose bins are
// dominated by pos; a dimension left at its maximum index means "any".
//   reach(stage t+1) = P_cnt[pos with k_0..k_t set]
//   correct         = sum_t (P_c[m_t] before setting k_t - after) + P_c[m_K] at the end
// which is exactly the per-record walk's count.  The f64 epilogue then
// follows the reference's order (frac = count / n, mean += frac * cost1,
// acc = correct / n) with non-contracted multiply/add.
//
// Kernels: hist (one pass over the records, vector loads, warp-aggregated
// u64 atomics), scan along each table dimension (L2-resident), epilogue
// (one thread per config, coalesced output rows).
#include <algorithm>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kMaxM = GS_MAX_MODELS;
constexpr int kMaxW = 5;  // ceil((8 + 1) / 2)

struct Plan {
  int M = 0, D = 0, bits = 0, F = 0, W = 0, n_struct = 0;
  int glen[kMaxM] = {};
  int64_t dims[kMaxM] = {};
  int64_t stride[kMaxM] = {};
  int64_t n_cells = 1;
  int64_t n_configs = 0;
  int64_t struct_begin[256 + 1] = {};
  uint32_t struct_mask[256] = {};
  size_t table_bytes = 0;
};

int make_plan(int64_t n_rec, int32_t M, const int32_t* grid_len, Plan* p) {
  if (M < 1 || !grid_len || n_rec < 1) return GS_EINVAL;
  if (M > kMaxM || n_rec >= (int64_t)UINT32_MAX) return GS_EUNSUPPORTED;
  p->M = M;
  p->D = M - 1;
  for (int j = 0; j < M; ++j) {
    if (grid_len[j] < 1) return GS_EINVAL;
    p->glen[j] = grid_len[j];
  }
  // packed fields
  int bits = 1;
  while (bits < 63 && ((int64_t)1 << bits) <= n_rec) ++bits;
  p->bits = bits;
  p->F = 64 / bits;
  p->W = (M + 1 + p->F - 1) / p->F;
  if (p->W > kMaxW) return GS_EUNSUPPORTED;
  // table dims (b_j in [0, glen_j]) and row-major strides, last dim fastest
  double cells = 1.0;
  for (int j = 0; j < p->D; ++j) {
    p->dims[j] = (int64_t)p->glen[j] + 1;
    cells *= (double)p->dims[j];
  }
  if (cells * p->W * 8.0 > 1.4e11) return GS_EUNSUPPORTED;  // > 140 GB of table
  int64_t s = 1;
  for (int j = p->D - 1; j >= 0; --j) {
    p->stride[j] = s;
    s *= p->dims[j];
  }
  p->n_cells = s;
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
  p->table_bytes = round_up((size_t)p->n_cells * p->W * sizeof(uint64_t), 256);
  return GS_OK;
}

// ------------------------------------------------------------------ hist --
struct HistArgs {
  const double* cert;
  const uint8_t* corr;
  int64_t n_rec;
  const double* grids;  // concatenated
  int32_t goff[kMaxM];
  int32_t glen[kMaxM];
  int64_t stride[kMaxM];
  int64_t n_cells;
  int32_t bits, F, W;
  int32_t vec_ok;  // 16-byte aligned rows (M even, aligned base)
  uint64_t* P;
};

constexpr int kHistThreads = 256;

__device__ __forceinline__ int upper_count(const double* g, int n, double x) {
  // #{g[i] <= x} for strictly increasing g
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (g[mid] <= x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

template <int M>
__global__ void __launch_bounds__(kHistThreads) grid_hist_kernel(HistArgs a) {
  extern __shared__ __align__(16) double s_grid[];
  constexpr int D = M - 1;
  int total = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) total = max(total, a.goff[j] + a.glen[j]);
  for (int i = threadIdx.x; i < total; i += blockDim.x) s_grid[i] = a.grids[i];
  __syncthreads();

  const int64_t stride_r = (int64_t)gridDim.x * blockDim.x;
  const int64_t n_iter = (a.n_rec + stride_r - 1) / stride_r;
  for (int64_t it = 0; it < n_iter; ++it) {
    const int64_t r = it * stride_r + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = r < a.n_rec;
    double x[M];
    uint32_t k[M];
    if (valid) {
      const double* row = a.cert + r * M;
      if constexpr (M % 2 == 0) {
        if (a.vec_ok) {
#pragma unroll
          for (int j = 0; j < M; j += 2) {
            double2 v = __ldg(reinterpret_cast<const double2*>(row + j));
            x[j] = v.x;
            x[j + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int j = 0; j < M; ++j) x[j] = __ldg(row + j);
        }
      } else {
#pragma unroll
        for (int j = 0; j < M; ++j) x[j] = __ldg(row + j);
      }
#pragma unroll
      for (int j = 0; j < M; ++j) k[j] = __ldg(a.corr + r * M + j);
    }
    int64_t cell = 0;
    uint64_t w[kMaxW];
#pragma unroll
    for (int q = 0; q < kMaxW; ++q) w[q] = 0;
    if (valid) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const int b = upper_count(s_grid + a.goff[j], a.glen[j], x[j]);
        cell += (int64_t)b * a.stride[j];
      }
      w[0] = 1ull;  // channel 0: record count
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const int ch = 1 + j;
        const int q = ch / a.F;
        const int sh = (ch % a.F) * a.bits;
        w[q] += (uint64_t)(k[j] != 0) << sh;
      }
    }
    // warp aggregation of duplicate cells (heavy ties, tiny tables)
    const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
    const uint64_t key = valid ? (uint64_t)cell : ~0ull;
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    const bool dup = __any_sync(0xffffffffu, valid && __popc(peers) > 1);
    bool leader = valid;
    if (dup) {
      const int lane = (int)lane_id();
      leader = valid && (__ffs(peers) - 1) == lane;
#pragma unroll
      for (int q = 0; q < kMaxW; ++q) {
        if (q >= a.W) break;
        uint64_t s = 0;
        for (int src = 0; src < 32; ++src) {
          const uint64_t v = __shfl_sync(0xffffffffu, w[q], src);
          if (((peers >> src) & 1u) && ((vmask >> src) & 1u)) s += v;
        }
        w[q] = s;
      }
    }
    if (leader) {
#pragma unroll
      for (int q = 0; q < kMaxW; ++q) {
        if (q >= a.W) break;
        if (w[q]) atomicAdd(reinterpret_cast<unsigned long long*>(a.P + (int64_t)q * a.n_cells + cell),
                            (unsigned long long)w[q]);
      }
    }
  }
}

// ----------------------------------------------------------------- scans --
// Inclusive prefix along a dimension whose stride is 1: one warp per row.
__global__ void scan_rows_kernel(uint64_t* P, int64_t n_cells, int64_t len, int64_t n_rows, int W) {
  const int64_t warp_global = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = (int)lane_id();
  const int64_t total = n_rows * W;
  for (int64_t wr = warp_global; wr < total; wr += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int q = (int)(wr / n_rows);
    const int64_t row = wr - (int64_t)q * n_rows;
    uint64_t* p = P + (int64_t)q * n_cells + row * len;
    uint64_t carry = 0;
    for (int64_t base = 0; base < len; base += 32) {
      const int64_t t = base + lane;
      uint64_t v = t < len ? p[t] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      v += carry;
      if (t < len) p[t] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
}

// Inclusive prefix along a dimension with stride `inner` > 1: one thread per
// (outer, inner) column, coalesced across threads, 8 loads in flight.
__global__ void scan_cols_kernel(uint64_t* P, int64_t n_cells, int64_t outer, int64_t len,
                                 int64_t inner, int W) {
  const int64_t n_cols = outer * inner;
  const int64_t total = n_cols * W;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(t / n_cols);
    const int64_t col = t - (int64_t)q * n_cols;
    const int64_t o = col / inner;
    const int64_t i = col - o * inner;
    uint64_t* p = P + (int64_t)q * n_cells + o * len * inner + i;
    uint64_t acc = 0;
    int64_t k = 0;
    for (; k + 8 <= len; k += 8) {
      uint64_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = p[(k + u) * inner];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc += v[u];
        p[(k + u) * inner] = acc;
      }
    }
    for (; k < len; ++k) {
      acc += p[k * inner];
      p[k * inner] = acc;
    }
  }
}

// -------------------------------------------------------------- epilogue --
struct EvalGridArgs {
  int32_t M, W, bits, F, n_struct;
  int32_t glen[kMaxM];
  int64_t stride[kMaxM];
  int64_t n_rec, n_cells;
  int64_t cfg_begin, cfg_count;
  int64_t struct_begin[256 + 1];
  uint32_t struct_mask[256];
  const uint64_t* P;
  const double* cost1;
  double* acc;
  double* cost;
  double* frac;
  uint32_t* n_correct;
};

__device__ __forceinline__ uint32_t field(const uint64_t* w, int ch, int F, int bits) {
  const uint64_t mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
  return (uint32_t)((w[ch / F] >> ((ch % F) * bits)) & mask);
}

__device__ __forceinline__ int find_struct(const EvalGridArgs& a, int64_t c) {
  int lo = 0, hi = a.n_struct - 1;  // last s with struct_begin[s] <= c
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.struct_begin[mid] <= c)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

template <int M>
__global__ void __launch_bounds__(256) grid_eval_kernel(const __grid_constant__ EvalGridArgs a) {
  const int W = a.W;
  const double n = (double)a.n_rec;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.cfg_count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = a.cfg_begin + i;
    const int s = find_struct(a, c);
    const uint32_t mask = a.struct_mask[s];
    int K = 0;
    int mdl[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      if ((mask >> j) & 1u) {
        mdl[K] = j;
        ++K;
      }
    }
    // decode threshold indices, last forwarding stage fastest
    int64_t local = c - a.struct_begin[s];
    int kidx[M];
#pragma unroll
    for (int t = M - 2; t >= 0; --t) {
      if (t < K - 1) {
        const int g = a.glen[mdl[t]];
        if (local < 0x7fffffffLL) {
          const int l32 = (int)local;
          kidx[t] = l32 % g;
          local = l32 / g;
        } else {
          kidx[t] = (int)(local % g);
          local /= g;
        }
      }
    }
    // dominance-count walk
    int64_t cell = a.n_cells - 1;  // every dimension at "any"
    uint64_t wv[kMaxW];
#pragma unroll
    for (int q = 0; q < kMaxW; ++q)
      if (q < W) wv[q] = __ldg(a.P + (int64_t)q * a.n_cells + cell);
    uint32_t reach[M];
    reach[0] = (uint32_t)a.n_rec;
    int64_t correct = 0;
#pragma unroll
    for (int t = 0; t < M - 1; ++t) {
      if (t < K - 1) {
        const int m = mdl[t];
        const int64_t before = field(wv, 1 + m, a.F, a.bits);
        cell -= (int64_t)(a.glen[m] - kidx[t]) * a.stride[m];
#pragma unroll
        for (int q = 0; q < kMaxW; ++q)
          if (q < W) wv[q] = __ldg(a.P + (int64_t)q * a.n_cells + cell);
        reach[t + 1] = field(wv, 0, a.F, a.bits);
        correct += before - (int64_t)field(wv, 1 + m, a.F, a.bits);
      }
    }
    correct += field(wv, 1 + mdl[K - 1], a.F, a.bits);
    // f64 epilogue in the reference's order (src/kernels.py:57-61)
    double mean = 0.0;
    double fr[M];
#pragma unroll
    for (int t = 0; t < M; ++t) {
      fr[t] = 0.0;
      if (t < K) {
        fr[t] = ddiv((double)reach[t], n);
        mean = dadd(mean, dmul(fr[t], __ldg(a.cost1 + mdl[t])));
      }
    }
    if (a.frac) {
      double* row = a.frac + i * M;
      if constexpr (M % 2 == 0) {
#pragma unroll
        for (int t = 0; t < M; t += 2)
          reinterpret_cast<double2*>(row)[t / 2] = make_double2(fr[t], fr[t + 1]);
      } else {
#pragma unroll
        for (int t = 0; t < M; ++t) row[t] = fr[t];
      }
    }
    if (a.cost) a.cost[i] = mean;
    if (a.acc) a.acc[i] = ddiv((double)correct, n);
    if (a.n_correct) a.n_correct[i] = (uint32_t)correct;
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

template <int M>
cudaError_t launch_hist(const HistArgs& h, int64_t n_rec, size_t smem, cudaStream_t st) {
  auto k = grid_hist_kernel<M>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int64_t blocks = (n_rec + kHistThreads - 1) / kHistThreads;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 8));
  k<<<(unsigned)blocks, kHistThreads, smem, st>>>(h);
  return cudaGetLastError();
}

template <int M>
cudaError_t launch_grid_eval(const EvalGridArgs& a, cudaStream_t st) {
  int64_t blocks = (a.cfg_count + 255) / 256;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 16));
  grid_eval_kernel<M><<<(unsigned)blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
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
  info->n_cells = p.n_cells;
  info->n_structures = p.n_struct;
  info->words_per_cell = p.W;
  info->field_bits = p.bits;
  info->max_len = p.M;
  info->workspace_bytes = p.table_bytes;
  return GS_OK;
}

extern "C" int gs_grid_build(const double* certainty, const uint8_t* correct, int64_t n_rec,
                             int32_t n_models, const double* grids, const int32_t* grid_len,
                             void* workspace, size_t workspace_bytes, void* stream) {
  Plan p;
  int rc = make_plan(n_rec, n_models, grid_len, &p);
  if (rc != GS_OK) return rc;
  GS_REQUIRE(certainty && correct && grids);
  if (!workspace || workspace_bytes < p.table_bytes) return GS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t* P = static_cast<uint64_t*>(workspace);
  GS_CUDA_TRY(cudaMemsetAsync(P, 0, (size_t)p.n_cells * p.W * sizeof(uint64_t), st));

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
  for (int j = 0; j < p.D; ++j) h.stride[j] = p.stride[j];
  h.n_cells = p.n_cells;
  h.bits = p.bits;
  h.F = p.F;
  h.W = p.W;
  h.vec_ok = aligned16(certainty) && (n_models % 2 == 0);
  h.P = P;
  // shared memory holds the grids of the forwarding models 0..M-2
  const size_t smem = (size_t)std::max(1, p.D > 0 ? h.goff[p.D - 1] + h.glen[p.D - 1] : 1) * sizeof(double);
  if (smem > 200 * 1024) return GS_EUNSUPPORTED;
  cudaError_t e = cudaSuccess;
  switch (n_models) {
    case 1: e = launch_hist<1>(h, n_rec, smem, st); break;
    case 2: e = launch_hist<2>(h, n_rec, smem, st); break;
    case 3: e = launch_hist<3>(h, n_rec, smem, st); break;
    case 4: e = launch_hist<4>(h, n_rec, smem, st); break;
    case 5: e = launch_hist<5>(h, n_rec, smem, st); break;
    case 6: e = launch_hist<6>(h, n_rec, smem, st); break;
    case 7: e = launch_hist<7>(h, n_rec, smem, st); break;
    case 8: e = launch_hist<8>(h, n_rec, smem, st); break;
    default: return GS_EUNSUPPORTED;
  }
  GS_CUDA_TRY(e);

  // inclusive prefix along every dimension
  for (int d = p.D - 1; d >= 0; --d) {
    const int64_t len = p.dims[d];
    const int64_t inner = p.stride[d];
    const int64_t outer = p.n_cells / (len * inner);
    if (inner == 1) {
      const int64_t warps = outer * p.W;
      int64_t blocks = (warps * 32 + 255) / 256;
      blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 32));
      scan_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(P, p.n_cells, len, outer, p.W);
    } else {
      const int64_t cols = outer * inner * p.W;
      int64_t blocks = (cols + 255) / 256;
      blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 32));
      scan_cols_kernel<<<(unsigned)blocks, 256, 0, st>>>(P, p.n_cells, outer, len, inner, p.W);
    }
    GS_LAUNCH_CHECK();
  }
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
  if (!workspace || workspace_bytes < p.table_bytes) return GS_EWORKSPACE;
  if (forward_frac && n_models % 2 == 0 && !aligned16(forward_frac)) return GS_EINVAL;
  EvalGridArgs a{};
  a.M = p.M;
  a.W = p.W;
  a.bits = p.bits;
  a.F = p.F;
  a.n_struct = p.n_struct;
  for (int j = 0; j < p.M; ++j) a.glen[j] = p.glen[j];
  for (int j = 0; j < p.D; ++j) a.stride[j] = p.stride[j];
  a.n_rec = n_rec;
  a.n_cells = p.n_cells;
  a.cfg_begin = config_begin;
  a.cfg_count = config_count;
  for (int s = 0; s <= p.n_struct; ++s) a.struct_begin[s] = p.struct_begin[s];
  for (int s = 0; s < p.n_struct; ++s) a.struct_mask[s] = p.struct_mask[s];
  a.P = static_cast<const uint64_t*>(workspace);
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
