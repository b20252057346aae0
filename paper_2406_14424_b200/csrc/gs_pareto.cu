// gs_pareto.cu — Pareto front of (accuracy, mean_cost) points.
//
// Reference: cascades.pareto_filter (/root/reference/pkg/src/gearserve/
// cascades.py:116-129): an item is dropped iff another item has accuracy >=
// and cost <=, with at least one strict; exact ties survive; order is kept.
//
// gs_pareto_counts (sweep outputs, O(n + n_rec), no sort).  Accuracy is the
// integer correct count a in [0, n_rec] (acc = a / n_rec is monotone in a).
//   mincost[a]  = min cost over items with count a            (u64 atomicMin)
//   above[a]    = min cost over items with count > a          (suffix min,
//                 stored beside mincost[a] as one 16-byte pair)
//   keep(i)     = cost_i == mincost[a_i]  &&  cost_i < above[a_i]
// (an item with the same count and lower cost, or a higher count and cost
// <=, is exactly what dominates it).  Costs are compared through an
// order-preserving u64 key, -0.0 folded into +0.0 so equal doubles get equal
// keys.  The kept indices are then compacted stably with a decoupled
// look-back scan.
//
// gs_pareto_generic (float accuracies, small n): every item tests every
// other item, tiles of candidates staged in shared memory.
#include <algorithm>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kChunk = 2048;  // suffix-min chunk (8 entries per thread)

__device__ __forceinline__ uint64_t cost_key(double x) {
  x = x + 0.0;  // -0.0 -> +0.0
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Many configs share a correct count (thresholds that change no decision),
// so the per-bucket atomicMin is aggregated first: lanes with the same count
// take their group minimum, and the group leader only issues the atomic when
// it would lower the bucket (a stale read can only be too high, never too
// low, so skipping on it is safe).
__global__ void bucket_min_kernel(const uint32_t* n_correct, const double* cost, int64_t n,
                                  int64_t n_rec, unsigned long long* mincost) {
  const int lane = (int)lane_id();
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += step) {
    const int64_t i = base + lane;
    const bool valid = i < n;
    uint32_t a = valid ? n_correct[i] : 0xffffffffu;
    if (valid && (int64_t)a > n_rec) a = (uint32_t)n_rec;
    unsigned long long key = valid ? cost_key(cost[i]) : ~0ull;
    const uint32_t peers = __match_any_sync(0xffffffffu, a);
    unsigned long long m = key;
    for (int src = 0; src < 32; ++src) {
      const unsigned long long v = __shfl_sync(0xffffffffu, key, src);
      if ((peers >> src) & 1u) m = min(m, v);
    }
    if (valid && (__ffs(peers) - 1) == lane) {
      volatile unsigned long long* slot = mincost + a;
      if (m < *slot) atomicMin(mincost + a, m);
    }
  }
}

__global__ void chunk_min_kernel(const unsigned long long* v, int64_t len, unsigned long long* out) {
  __shared__ unsigned long long s[32];
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  unsigned long long m = ~0ull;
  for (int j = threadIdx.x; j < kChunk; j += blockDim.x) {
    const int64_t k = base + j;
    if (k < len) m = min(m, v[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0) s[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? s[threadIdx.x] : ~0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) out[blockIdx.x] = m;
  }
}

// pair[k] = {v[k], min(v[k+1 ..])} ; 256 threads x 8 entries per chunk.
// (The select pass reads both for a count with one 16-byte load.)
__global__ void __launch_bounds__(256) suffix_min_kernel(const unsigned long long* v, int64_t len,
                                                         const unsigned long long* chunk_min,
                                                         int64_t n_chunks, ulonglong2* pair) {
  __shared__ unsigned long long s_warp[8];
  __shared__ unsigned long long s_carry;
  const int64_t b = blockIdx.x;
  // carry: min over all later chunks
  unsigned long long carry = ~0ull;
  for (int64_t j = b + 1 + threadIdx.x; j < n_chunks; j += blockDim.x) carry = min(carry, chunk_min[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) carry = min(carry, __shfl_xor_sync(0xffffffffu, carry, o));
  if (lane_id() == 0) s_warp[threadIdx.x >> 5] = carry;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long c = ~0ull;
    for (int w = 0; w < 8; ++w) c = min(c, s_warp[w]);
    s_carry = c;
  }
  __syncthreads();
  carry = s_carry;
  __syncthreads();

  const int64_t base = b * kChunk + (int64_t)threadIdx.x * 8;
  unsigned long long x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = (base + u < len) ? v[base + u] : ~0ull;
  // thread total
  unsigned long long t = ~0ull;
#pragma unroll
  for (int u = 0; u < 8; ++u) t = min(t, x[u]);
  // exclusive suffix over threads (threads with higher index come later)
  const int lane = (int)lane_id();
  unsigned long long incl = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_down_sync(0xffffffffu, incl, o);
    if (lane + o < 32) incl = min(incl, y);
  }
  if (lane == 0) s_warp[threadIdx.x >> 5] = incl;  // warp total
  __syncthreads();
  unsigned long long after_warp = carry;
  for (int w = (threadIdx.x >> 5) + 1; w < 8; ++w) after_warp = min(after_warp, s_warp[w]);
  unsigned long long after_thread = __shfl_down_sync(0xffffffffu, incl, 1);
  if (lane == 31) after_thread = ~0ull;
  unsigned long long run = min(after_warp, after_thread);
#pragma unroll
  for (int u = 7; u >= 0; --u) {
    if (base + u < len) pair[base + u] = make_ulonglong2(x[u], run);
    run = min(run, x[u]);
  }
}

constexpr int kSelItems = 16;  // consecutive items per thread
constexpr int kSelTile = 256 * kSelItems;

// keep flags for kSelTile consecutive items per CTA (kSelItems per thread,
// in order), block scan of the per-thread counts, decoupled look-back over
// the (few) tiles, then each thread writes its kept indices in order.
__global__ void __launch_bounds__(256) pareto_select_kernel(
    const uint32_t* n_correct, const double* cost, int64_t n, int64_t n_rec,
    const ulonglong2* pair, int64_t base_index,
    uint8_t* keep, int64_t* kept_idx, int64_t* n_kept, uint64_t* states,
    unsigned long long* counter, int64_t n_tiles) {
  __shared__ uint32_t s_warp[8];
  __shared__ uint64_t s_excl;
  __shared__ int64_t s_tile;
  const int64_t tile = next_tile_id(counter, &s_tile);
  const int64_t i0 = tile * kSelTile + (int64_t)threadIdx.x * kSelItems;
  uint32_t kmask = 0;
#pragma unroll
  for (int u = 0; u < kSelItems; ++u) {
    const int64_t i = i0 + u;
    if (i < n) {
      uint32_t a = __ldg(n_correct + i);
      if ((int64_t)a > n_rec) a = (uint32_t)n_rec;
      const unsigned long long key = cost_key(__ldg(cost + i));
      const ulonglong2 mb = pair[a];  // {min cost at a, min cost above a}
      const bool k = (mb.x == key) && (key < mb.y);
      kmask |= (uint32_t)k << u;
      if (keep) keep[i] = k ? 1 : 0;
    }
  }
  const uint32_t cnt = __popc(kmask);
  const int lane = (int)lane_id(), warp = threadIdx.x >> 5;
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < 8 ? s_warp[lane] : 0u, wi = w;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, wi, 7);
    if (lane < 8) s_warp[lane] = wi - w;  // exclusive warp offsets
    const uint64_t excl = lookback_exclusive(states, tile, (uint64_t)total);
    if (lane == 0) {
      s_excl = excl;
      if (tile == n_tiles - 1) *n_kept = (int64_t)(excl + total);
    }
  }
  __syncthreads();
  int64_t out = (int64_t)s_excl + s_warp[warp] + (incl - cnt);
  while (kmask) {
    const int u = __ffs(kmask) - 1;
    kmask &= kmask - 1;
    kept_idx[out++] = base_index + i0 + u;
  }
}

__global__ void __launch_bounds__(256) pareto_generic_kernel(const double* acc, const double* cost,
                                                             int64_t n, uint8_t* keep) {
  __shared__ double s_acc[1024];
  __shared__ double s_cost[1024];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double ai = i < n ? acc[i] : 0.0;
  const double ci = i < n ? cost[i] : 0.0;
  bool dominated = false;
  for (int64_t base = 0; base < n; base += 1024) {
    const int cnt = (int)min((int64_t)1024, n - base);
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
      s_acc[j] = acc[base + j];
      s_cost[j] = cost[base + j];
    }
    __syncthreads();
    if (!dominated) {
      for (int j = 0; j < cnt; ++j) {
        const double ao = s_acc[j], co = s_cost[j];
        if (ao >= ai && co <= ci && (ao > ai || co < ci)) {
          dominated = true;
          break;
        }
      }
    }
  }
  if (i < n) keep[i] = dominated ? 0 : 1;
}

struct CountsWs {
  size_t mincost, above, chunk_min, states, counter, total;
};

CountsWs counts_ws(int64_t n, int64_t n_rec) {
  CountsWs w;
  const int64_t len = n_rec + 1;
  const int64_t n_chunks = (len + kChunk - 1) / kChunk;
  const int64_t n_tiles = (n + kSelTile - 1) / kSelTile;
  size_t off = 0;
  w.mincost = off;
  off += round_up((size_t)len * 8, 256);
  w.above = off;
  off += round_up((size_t)len * 16, 256);
  w.chunk_min = off;
  off += round_up((size_t)n_chunks * 8, 256);
  w.states = off;
  off += round_up((size_t)std::max<int64_t>(n_tiles, 1) * 8, 256);
  w.counter = off;
  off += 256;
  w.total = off;
  return w;
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" int gs_pareto_counts_workspace(int64_t n, int64_t n_rec, size_t* bytes) {
  GS_REQUIRE(bytes && n >= 0 && n_rec >= 0);
  *bytes = counts_ws(n, n_rec).total;
  return GS_OK;
}

extern "C" int gs_pareto_counts(const uint32_t* n_correct, const double* cost, int64_t n,
                                int64_t n_rec, int64_t base_index, uint8_t* keep,
                                int64_t* kept_idx, int64_t* n_kept, void* workspace,
                                size_t workspace_bytes, void* stream) {
  GS_REQUIRE(n >= 0 && n_rec >= 0 && n_kept && kept_idx);
  if (n >= (int64_t)1 << 31) return GS_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 0) {
    GS_CUDA_TRY(cudaMemsetAsync(n_kept, 0, sizeof(int64_t), st));
    return GS_OK;
  }
  GS_REQUIRE(n_correct && cost);
  const CountsWs w = counts_ws(n, n_rec);
  if (!workspace || workspace_bytes < w.total) return GS_EWORKSPACE;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  auto* mincost = reinterpret_cast<unsigned long long*>(ws + w.mincost);
  auto* pair = reinterpret_cast<ulonglong2*>(ws + w.above);
  auto* chunk_min = reinterpret_cast<unsigned long long*>(ws + w.chunk_min);
  auto* states = reinterpret_cast<uint64_t*>(ws + w.states);
  auto* counter = reinterpret_cast<unsigned long long*>(ws + w.counter);
  const int64_t len = n_rec + 1;
  const int64_t n_chunks = (len + kChunk - 1) / kChunk;
  const int64_t n_tiles = (n + kSelTile - 1) / kSelTile;
  GS_CUDA_TRY(cudaMemsetAsync(mincost, 0xff, (size_t)len * 8, st));
  GS_CUDA_TRY(cudaMemsetAsync(states, 0, (size_t)n_tiles * 8, st));
  GS_CUDA_TRY(cudaMemsetAsync(counter, 0, 8, st));
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16));
  bucket_min_kernel<<<(unsigned)blocks, 256, 0, st>>>(n_correct, cost, n, n_rec, mincost);
  GS_LAUNCH_CHECK();
  chunk_min_kernel<<<(unsigned)n_chunks, 256, 0, st>>>(mincost, len, chunk_min);
  GS_LAUNCH_CHECK();
  suffix_min_kernel<<<(unsigned)n_chunks, 256, 0, st>>>(mincost, len, chunk_min, n_chunks, pair);
  GS_LAUNCH_CHECK();
  pareto_select_kernel<<<(unsigned)n_tiles, 256, 0, st>>>(n_correct, cost, n, n_rec, pair, base_index,
                                                          keep, kept_idx, n_kept, states, counter,
                                                          n_tiles);
  GS_LAUNCH_CHECK();
  return GS_OK;
}

extern "C" int gs_pareto_generic(const double* accuracy, const double* cost, int64_t n,
                                 uint8_t* keep, void* stream) {
  GS_REQUIRE(n >= 0);
  if (n == 0) return GS_OK;
  GS_REQUIRE(accuracy && cost && keep);
  const int64_t blocks = (n + 255) / 256;
  if (blocks > 0x7fffffff) return GS_EUNSUPPORTED;
  pareto_generic_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      accuracy, cost, n, keep);
  GS_LAUNCH_CHECK();
  return GS_OK;
}
