// gs_quantile.cu — threshold-grid quantiles on the device.
//
// Reference: cascades.build_threshold_grid (/root/reference/pkg/src/
// gearserve/cascades.py:150-163) takes np.quantile(cert[:, j], k/levels)
// with numpy's default "linear" method.  numpy (lib/_function_base_impl.py,
// _quantile / _get_indexes / _lerp, pinned numpy 2.3.5) computes, for a
// sorted column a of n values:
//   v = (n - 1) * q                      virtual index (f64)
//   prev = floor(v), next = prev + 1     both -> n-1 when v >= n - 1
//   g = v - prev                         (f64; the -1 index case keeps g)
//   diff = a[next] - a[prev]
//   r = a[prev] + diff * g,  or  a[next] - diff * (1 - g) when g >= 0.5
// (separate multiplies and adds, no FMA) and returns a[n-1] (NaN) for every
// q when the column holds a NaN (NaNs sort last).
//
// Only the 2 n_q + 1 order statistics a[prev], a[next], a[n-1] are needed,
// not the sorted column, so they are found by a most-significant-digit radix
// select instead of a sort, on u64 keys whose unsigned order is numpy's sort
// order (-0.0 taken as +0.0, NaN above +inf):
//   gather + pass 0   the column (any stride) -> keys; a shared-memory
//                     histogram of their top 12 bits;
//   resolve           a CTA per target: the bin holding its rank becomes the
//                     next 12 bits of its prefix;
//   pass 1, resolve   the keys under a target's prefix counted by their next
//                     12 bits (targets sharing a prefix share a histogram
//                     row; a shared-memory hash maps prefixes to rows);
//   plan, collect     the keys under each distinct 24-bit prefix (a few
//                     hundred on quantile grids) compacted into one list;
//   final             a CTA per target: the remaining 40 bits by four 10-bit
//                     shared-memory passes over its list;
//   lerp              numpy's interpolation on the 2 n_q + 1 values.
// Two streaming reads of the 8n-byte keys (L2-resident) plus the collect,
// instead of an eight-pass 64-bit radix sort of the whole column.
#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kQBits = 12;
constexpr int kQBins = 1 << kQBits;
constexpr int kQFinalBits = 10;        // 24 + 4 x 10 = 64
constexpr int kQChunk = 255;  // quantiles per select round (more: several rounds over the same keys)
constexpr int kQMaxTargets = 2 * kQChunk + 1;
constexpr int kQHash = 1024;           // >= 2 x targets, power of two
constexpr uint64_t kQEmpty = ~0ull;    // never a prefix (its low 40 bits are zero)
constexpr int kQPassThreads = 512;
static_assert(kQMaxTargets <= kQPassThreads, "build_hash scans one target a thread");
constexpr int kQResolveThreads = 256;

// f64 -> u64 with the unsigned order of numpy's sort: -0.0 == +0.0, NaNs
// last.  The bits cross through mov.b64 so that the sign-bit arithmetic stays
// integer (nvcc otherwise folds it into an FP |x| / -|x|, which turns a NaN
// into the canonical NaN and breaks its order).
__device__ __forceinline__ uint64_t f64_bits(double x) {
  uint64_t b;
  asm("mov.b64 %0, %1;" : "=l"(b) : "d"(x));
  return b;
}
__device__ __forceinline__ double bits_f64(uint64_t b) {
  double x;
  asm("mov.b64 %0, %1;" : "=d"(x) : "l"(b));
  return x;
}
__device__ __forceinline__ uint64_t order_key(double x) {
  uint64_t b = f64_bits(x + 0.0);  // -0.0 -> +0.0
  const bool nan = (b & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
  if (nan) b &= ~(1ull << 63);  // a NaN sorts above +inf whatever its sign
  return (b >> 63) ? ~b : b | (1ull << 63);
}
__device__ __forceinline__ double key_value(uint64_t k) {
  return bits_f64((k >> 63) ? k & ~(1ull << 63) : ~k);
}

__device__ __forceinline__ uint64_t hi_mask(int resolved) {
  return resolved == 0 ? 0ull : ~0ull << (64 - resolved);
}
__device__ __forceinline__ uint32_t hash_prefix(uint64_t p) {
  return (uint32_t)((p * 0x9E3779B97F4A7C15ull) >> 54) & (kQHash - 1);
}

// numpy's indexes for quantile i: prev / next ranks (targets 2i, 2i + 1);
// target 2 n_q is rank n - 1 (the NaN check)
__device__ __forceinline__ void quantile_ranks(int64_t n, double q, int64_t& prev, int64_t& next,
                                               double& v, double& fl) {
  v = __dmul_rn((double)(n - 1), q);
  fl = floor(v);
  if (v >= (double)(n - 1)) {
    prev = next = n - 1;
  } else if (v < 0.0) {
    prev = next = 0;
  } else {
    prev = (int64_t)fl;
    next = prev + 1;
  }
}

struct Target {
  uint64_t pre;  // resolved high bits of the target's key (lower bits zero)
  uint64_t rem;  // its rank among the keys that share pre
  uint64_t cnt;  // how many keys share pre
};
struct RowInfo {
  uint32_t row;   // smallest target index with this target's prefix
  uint32_t fill;  // keys collected so far (row heads only)
  uint64_t off;   // the row's list: [off, off + size) of the collect buffer
  uint64_t size;
};

__global__ void init_targets_kernel(const double* qs, int32_t n_q, int64_t n, Target* t) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_q) {
    int64_t prev, next;
    double v, fl;
    quantile_ranks(n, qs[i], prev, next, v, fl);
    t[2 * i] = {0ull, (uint64_t)prev, (uint64_t)n};
    t[2 * i + 1] = {0ull, (uint64_t)next, (uint64_t)n};
  } else if (i == n_q) {
    t[2 * n_q] = {0ull, (uint64_t)(n - 1), (uint64_t)n};
  }
}

// The targets' prefixes in a shared-memory hash: prefix -> smallest target
// index holding it (its histogram row / list).
struct PrefixHash {
  uint64_t key[kQHash];
  int row[kQHash];
  int cid[kQHash];  // the row's index among the distinct rows, by row order
  int slot_of[kQMaxTargets];  // compact id -> hash slot
  int n_rows;
};
__device__ __forceinline__ void build_hash(PrefixHash& h, const Target* t, int n_t) {
  for (int i = threadIdx.x; i < kQHash; i += blockDim.x) {
    h.key[i] = kQEmpty;
    h.row[i] = 0x7fffffff;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n_t; j += blockDim.x) {
    const uint64_t p = t[j].pre;
    for (uint32_t x = hash_prefix(p);; x = (x + 1) & (kQHash - 1)) {
      const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(h.key + x), kQEmpty, p);
      if (old == kQEmpty || old == p) {
        atomicMin(h.row + x, j);
        break;
      }
    }
  }
  __syncthreads();
  // compact ids: a row's rank among the distinct rows, by a block scan of
  // "target j heads its row" (one target a thread: n_t <= blockDim)
  __shared__ int s_wsum[32];
  const int j = threadIdx.x, lane = j & 31, warp = j >> 5;
  int x = -1, head = 0;
  if (j < n_t) {
    const uint64_t p = t[j].pre;
    for (x = (int)hash_prefix(p); h.key[x] != p; x = (x + 1) & (kQHash - 1)) {
    }
    head = h.row[x] == j ? 1 : 0;
  }
  int incl = head;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  int before = incl - head;
  for (int w = 0; w < warp; ++w) before += s_wsum[w];
  if (head) {
    h.cid[x] = before;
    h.slot_of[before] = x;
  }
  if (j == (int)blockDim.x - 1) h.n_rows = before + head;
  __syncthreads();
}
// the prefix's hash slot, or -1
__device__ __forceinline__ int find_slot(const PrefixHash& h, uint64_t p) {
  for (uint32_t x = hash_prefix(p);; x = (x + 1) & (kQHash - 1)) {
    const uint64_t e = h.key[x];
    if (e == p) return (int)x;
    if (e == kQEmpty) return -1;
  }
}

// Pass 0 with the gather: every key counted by its top 12 bits in shared
// memory, the CTA's bins added to row 0 (every target starts at prefix 0).
__global__ void __launch_bounds__(kQPassThreads) gather_pass0_kernel(const double* __restrict__ col, int64_t n,
                                                                     int64_t stride, uint64_t* __restrict__ keys,
                                                                     uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_hist[kQBins];
  for (int i = threadIdx.x; i < kQBins; i += blockDim.x) s_hist[i] = 0u;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = order_key(col[i * stride]);
    keys[i] = k;
    atomicAdd(s_hist + (uint32_t)(k >> (64 - kQBits)), 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kQBins; i += blockDim.x)
    if (s_hist[i]) atomicAdd(hist + i, s_hist[i]);
}

// Pass 1: the keys under a target's 12-bit prefix, counted by their next 12
// bits into that prefix's row: in shared memory when the distinct prefixes
// are few (the usual case: a column's values share a few exponents), which
// also keeps heavily tied values off a handful of global counters.
constexpr int kQPrivRows = 4;  // 64 KB of shared histograms (dynamic)
__global__ void __launch_bounds__(kQPassThreads) pass1_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                              const Target* __restrict__ t, int n_t,
                                                              uint32_t* __restrict__ hist) {
  __shared__ PrefixHash h;
  extern __shared__ uint32_t s_hist[];  // [kQPrivRows][kQBins]
  build_hash(h, t, n_t);
  const uint64_t m = hi_mask(kQBits);
  const int shift = 64 - 2 * kQBits;
  if (h.n_rows <= kQPrivRows) {
    for (int i = threadIdx.x; i < kQPrivRows * kQBins; i += blockDim.x) s_hist[i] = 0u;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      const uint64_t k = keys[i];
      const int x = find_slot(h, k & m);
      if (x >= 0) atomicAdd(s_hist + h.cid[x] * kQBins + ((uint32_t)(k >> shift) & (kQBins - 1)), 1u);
    }
    __syncthreads();
    for (int c = 0; c < h.n_rows; ++c) {  // each distinct row merged once
      const uint32_t* src = s_hist + c * kQBins;
      uint32_t* dst = hist + (size_t)h.row[h.slot_of[c]] * kQBins;
      for (int i = threadIdx.x; i < kQBins; i += blockDim.x)
        if (src[i]) atomicAdd(dst + i, src[i]);
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const int x = find_slot(h, k & m);
    if (x >= 0) atomicAdd(hist + (size_t)h.row[x] * kQBins + ((uint32_t)(k >> shift) & (kQBins - 1)), 1u);
  }
}

// Exclusive scan of a CTA's bins (PER consecutive bins a thread): the bin
// whose range holds rank `rem` is reported through `hit` (bin, rank in bin,
// count).  THREADS threads, all of which call it.
template <int THREADS, int PER>
__device__ __forceinline__ void find_bin(const uint32_t (&c)[PER], uint64_t rem, uint32_t* s_wsum,
                                         uint64_t* hit) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t sum = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) sum += c[q];
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  uint64_t acc = x - sum;
  for (int w = 0; w < warp; ++w) acc += s_wsum[w];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (c[q] && rem >= acc && rem < acc + c[q]) {
      hit[0] = (uint64_t)(tid * PER + q);
      hit[1] = rem - acc;
      hit[2] = c[q];
    }
    acc += c[q];
  }
  __syncthreads();
}

// A CTA per target: its prefix's row (the smallest target index sharing the
// prefix), the bin holding its rank becomes the next 12 bits of its prefix.
// Target state is double-buffered (the row lookup reads every target's
// current prefix); the CTA zeroes its own row of the next pass's histogram.
__global__ void __launch_bounds__(kQResolveThreads) resolve_kernel(const Target* __restrict__ cur,
                                                                   Target* __restrict__ nxt, int n_t,
                                                                   int resolved,
                                                                   const uint32_t* __restrict__ hist,
                                                                   uint32_t* __restrict__ next_hist) {
  constexpr int per = kQBins / kQResolveThreads;  // 16 bins a thread
  __shared__ int s_row;
  __shared__ uint32_t s_wsum[kQResolveThreads / 32];
  __shared__ uint64_t s_hit[3];
  const int t = blockIdx.x, tid = threadIdx.x;
  const Target me = cur[t];
  if (tid == 0) s_row = t;
  __syncthreads();
  for (int j = tid; j < t; j += blockDim.x)
    if (cur[j].pre == me.pre) atomicMin(&s_row, j);
  __syncthreads();
  const uint32_t* row = hist + (size_t)s_row * kQBins;
  uint32_t c[per];
#pragma unroll
  for (int q = 0; q < per; ++q) c[q] = row[tid * per + q];
  find_bin<kQResolveThreads, per>(c, me.rem, s_wsum, s_hit);
  if (tid == 0) nxt[t] = {me.pre | (s_hit[0] << (64 - resolved - kQBits)), s_hit[1], s_hit[2]};
  if (next_hist) {
    uint32_t* mine = next_hist + (size_t)t * kQBins;
#pragma unroll
    for (int q = 0; q < per; ++q) mine[tid * per + q] = 0u;
  }
}

// One CTA: the distinct 24-bit prefixes (a row = the smallest target index
// holding one), each row's list size (its bucket's count) and offset.
__global__ void __launch_bounds__(1024) plan_rows_kernel(const Target* __restrict__ t, int n_t,
                                                         RowInfo* __restrict__ ri) {
  __shared__ uint32_t s_row[kQMaxTargets];
  __shared__ uint64_t s_pre[kQMaxTargets], s_cnt[kQMaxTargets];
  for (int j = threadIdx.x; j < n_t; j += blockDim.x) {
    s_pre[j] = t[j].pre;
    s_cnt[j] = t[j].cnt;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n_t; j += blockDim.x) {
    uint32_t r = (uint32_t)j;
    for (int i = 0; i < j; ++i)
      if (s_pre[i] == s_pre[j]) {
        r = (uint32_t)i;
        break;
      }
    s_row[j] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // a few hundred rows: serial offsets
    uint64_t o = 0;
    for (int j = 0; j < n_t; ++j)
      if (s_row[j] == (uint32_t)j) {
        ri[j].off = o;
        ri[j].size = s_cnt[j];
        o += s_cnt[j];
      }
  }
  for (int j = threadIdx.x; j < n_t; j += blockDim.x) {
    ri[j].row = s_row[j];
    ri[j].fill = 0u;
  }
}

// The keys under each 24-bit target prefix, appended to that prefix's list.
// A CTA takes a contiguous chunk: counts per row in shared memory, reserves
// each row's share with one global atomic, then places its keys (heavily
// tied columns would otherwise queue on a few global counters).
__global__ void __launch_bounds__(kQPassThreads) collect_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                                const Target* __restrict__ t, int n_t,
                                                                RowInfo* __restrict__ ri,
                                                                uint64_t* __restrict__ list) {
  __shared__ PrefixHash h;
  __shared__ uint32_t s_cnt[kQMaxTargets];
  __shared__ uint64_t s_base[kQMaxTargets];
  build_hash(h, t, n_t);
  const uint64_t m = hi_mask(2 * kQBits);
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  for (int i = threadIdx.x; i < h.n_rows; i += blockDim.x) s_cnt[i] = 0u;
  __syncthreads();
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const int x = find_slot(h, keys[i] & m);
    if (x >= 0) atomicAdd(s_cnt + h.cid[x], 1u);
  }
  __syncthreads();
  for (int x = threadIdx.x; x < kQHash; x += blockDim.x)
    if (h.key[x] != kQEmpty) {
      const int c = h.cid[x], r = h.row[x];
      s_base[c] = s_cnt[c] ? ri[r].off + atomicAdd(&ri[r].fill, s_cnt[c]) : 0ull;
    }
  __syncthreads();
  for (int i = threadIdx.x; i < h.n_rows; i += blockDim.x) s_cnt[i] = 0u;
  __syncthreads();
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint64_t k = keys[i];
    const int x = find_slot(h, k & m);
    if (x >= 0) {
      const int c = h.cid[x];
      list[s_base[c] + atomicAdd(s_cnt + c, 1u)] = k;
    }
  }
}

// A CTA per target: the key of rank rem in its row's list (every key there
// shares the target's 24-bit prefix), by four 10-bit passes over the list
// with a shared-memory histogram.
__global__ void __launch_bounds__(kQResolveThreads) final_select_kernel(Target* __restrict__ t,
                                                                        const RowInfo* __restrict__ ri,
                                                                        const uint64_t* __restrict__ list) {
  constexpr int bins = 1 << kQFinalBits, per = bins / kQResolveThreads;
  __shared__ uint32_t s_hist[bins];
  __shared__ uint32_t s_wsum[kQResolveThreads / 32];
  __shared__ uint64_t s_hit[3];
  const int tid = threadIdx.x;
  const RowInfo head = ri[ri[blockIdx.x].row];
  const uint64_t* L = list + head.off;
  uint64_t pre = t[blockIdx.x].pre, rem = t[blockIdx.x].rem;
  for (int resolved = 2 * kQBits; resolved < 64; resolved += kQFinalBits) {
    const int shift = 64 - resolved - kQFinalBits;  // 30, 20, 10, 0
    const uint64_t m = hi_mask(resolved);
    for (int i = tid; i < bins; i += blockDim.x) s_hist[i] = 0u;
    __syncthreads();
    for (uint64_t i = tid; i < head.size; i += blockDim.x) {
      const uint64_t k = L[i];
      if ((k & m) == pre) atomicAdd(s_hist + ((uint32_t)(k >> shift) & (bins - 1)), 1u);
    }
    __syncthreads();
    uint32_t c[per];
#pragma unroll
    for (int q = 0; q < per; ++q) c[q] = s_hist[tid * per + q];
    find_bin<kQResolveThreads, per>(c, rem, s_wsum, s_hit);
    pre |= s_hit[0] << shift;
    rem = s_hit[1];
  }
  if (tid == 0) t[blockIdx.x].pre = pre;
}

__global__ void lerp_kernel(const Target* t, int64_t n, const double* qs, int32_t n_q, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_q) return;
  const double last = key_value(t[2 * n_q].pre);
  if (isnan(last)) {
    out[i] = last;
    return;
  }
  int64_t prev, next;
  double v, fl;
  quantile_ranks(n, qs[i], prev, next, v, fl);
  // numpy: gamma = v - previous_indexes after the bound fix-ups (-1 / 0)
  const double prev_idx = v >= (double)(n - 1) ? -1.0 : (v < 0.0 ? 0.0 : fl);
  const double g = __dadd_rn(v, -prev_idx);
  const double lo = key_value(t[2 * i].pre), hi = key_value(t[2 * i + 1].pre);
  const double diff = __dadd_rn(hi, -lo);
  out[i] = g >= 0.5 ? __dadd_rn(hi, -__dmul_rn(diff, __dadd_rn(1.0, -g)))
                    : __dadd_rn(lo, __dmul_rn(diff, g));
}

struct QLayout {
  size_t keys, list, qs, tgt0, tgt1, rows, hist0, hist1, bytes;
};
QLayout q_layout(int64_t n, int32_t n_q) {
  const int n_t = 2 * std::min(n_q, kQChunk) + 1;
  QLayout L{};
  size_t o = 0;
  auto take = [&](size_t b) {
    const size_t at = o;
    o += round_up(b, 256);
    return at;
  };
  L.keys = take((size_t)n * 8);
  L.list = take((size_t)n * 8);
  L.qs = take((size_t)std::max(n_q, 1) * 8);
  L.tgt0 = take((size_t)n_t * sizeof(Target));
  L.tgt1 = take((size_t)n_t * sizeof(Target));
  L.rows = take((size_t)n_t * sizeof(RowInfo));
  L.hist0 = take((size_t)kQBins * 4);
  L.hist1 = take((size_t)n_t * kQBins * 4);
  L.bytes = o;
  return L;
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" int gs_quantiles_workspace(int64_t n, int32_t n_q, size_t* bytes) {
  GS_REQUIRE(bytes && n > 0 && n_q >= 0);
  if (n >= (int64_t)1 << 40) return GS_EUNSUPPORTED;
  *bytes = q_layout(n, n_q).bytes;
  return GS_OK;
}

extern "C" int gs_quantiles(const double* column, int64_t n, int64_t stride, const double* qs,
                            int32_t n_q, double* out, void* workspace, size_t workspace_bytes,
                            void* stream) {
  GS_REQUIRE(column && n > 0 && stride >= 1 && n_q >= 0 && (n_q == 0 || (qs && out)));
  size_t need = 0;
  int rc = gs_quantiles_workspace(n, n_q, &need);
  if (rc != GS_OK) return rc;
  if (!workspace || workspace_bytes < need) return GS_EWORKSPACE;
  for (int i = 0; i < n_q; ++i)
    if (!(qs[i] >= 0.0 && qs[i] <= 1.0)) return GS_EINVAL;  // numpy: "Quantiles must be in [0, 1]"
  if (n_q == 0) return GS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const QLayout L = q_layout(n, n_q);
  uint64_t* keys = reinterpret_cast<uint64_t*>(ws + L.keys);
  uint64_t* list = reinterpret_cast<uint64_t*>(ws + L.list);
  double* dq = reinterpret_cast<double*>(ws + L.qs);
  Target* t0 = reinterpret_cast<Target*>(ws + L.tgt0);
  Target* t1 = reinterpret_cast<Target*>(ws + L.tgt1);
  RowInfo* rows = reinterpret_cast<RowInfo*>(ws + L.rows);
  uint32_t* hist0 = reinterpret_cast<uint32_t*>(ws + L.hist0);
  uint32_t* hist1 = reinterpret_cast<uint32_t*>(ws + L.hist1);
  // the key passes: a few CTAs per SM (each builds the prefix hash once)
  const int64_t blocks =
      std::max<int64_t>(1, std::min<int64_t>((n + kQPassThreads - 1) / kQPassThreads, (int64_t)sm_count() * 2));
  GS_CUDA_TRY(cudaMemcpyAsync(dq, qs, (size_t)n_q * 8, cudaMemcpyHostToDevice, st));
  GS_CUDA_TRY(cudaMemsetAsync(hist0, 0, (size_t)kQBins * 4, st));
  // the keys and their top-12-bit histogram serve every round of targets
  gather_pass0_kernel<<<(unsigned)blocks, kQPassThreads, 0, st>>>(column, n, stride, keys, hist0);
  GS_LAUNCH_CHECK();
  static SmemAttr pass1_attr;
  const size_t pass1_smem = (size_t)kQPrivRows * kQBins * 4;
  GS_CUDA_TRY(ensure_smem(pass1_kernel, pass1_attr, pass1_smem));
  for (int q0 = 0; q0 < n_q; q0 += kQChunk) {  // up to kQChunk quantiles (2 kQChunk + 1 targets) a round
    const int nq = std::min(kQChunk, n_q - q0), n_t = 2 * nq + 1;
    init_targets_kernel<<<(nq + 1 + 127) / 128, 128, 0, st>>>(dq + q0, nq, n, t0);
    GS_LAUNCH_CHECK();
    // every target starts at prefix 0 (row 0 of the one-row pass-0 histogram);
    // this resolve also zeroes pass 1's rows
    resolve_kernel<<<(unsigned)n_t, kQResolveThreads, 0, st>>>(t0, t1, n_t, 0, hist0, hist1);
    GS_LAUNCH_CHECK();
    pass1_kernel<<<(unsigned)blocks, kQPassThreads, pass1_smem, st>>>(keys, n, t1, n_t, hist1);
    GS_LAUNCH_CHECK();
    resolve_kernel<<<(unsigned)n_t, kQResolveThreads, 0, st>>>(t1, t0, n_t, kQBits, hist1, nullptr);
    GS_LAUNCH_CHECK();
    plan_rows_kernel<<<1, 1024, 0, st>>>(t0, n_t, rows);
    GS_LAUNCH_CHECK();
    collect_kernel<<<(unsigned)blocks, kQPassThreads, 0, st>>>(keys, n, t0, n_t, rows, list);
    GS_LAUNCH_CHECK();
    final_select_kernel<<<(unsigned)n_t, kQResolveThreads, 0, st>>>(t0, rows, list);
    GS_LAUNCH_CHECK();
    lerp_kernel<<<(nq + 127) / 128, 128, 0, st>>>(t0, n, dq + q0, nq, out + q0);
    GS_LAUNCH_CHECK();
  }
  return GS_OK;
}
