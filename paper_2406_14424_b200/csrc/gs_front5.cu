// gs_front5.cu — config 4a: the exact Pareto front of a five-model cascade
// over 1000-level threshold grids (~1e12 configs), never materialising a
// per-config output or a 4-D table.
//
// Reference semantics: every config (k0, k1, k2, k3) of the full cascade
// m0 -> m1 -> m2 -> m3 -> m4 is scored exactly as _evaluate_numba scores it
// (/root/reference/pkg/src/gearserve/kernels.py:39-62: correct count,
// frac = count / n, mean += frac * cost1 in stage order), and the output is
// pareto_filter's front over (accuracy, mean_cost) with exact ties
// (src/cascades.py:116-129).  A 1001^4 dominance table (16 TB) is out of
// reach, so the counts come from streaming instead:
//
//   records are sorted by (b2, b0); a CTA owns one k0 and a group of k1
//   values (a warp each).  It walks k2 = 0 .. g2-1: the records of bucket
//   b2 = k2 with b0 <= k0 are a prefix of that bucket (pre02), streamed
//   through shared memory; each warp adds those with b1 <= k1 to its b3
//   histogram (R4 = the records reaching stage 4; a bin is one u64: the
//   count in the low word, C4 - C3 two's-complement in the high word -- the
//   low word never carries, n < 2^21 -- so a prefix sum gives reach5 and
//   the correct count's change without unpacking), then scores
//   the row (k0, k1, k2, k3 = 0 .. g3-1) from the histogram's prefix:
//     reach5(k3) = #(R4, b3 <= k3), correct = C0 + C1 + C2 (row terms)
//                + C3(R4) - C3(R4, b3 <= k3) + C4(R4, b3 <= k3)
//   O(1) per config after an O(d3) prefix per row.
//
// Two passes (exactness): the cost of a row's configs is non-decreasing in
// k3, so only configs whose correct count reaches the row's running maximum
// can be Pareto points ("staircase"); of those, any that some already seen
// config strictly dominates is dropped (a suffix minimum of the best cost per
// accuracy bucket, refreshed from a global array); the rest lower
// mincost[correct] (atomicMin on the order-preserving cost bits).  A dropped
// config is dominated by a recorded one, so after pass 1 mincost is exact
// for every accuracy on the front, and the front's accuracies are those
// whose mincost is below every higher accuracy's.  Pass 2 re-walks and
// emits every config whose (correct, cost) equals a front pair -- ties
// included -- with its stage reach counts.
#include "gs_front5.cuh"

namespace gs {
namespace {

constexpr int kF5Warps = 24;              // k1 values per CTA (a warp each)
constexpr int kF5Bins = 1024;             // histogram bins (d3 <= 1024)
constexpr uint64_t kF5Inf = 0x7f7f7f7f7f7f7f7full;  // empty min-cost key (a memset 0x7f fill);
                                                    // above every cost key (costs < 1e300)

__device__ __forceinline__ uint64_t cost_key(double c) {  // c >= 0: bits are monotone
  return (uint64_t)__double_as_longlong(c);
}

// bin b = 32 l + t lives at t * 32 + l, so lane l reading its 32 bins in
// order touches 32 consecutive words per step (no bank conflicts)
__device__ __forceinline__ int bin_pos(int b) { return (b & 31) * 32 + (b >> 5); }

__device__ __forceinline__ int bin_of10(const double* g, int n, double x) {
  int base = 0, len = n;
  while (len > 1) {
    const int half = len >> 1;
    base = (g[base + half - 1] <= x) ? base + half : base;
    len -= half;
  }
  return base + (g[base] <= x ? 1 : 0);
}

struct F5BinArgs {
  const double* cert;
  const uint8_t* corr;
  int64_t n_rec;
  const double* grids;
  int32_t goff[4], glen[4];
  int32_t d0, d1;
  uint64_t* tmp;      // [n] sort key (b2 << 10 | b0) << 32 | record key
  uint32_t* cnt02;    // [d2][d0] records per (b2, b0)  (zero on entry)
  uint32_t* s01;      // [d0][d1][4] {cnt, c1, c2, -} per (b0, b1) (zero on entry)
  uint32_t* c0;       // [d0] model 0 correct per b0 (zero on entry)
};

__global__ void __launch_bounds__(256) f5_bin_kernel(const __grid_constant__ F5BinArgs a) {
  extern __shared__ double s_g[];
  const int ng = a.goff[3] + a.glen[3];
  for (int i = threadIdx.x; i < ng; i += blockDim.x) s_g[i] = a.grids[i];
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.n_rec;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double* x = a.cert + r * 5;
    const uint8_t* k = a.corr + r * 5;
    const uint32_t b0 = bin_of10(s_g + a.goff[0], a.glen[0], __ldg(x + 0));
    const uint32_t b1 = bin_of10(s_g + a.goff[1], a.glen[1], __ldg(x + 1));
    const uint32_t b2 = bin_of10(s_g + a.goff[2], a.glen[2], __ldg(x + 2));
    const uint32_t b3 = bin_of10(s_g + a.goff[3], a.glen[3], __ldg(x + 3));
    const uint32_t k0 = __ldg(k + 0) != 0, k1 = __ldg(k + 1) != 0, k2 = __ldg(k + 2) != 0,
                   k3 = __ldg(k + 3) != 0, k4 = __ldg(k + 4) != 0;
    const uint32_t key = b1 | (b3 << 10) | (k2 << 20) | (k3 << 21) | (k4 << 22);
    a.tmp[r] = ((uint64_t)((b2 << 10) | b0) << 32) | key;
    atomicAdd(a.cnt02 + (int64_t)b2 * a.d0 + b0, 1u);
    uint32_t* s = a.s01 + ((int64_t)b0 * a.d1 + b1) * 4;
    atomicAdd(s, 1u);
    if (k1) atomicAdd(s + 1, 1u);
    if (k2) atomicAdd(s + 2, 1u);
    if (k0) atomicAdd(a.c0 + b0, 1u);
  }
}

// Inclusive prefix along the last dimension of rows of uint32 x vec (a CTA
// per row, a warp scan per 32 elements), optionally rewriting in place.
__global__ void __launch_bounds__(256) f5_rowscan_kernel(uint32_t* t, int64_t rows, int len, int vec) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t row = blockIdx.x * 8 + warp; row < rows; row += (int64_t)gridDim.x * 8) {
    uint32_t* base = t + row * len * vec;
    for (int c = 0; c < vec; ++c) {
      uint32_t carry = 0;
      for (int j0 = 0; j0 < len; j0 += 32) {
        const int j = j0 + lane;
        uint32_t x = j < len ? base[j * vec + c] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        x += carry;
        if (j < len) base[j * vec + c] = x;
        carry = __shfl_sync(0xffffffffu, x, 31);
      }
    }
  }
}

// Inclusive prefix along the first dimension of a [rows][cols x vec] table
// (a thread per column element, rows walked in order).
__global__ void __launch_bounds__(256) f5_colscan_kernel(uint32_t* t, int rows, int64_t cols_x_vec) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cols_x_vec;
       c += (int64_t)gridDim.x * blockDim.x) {
    uint32_t run = 0;
    for (int r = 0; r < rows; ++r) {
      run += t[r * cols_x_vec + c];
      t[r * cols_x_vec + c] = run;
    }
  }
}

// bucket starts of b2 (exclusive scan of the (b2, b0) counts, which the
// row scan turned into per-b2 inclusive prefixes over b0) and scatter
// cursors; one CTA.
__global__ void __launch_bounds__(1024) f5_offsets_kernel(const uint32_t* pre02, int d2, int d0,
                                                          uint32_t* bstart, uint32_t* cur) {
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int b = 0; b < d2; b += 1024) {
    const int i = b + threadIdx.x;
    const uint32_t v = i < d2 ? pre02[(int64_t)i * d0 + d0 - 1] : 0u;  // bucket size
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
    if (i < d2) bstart[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) bstart[d2] = s_carry;
  __syncthreads();
  // cursor of (b2, b0) = bucket start + records of the bucket with smaller b0
  for (int64_t i = threadIdx.x; i < (int64_t)d2 * d0; i += 1024) {
    const int b2 = (int)(i / d0), b0 = (int)(i % d0);
    cur[i] = bstart[b2] + (b0 ? pre02[i - 1] : 0u);
  }
}

__global__ void __launch_bounds__(256) f5_scatter_kernel(const uint64_t* tmp, int64_t n, int d0, uint32_t* cur,
                                                         uint32_t* keys) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t t = tmp[r];
    const uint32_t sk = (uint32_t)(t >> 32);
    const int64_t cell = (int64_t)(sk >> 10) * d0 + (sk & 1023u);
    keys[atomicAdd(cur + cell, 1u)] = (uint32_t)t;
  }
}

struct F5PassArgs {
  int32_t g0, g1, g2, g3, d0, d1;
  int32_t pass;                 // 1: min costs, 2: emit the front
  int32_t k0_begin, k0_end;
  int32_t k0_stride;            // CTA group i takes k0 = k0_begin + i * k0_stride (< k0_end)
  int32_t n_groups;             // k1 groups of kF5Warps
  int32_t bucket_shift;         // accuracy bucket = correct >> shift (kF5Bins buckets)
  int64_t n_rec;
  double rcp_n;
  const double* cost1;
  const uint32_t* keys;         // records sorted by (b2, b0)
  const uint32_t* bstart;       // [d2 + 1]
  const uint32_t* pre02;        // [d2][d0] inclusive prefix over b0 of bucket b2's counts
  const uint32_t* s01;          // [d0][d1][4] 2-D prefix {cnt, c1, c2, -}
  const uint32_t* c0pre;        // [d0] prefix of model 0's correct count
  unsigned long long* mincost;  // [n_rec + 1] order-preserving cost keys
  unsigned long long* gbest;    // [kF5Bins] min cost key per accuracy bucket
  const unsigned long long* front_key;  // pass 2: [n_rec + 1] the front pair's cost key or kF5Inf
  uint32_t* row_flag;           // [g0][g1][n_words] bit k2: pass 1 saw a config of row (k0, k1, k2)
                                // at or below mincost[correct] as it stood then
  const uint8_t* k0_done;       // [g0] pass 1 has flagged this k0's rows
  int32_t n_words;
  // pass 2 outputs
  unsigned long long* out_idx;  // config index within the full cascade
  double* out_cost;
  uint32_t* out_rec;            // [cap][6] correct, reach1..reach5 (reach1 = n)
  unsigned long long* out_count;
  int64_t out_cap;              // 0: the per-point summary only
  unsigned long long* ties;     // [n_rec + 1] front configs per accuracy
  unsigned long long* min_index;  // [n_rec + 1] smallest front config index per accuracy
};

// the suffix minimum of gbest (smin[j] = min over buckets >= j): every
// thread of the CTA fetches part of gbest into smin (all loads in flight at
// once), then one warp turns it into suffix minima in place.  Called by the
// whole CTA (it synchronises).
__device__ void refresh_bound(const F5PassArgs& a, unsigned long long* smin) {
  for (int j = threadIdx.x; j < kF5Bins; j += blockDim.x)
    smin[j] = *reinterpret_cast<volatile const unsigned long long*>(a.gbest + j);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  unsigned long long carry = kF5Inf;
  for (int j0 = kF5Bins - 32; j0 >= 0; j0 -= 32) {
    unsigned long long x = smin[j0 + lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_down_sync(0xffffffffu, x, o);
      if (lane + o < 32 && y < x) x = y;
    }
    x = x < carry ? x : carry;
    smin[j0 + lane] = x;
    carry = __shfl_sync(0xffffffffu, x, 0);
  }
}

// The same, by one warp and without barriers, while the other warps keep
// reading: each entry is only ever lowered to a suffix minimum of a newer
// gbest, and any value an entry holds is the cost of a recorded config in a
// bucket at or above it -- a valid bound at every moment.
__device__ void refresh_bound_warp(const F5PassArgs& a, unsigned long long* smin) {
  const int lane = threadIdx.x & 31;
  unsigned long long carry = kF5Inf;
#pragma unroll 4
  for (int j0 = kF5Bins - 32; j0 >= 0; j0 -= 32) {
    unsigned long long x = __ldcg(a.gbest + j0 + lane);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_down_sync(0xffffffffu, x, o);
      if (lane + o < 32 && y < x) x = y;
    }
    x = x < carry ? x : carry;
    atomicMin(smin + j0 + lane, x);  // an atomic: the readers race with it by design
    carry = __shfl_sync(0xffffffffu, x, 0);
  }
}

__global__ void __launch_bounds__(kF5Warps * 32, 1) f5_pass_kernel(const __grid_constant__ F5PassArgs a) {
  extern __shared__ __align__(16) unsigned long long s_hist[];  // [kF5Warps][kF5Bins]
  __shared__ unsigned long long s_smin[kF5Bins + 1];             // suffix min of gbest
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k0 = a.k0_begin + (int)(blockIdx.x / a.n_groups) * a.k0_stride;
  const int k1 = (blockIdx.x % a.n_groups) * kF5Warps + warp;
  const bool wlive = k1 < a.g1;
  __shared__ int s_k2end;
  unsigned long long* hist = s_hist + (size_t)warp * kF5Bins;
  for (int b = lane; b < kF5Bins; b += 32) hist[b] = 0ull;
  if (threadIdx.x == 0) s_k2end = a.pass == 1 ? a.g2 - 1 : -1;
  refresh_bound(a, s_smin);
  if (threadIdx.x == 0) s_smin[kF5Bins] = kF5Inf;
  // pass 2 scores only the rows pass 1 flagged (every row on the front is
  // one: see f5_pass2), and walks k2 only as far as the last of them; lane
  // j holds the warp's flag word j (k2 = 32 j ..)
  uint32_t fword = 0xffffffffu;
  int wlast = a.g2 - 1;
  if (a.pass == 2) {
    if (!wlive) {
      fword = 0u;
    } else if (__ldg(a.k0_done + k0)) {
      fword = lane < a.n_words ? __ldg(a.row_flag + ((int64_t)k0 * a.g1 + k1) * a.n_words + lane) : 0u;
    }
    const uint32_t nz = __ballot_sync(0xffffffffu, fword != 0u);
    const int hl = nz ? 31 - __clz(nz) : -1;
    wlast = hl < 0 ? -1 : 32 * hl + 31 - __clz(__shfl_sync(0xffffffffu, fword, hl));
    wlast = min(wlast, a.g2 - 1);
    if (lane == 0 && wlast >= 0) atomicMax(&s_k2end, wlast);
  }
  __syncthreads();
  const int k2_end = s_k2end;
  const double n = (double)a.n_rec, rcp = a.rcp_n;
  const double one = div_count(n, n, rcp);
  const double c0 = __ldg(a.cost1), c1 = __ldg(a.cost1 + 1), c2 = __ldg(a.cost1 + 2),
               c3 = __ldg(a.cost1 + 3), c4 = __ldg(a.cost1 + 4);
  // row-shared terms of (k0, k1): reach2 = #(b0 <= k0), reach3 = #(b0 <= k0, b1 <= k1)
  const int g0 = a.g0, g1 = a.g1, g3 = a.g3;
  const uint4 s0g = *reinterpret_cast<const uint4*>(a.s01 + ((int64_t)k0 * a.d1 + g1) * 4);
  const uint4 s01 = wlive ? *reinterpret_cast<const uint4*>(a.s01 + ((int64_t)k0 * a.d1 + k1) * 4)
                          : make_uint4(0, 0, 0, 0);
  const uint32_t reach2 = s0g.x, reach3 = s01.x;
  const double fr1 = div_count((double)reach2, n, rcp);
  const double fr2 = div_count((double)reach3, n, rcp);
  const double m2 = dadd(dadd(dadd(0.0, dmul(one, c0)), dmul(fr1, c1)), dmul(fr2, c2));
  // correct through stage 1: C0 of b0 > k0, C1 of (b0 <= k0, b1 > k1)
  const uint32_t base01 = (__ldg(a.c0pre + g0) - __ldg(a.c0pre + k0)) + (s0g.y - s01.y);
  const uint32_t c2_r3 = s01.z;  // C2 over R3
  uint32_t c2_r4 = 0, reach4 = 0, c3_r4 = 0, p4_r4 = 0;
  const int64_t k01 = ((int64_t)k0 * g1 + k1) * a.g2;
  bool rflag = false;  // pass 1: this row has a config at or below mincost
  // the warps walk their rows independently (no barriers): each streams the
  // records itself (the CTA's warps read the same lines, L1 hits after the
  // first), and in pass 1 one warp in turn pulls in the bound the rest of the
  // grid has found every 16 rows
  for (int k2 = 0; k2 <= k2_end; ++k2) {
    if (a.pass == 1 && (k2 & 15) == 15 && ((k2 >> 4) % kF5Warps) == warp) refresh_bound_warp(a, s_smin);
    if (!wlive || k2 > wlast) continue;
    // stream bucket b2 = k2, records with b0 <= k0 (a prefix of the bucket)
    const uint32_t beg = __ldg(a.bstart + k2), cnt = __ldg(a.pre02 + (int64_t)k2 * a.d0 + k0);
    {
      for (uint32_t t0 = 0; t0 < cnt; t0 += 32) {
        const uint32_t t = t0 + lane;
        const uint32_t k = t < cnt ? __ldg(a.keys + beg + t) : 0xffffffffu;
        const bool in = t < cnt && (k & 1023u) <= (uint32_t)k1;
        const uint32_t m = __ballot_sync(0xffffffffu, in);
        const uint32_t m3 = __ballot_sync(0xffffffffu, in && ((k >> 21) & 1u));
        const uint32_t m4 = __ballot_sync(0xffffffffu, in && ((k >> 22) & 1u));
        reach4 += __popc(m);
        c2_r4 += __popc(__ballot_sync(0xffffffffu, in && ((k >> 20) & 1u)));
        c3_r4 += __popc(m3);
        p4_r4 += __popc(m4 & ~m3);  // R4 records whose stage-4 answer adds a correct one
        if (in) {  // the lanes of one b3 bin add as one: its lowest lane applies their sum
          const uint32_t b3 = (k >> 10) & 1023u;
          const uint32_t peers = __match_any_sync(m, b3);
          if (lane == __ffs(peers) - 1)
            hist[bin_pos((int)b3)] +=
                (uint64_t)__popc(peers) +
                ((uint64_t)(int64_t)(__popc(peers & m4) - __popc(peers & m3)) << 32);
        }
        __syncwarp();
      }
    }
    const bool flagged = (__shfl_sync(0xffffffffu, fword, k2 >> 5) >> (k2 & 31)) & 1u;
    if (!flagged) continue;
    // score row (k0, k1, k2): lane l owns k3 = 32 l .. 32 l + 31
    const double fr3 = div_count((double)reach4, n, rcp);
    const double m3 = dadd(m2, dmul(fr3, c3));
    const uint32_t crow = base01 + (c2_r3 - c2_r4) + c3_r4;  // + C4(k3) - C3(k3) per config
    {  // the whole row at once: no config of it is more accurate than
       // crow + #(R4 records with C4 and not C3) -- a config's count is crow
       // plus its prefix of C4 - C3, at most the +1 records -- and none is
       // cheaper than k3 = 0 (reach5 = bin 0); if the bound of that accuracy
       // already beats that cost, every config of the row would be dropped
      const uint64_t key0 = cost_key(dadd(m3, dmul(div_count((double)(uint32_t)hist[0], n, rcp), c4)));
      const uint32_t ub = min(crow + p4_r4, (uint32_t)a.n_rec);
      if (s_smin[(int)(ub >> a.bucket_shift) + 1] <= key0) continue;
    }
    // lane totals, their exclusive scan (the prefix before this lane's bins),
    // each lane's highest correct count, and the running maximum over the
    // lanes before it (configs with smaller k3 cost no more)
    // one pass over the lane's bins: its total and the largest C4 - C3 of
    // its local prefixes (a config's correct count is crow + (C4 - C3)(prefix
    // before the lane) + that local difference)
#ifndef GS_F5_SUB
#define GS_F5_SUB 2  // halves: 4 and 8 blocks measured slower (1.18, 1.43 s against 1.16)
#endif
    constexpr int kSub = GS_F5_SUB, kLen = 32 / GS_F5_SUB;  // blocks of configs per lane
    uint64_t tot = 0;
    uint64_t pre[kSub];  // the prefix of the lane's bins before block q
    int dq[kSub];        // the largest local C4 - C3 over block q's configs
#pragma unroll
    for (int q = 0; q < kSub; ++q) {
      pre[q] = tot;
      int d = -(1 << 22);
#pragma unroll
      for (int u = 0; u < kLen; ++u) {
        tot += hist[(q * kLen + u) * 32 + lane];
        d = max(d, (int)(tot >> 32));
      }
      dq[q] = d;
    }
    int dmax = dq[0];
#pragma unroll
    for (int q = 1; q < kSub; ++q) dmax = max(dmax, dq[q]);
    uint64_t excl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, excl, o);
      if (lane >= o) excl += y;
    }
    excl -= tot;
    const uint32_t amax =
        32 * lane < g3 ? (uint32_t)((int)crow + (int)(excl >> 32) + dmax) : 0u;
    uint32_t pmax = amax;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, pmax, o);
      if (lane >= o) pmax = max(pmax, y);
    }
    uint32_t run_max = __shfl_up_sync(0xffffffffu, pmax, 1);
    if (lane == 0) run_max = 0;
    uint64_t acc = excl;
    uint32_t cur_a = 0xffffffffu, run_n = 0, first_k3 = 0xffffffffu;  // pass 2: run of one front point
    // the whole lane at once: its cheapest config is its first (cost is
    // non-decreasing in k3) and every config's accuracy bucket is at most
    // amax's, whose bound is the loosest (a suffix minimum); if that bound
    // already beats the cheapest cost, the in-loop test below would drop
    // every config of the lane
    // The same per block of kLen configs (each block's own largest count
    // and cheapest config): a block whose bound beats its cheapest config
    // holds only dominated configs and is skipped.  (A skipped block leaves
    // run_max lower after it: more configs pass the staircase test there,
    // each still a real config's cost.)
    bool lane_live = 32 * lane < g3;
    uint64_t lane_bound = kF5Inf;
    uint64_t qbound[kSub];
    uint32_t qsuf[kSub];  // the largest count over blocks q.. (pass 1's exit)
    uint32_t live_mask = 0;
    if (lane_live) {
      const uint32_t r5 = (uint32_t)(excl + hist[lane]);
      const uint64_t key0 = cost_key(dadd(m3, dmul(div_count((double)r5, n, rcp), c4)));
      lane_bound = s_smin[(int)(amax >> a.bucket_shift) + 1];
      lane_live = lane_bound > key0;
      // pass 1 scores only configs above the row's running maximum: none
      // of this lane's is when an earlier lane already reached its amax
      if (a.pass == 1 && lane > 0 && amax <= run_max) lane_live = false;
      if (lane_live) {
        uint32_t suf = 0;
#pragma unroll
        for (int q = kSub - 1; q >= 0; --q) {
          const uint32_t am = (uint32_t)((int)crow + (int)(excl >> 32) + dq[q]);
          suf = max(suf, am);
          qsuf[q] = suf;
          qbound[q] = kF5Inf;
          bool lv = 32 * lane + q * kLen < g3;
          if (lv) {
            const uint64_t k0q =
                q == 0 ? key0
                       : cost_key(dadd(m3, dmul(div_count((double)(uint32_t)(excl + pre[q] +
                                                                              hist[q * kLen * 32 + lane]),
                                                          n, rcp),
                                               c4)));
            qbound[q] = s_smin[(int)(am >> a.bucket_shift) + 1];
            lv = qbound[q] > k0q && !(a.pass == 1 && lane > 0 && am <= run_max);
          }
          live_mask |= lv ? 1u << q : 0u;
        }
      }
    }
    if (!lane_live) live_mask = 0;
    bool stop = false;
#pragma unroll 1
    for (int q = 0; q < kSub && !stop; ++q) {
      if (!((live_mask >> q) & 1u)) continue;
      acc = excl + pre[q];
#pragma unroll 4
    for (int u = 0; u < kLen; ++u) {
      const int t = q * kLen + u;
      const int k3 = 32 * lane + t;
      // ... and none of the rest of the lane once it has reached the largest
      // count of the blocks left
      if (a.pass == 1 && k3 > 0 && run_max >= qsuf[q]) {
        stop = true;
        break;
      }
      acc += hist[t * 32 + lane];
      if (k3 >= g3) {
        stop = true;
        break;
      }
      const uint32_t reach5 = (uint32_t)acc;
      const uint32_t correct = crow + (uint32_t)(acc >> 32);
      // pass 1 keeps only a row's first config of each new correct count:
      // later ones with the same count cost no less (cost is non-decreasing
      // in k3), so they cannot lower mincost; pass 2 also needs their exact
      // ties
      const bool stair = a.pass == 1 ? (correct > run_max || k3 == 0) : correct >= run_max;
      run_max = max(run_max, correct);
      if (!stair) continue;
      const double fr4 = div_count((double)reach5, n, rcp);
      const double mean = dadd(m3, dmul(fr4, c4));
      const uint64_t key = cost_key(mean);
      // the same test for the rest of the lane: its later configs cost no
      // less and reach at most amax's bucket, whose bound is the loosest
      if (key >= qbound[q]) break;  // the rest of this block
      const int bk = (int)(correct >> a.bucket_shift);
      if (s_smin[bk + 1] <= key) continue;  // a strictly more accurate config costs no more
      if (a.pass == 1) {
        // most surviving configs tie the recorded minimum (routing-equivalent
        // threshold tuples): a read skips their atomic
        const unsigned long long cur = __ldcg(a.mincost + correct);
        rflag |= cur >= key;
        if (cur <= key) continue;
        const unsigned long long old = atomicMin(a.mincost + correct, (unsigned long long)key);
        if (key < old) atomicMin(a.gbest + bk, (unsigned long long)key);
      } else if (__ldg(a.front_key + correct) == key) {
        if (correct != cur_a) {  // this lane's run of one front point ends
          if (run_n) {
            atomicAdd(a.ties + cur_a, (unsigned long long)run_n);
            atomicMin(a.min_index + cur_a, (unsigned long long)((k01 + k2) * g3 + first_k3));
          }
          cur_a = correct;
          run_n = 0;
          first_k3 = (uint32_t)k3;
        }
        ++run_n;
        if (a.out_cap == 0) continue;
        const unsigned long long slot = atomicAdd(a.out_count, 1ull);
        if ((int64_t)slot < a.out_cap) {
          a.out_idx[slot] = (unsigned long long)((k01 + k2) * g3 + k3);
          a.out_cost[slot] = mean;
          uint32_t* o = a.out_rec + slot * 6;
          o[0] = correct;
          o[1] = (uint32_t)a.n_rec;
          o[2] = reach2;
          o[3] = reach3;
          o[4] = reach4;
          o[5] = reach5;
        }
      }
    }
    }
    if (a.pass == 1) {
      if (__any_sync(0xffffffffu, rflag) && lane == 0)
        atomicOr(a.row_flag + ((int64_t)k0 * a.g1 + k1) * a.n_words + (k2 >> 5), 1u << (k2 & 31));
      rflag = false;
    }
    if (a.pass == 2) {  // the lanes' last runs: one atomic per distinct point in the warp
      const uint32_t live = __ballot_sync(0xffffffffu, run_n > 0);
      if (run_n > 0) {
        const uint32_t peers = __match_any_sync(live, cur_a);
        const uint32_t sum = __reduce_add_sync(peers, run_n);
        const uint32_t k3min = __reduce_min_sync(peers, first_k3);
        if (lane == __ffs(peers) - 1) {
          atomicAdd(a.ties + cur_a, (unsigned long long)sum);
          atomicMin(a.min_index + cur_a, (unsigned long long)((k01 + k2) * g3 + k3min));
        }
      }
    }
  }
}

// Pass 1 -> pass 2: the front's accuracies are those whose min cost is
// below every higher accuracy's; front_key[a] = mincost[a] there, else
// kF5Inf.  gbest2 = the front keys' bucket minima (pass 2's pruning bound).
__global__ void __launch_bounds__(1024) f5_front_kernel(const unsigned long long* mincost, int64_t n1,
                                                         unsigned long long* front_key,
                                                         unsigned long long* gbest, int shift,
                                                         unsigned long long* n_front) {
  __shared__ unsigned long long s_w[32];
  __shared__ unsigned long long s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_carry = kF5Inf;
    *n_front = 0;
  }
  for (int j = threadIdx.x; j < kF5Bins; j += 1024) gbest[j] = kF5Inf;
  __syncthreads();
  // walk accuracies from the top: suffix min over a' > a, 1024 at a time
  for (int64_t hi = n1; hi > 0; hi -= 1024) {
    const int64_t a = hi - 1 - threadIdx.x;  // this thread's accuracy (descending)
    const unsigned long long v = a >= 0 ? mincost[a] : kF5Inf;
    // inclusive min-scan in descending-accuracy order
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o && y < x) x = y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
      unsigned long long w = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o && y < w) w = y;
      }
      s_w[lane] = w;
    }
    __syncthreads();
    unsigned long long before = s_carry;  // min over accuracies above this block
    if (warp > 0 && s_w[warp - 1] < before) before = s_w[warp - 1];
    // exclusive: min over threads before this one (higher accuracies)
    unsigned long long ex = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) ex = kF5Inf;
    if (ex < before) before = ex;
    if (a >= 0) {
      const bool on = v < before;
      front_key[a] = on ? v : kF5Inf;
      if (on) {
        atomicMin(gbest + (a >> shift), v);
        atomicAdd(n_front, 1ull);
      }
    }
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = before < x ? before : x;
    __syncthreads();
  }
}

}  // namespace

bool f5_supported(int64_t n_rec, const int32_t* glen) {
  if (n_rec < 1 || n_rec >= (1ll << 21)) return false;
  for (int j = 0; j < 5; ++j)
    if (glen[j] < 1 || glen[j] > 1023) return false;
  return glen[3] + 1 <= kF5Bins;
}

F5Layout f5_layout(const int32_t* glen, int64_t n_rec) {
  F5Layout L{};
  L.d0 = glen[0] + 1;
  L.d1 = glen[1] + 1;
  L.d2 = glen[2] + 1;
  L.d3 = glen[3] + 1;
  int shift = 0;
  while (((n_rec + 1) >> shift) > kF5Bins) ++shift;
  L.bucket_shift = shift;
  size_t o = 0;
  auto take = [&](size_t b) {
    const size_t at = o;
    o += round_up(b, 256);
    return at;
  };
  L.offTmp = take((size_t)n_rec * 8);
  L.offKeys = take((size_t)n_rec * 4);
  L.offPre02 = take((size_t)L.d2 * L.d0 * 4);
  L.offCur = take((size_t)L.d2 * L.d0 * 4);
  L.offBstart = take((size_t)(L.d2 + 1) * 4);
  L.offS01 = take((size_t)L.d0 * L.d1 * 16);
  L.offC0 = take((size_t)L.d0 * 4);
  L.offMin = take((size_t)(n_rec + 1) * 8);
  L.offFront = take((size_t)(n_rec + 1) * 8);
  L.offGbest = take((size_t)kF5Bins * 8);
  L.offTies = take((size_t)(n_rec + 1) * 8);
  L.offMinIdx = take((size_t)(n_rec + 1) * 8);
  L.offNFront = take(256);
  L.n_words = (glen[2] + 31) / 32;
  L.offRowFlag = take((size_t)glen[0] * glen[1] * L.n_words * 4);
  L.offK0Done = take((size_t)glen[0]);
  L.bytes = o;
  return L;
}

cudaError_t f5_prepare(const double* cert, const uint8_t* corr, int64_t n_rec, const double* grids,
                       const int32_t* glen, uint8_t* ws, cudaStream_t st) {
  const F5Layout L = f5_layout(glen, n_rec);
  cudaError_t e;
  uint32_t* pre02 = reinterpret_cast<uint32_t*>(ws + L.offPre02);
  uint32_t* s01 = reinterpret_cast<uint32_t*>(ws + L.offS01);
  uint32_t* c0 = reinterpret_cast<uint32_t*>(ws + L.offC0);
  if ((e = cudaMemsetAsync(pre02, 0, (size_t)L.d2 * L.d0 * 4, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(s01, 0, (size_t)L.d0 * L.d1 * 16, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(c0, 0, (size_t)L.d0 * 4, st)) != cudaSuccess) return e;
  F5BinArgs b{};
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
  b.d0 = L.d0;
  b.d1 = L.d1;
  b.tmp = reinterpret_cast<uint64_t*>(ws + L.offTmp);
  b.cnt02 = pre02;
  b.s01 = s01;
  b.c0 = c0;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n_rec + 255) / 256, (int64_t)sm_count() * 8));
  const size_t gsm = (size_t)og * 8;
  static SmemAttr bin_attr;
  if ((e = ensure_smem(f5_bin_kernel, bin_attr, gsm)) != cudaSuccess) return e;
  f5_bin_kernel<<<(unsigned)blocks, 256, gsm, st>>>(b);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // pre02: prefix over b0 within each b2 bucket; s01: prefix over b1 then b0;
  // c0: prefix over b0
  f5_rowscan_kernel<<<(unsigned)std::min<int64_t>((L.d2 + 7) / 8, 4096), 256, 0, st>>>(pre02, L.d2, L.d0, 1);
  f5_rowscan_kernel<<<(unsigned)std::min<int64_t>((L.d0 + 7) / 8, 4096), 256, 0, st>>>(s01, L.d0, L.d1, 4);
  const int64_t cv = (int64_t)L.d1 * 4;
  f5_colscan_kernel<<<(unsigned)std::max<int64_t>(1, (cv + 255) / 256), 256, 0, st>>>(s01, L.d0, cv);
  f5_rowscan_kernel<<<1, 256, 0, st>>>(c0, 1, L.d0, 1);
  uint32_t* bstart = reinterpret_cast<uint32_t*>(ws + L.offBstart);
  uint32_t* cur = reinterpret_cast<uint32_t*>(ws + L.offCur);
  f5_offsets_kernel<<<1, 1024, 0, st>>>(pre02, L.d2, L.d0, bstart, cur);
  f5_scatter_kernel<<<(unsigned)blocks, 256, 0, st>>>(b.tmp, n_rec, L.d0, cur,
                                                      reinterpret_cast<uint32_t*>(ws + L.offKeys));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // min-cost keys and bucket bounds start empty
  if ((e = cudaMemsetAsync(ws + L.offMin, 0x7f, (size_t)(n_rec + 1) * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(ws + L.offGbest, 0x7f, (size_t)kF5Bins * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(ws + L.offRowFlag, 0, (size_t)L.offK0Done - L.offRowFlag + L.d0 - 1, st)) != cudaSuccess)
    return e;
  return cudaSuccess;
}

static F5PassArgs pass_args(const F5Layout& L, const int32_t* glen, int64_t n_rec, const double* cost1,
                            uint8_t* ws, int pass, int k0_begin, int k0_end) {
  F5PassArgs a{};
  a.g0 = glen[0];
  a.g1 = glen[1];
  a.g2 = glen[2];
  a.g3 = glen[3];
  a.d0 = L.d0;
  a.d1 = L.d1;
  a.pass = pass;
  a.k0_begin = k0_begin;
  a.k0_end = k0_end;
  a.k0_stride = 1;
  a.n_groups = (glen[1] + kF5Warps - 1) / kF5Warps;
  a.bucket_shift = L.bucket_shift;
  a.n_rec = n_rec;
  a.rcp_n = 1.0 / (double)n_rec;
  a.cost1 = cost1;
  a.keys = reinterpret_cast<const uint32_t*>(ws + L.offKeys);
  a.bstart = reinterpret_cast<const uint32_t*>(ws + L.offBstart);
  a.pre02 = reinterpret_cast<const uint32_t*>(ws + L.offPre02);
  a.s01 = reinterpret_cast<const uint32_t*>(ws + L.offS01);
  a.c0pre = reinterpret_cast<const uint32_t*>(ws + L.offC0);
  a.mincost = reinterpret_cast<unsigned long long*>(ws + L.offMin);
  a.gbest = reinterpret_cast<unsigned long long*>(ws + L.offGbest);
  a.front_key = reinterpret_cast<const unsigned long long*>(ws + L.offFront);
  a.row_flag = reinterpret_cast<uint32_t*>(ws + L.offRowFlag);
  a.k0_done = ws + L.offK0Done;
  a.n_words = L.n_words;
  return a;
}

cudaError_t f5_pass1(const int32_t* glen, int64_t n_rec, const double* cost1, uint8_t* ws, int k0_begin,
                     int k0_end, cudaStream_t st) {
  const F5Layout L = f5_layout(glen, n_rec);
  static SmemAttr attr;
  const size_t smem = (size_t)kF5Warps * kF5Bins * 8;
  cudaError_t e = ensure_smem(f5_pass_kernel, attr, smem);
  if (e != cudaSuccess) return e;
  // k0 slices of ~one wave each: every slice starts from the bound the
  // slices before it found.  First one wave of k0 values spread over the
  // range, so every later slice starts from a bound that already spans the
  // whole front (the pruning only drops configs a recorded one dominates,
  // so the order does not change the front; the spread k0 are scored again
  // in their slices, a few percent of the work)
  const int groups = (glen[1] + kF5Warps - 1) / kF5Warps;
  const int per = std::max(1, sm_count() / std::max(1, groups));
  const int span = k0_end - k0_begin;
  const int spread = std::min(4 * per, span / 8);  // k0 values in the first pass
  if (spread >= 2) {
    F5PassArgs a = pass_args(L, glen, n_rec, cost1, ws, 1, k0_begin, k0_end);
    a.k0_stride = span / spread;
    f5_pass_kernel<<<(unsigned)(spread * groups), kF5Warps * 32, smem, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
#ifndef GS_F5_SLICE_WAVES
#define GS_F5_SLICE_WAVES 0  // 0: the whole range in one launch (the CTAs refresh the bound every 16 rows)
#endif
  const int slice = GS_F5_SLICE_WAVES > 0 ? per * GS_F5_SLICE_WAVES : span;
  for (int k = k0_begin; k < k0_end; k += slice) {
    F5PassArgs a = pass_args(L, glen, n_rec, cost1, ws, 1, k, std::min(k0_end, k + slice));
    f5_pass_kernel<<<(unsigned)((a.k0_end - a.k0_begin) * groups), kF5Warps * 32, smem, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // these k0's row flags are complete (stream-ordered after the passes)
  if (k0_end > k0_begin &&
      (e = cudaMemsetAsync(ws + L.offK0Done + k0_begin, 1, (size_t)(k0_end - k0_begin), st)) != cudaSuccess)
    return e;
  return cudaSuccess;
}

cudaError_t f5_select(const int32_t* glen, int64_t n_rec, uint8_t* ws, unsigned long long* n_front,
                      cudaStream_t st) {
  const F5Layout L = f5_layout(glen, n_rec);
  cudaError_t e;
  if ((e = cudaMemsetAsync(ws + L.offTies, 0, (size_t)(n_rec + 1) * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(ws + L.offMinIdx, 0xff, (size_t)(n_rec + 1) * 8, st)) != cudaSuccess) return e;
  f5_front_kernel<<<1, 1024, 0, st>>>(reinterpret_cast<const unsigned long long*>(ws + L.offMin), n_rec + 1,
                                      reinterpret_cast<unsigned long long*>(ws + L.offFront),
                                      reinterpret_cast<unsigned long long*>(ws + L.offGbest), L.bucket_shift,
                                      n_front);
  return cudaGetLastError();
}

// Pass 2 scores only the rows pass 1 flagged, for the k0 that pass 1 has
// walked (others: every row).  Every row holding a front config is flagged:
// pass 1 drops a config only for one that strictly dominates it (not a
// front config) or, by the strict staircase, for an earlier config of the
// row with the same correct count and no higher cost -- which then ties the
// front point and is visited instead; a visited front config has cost ==
// the final mincost <= mincost when pass 1 read it, which flags the row.
// So the ties and smallest indices are those of the full walk.
cudaError_t f5_pass2(const int32_t* glen, int64_t n_rec, const double* cost1, uint8_t* ws, int k0_begin,
                     int k0_end, unsigned long long* out_idx, double* out_cost, uint32_t* out_rec,
                     unsigned long long* out_count, int64_t out_cap, cudaStream_t st) {
  const F5Layout L = f5_layout(glen, n_rec);
  static SmemAttr attr;
  const size_t smem = (size_t)kF5Warps * kF5Bins * 8;
  cudaError_t e = ensure_smem(f5_pass_kernel, attr, smem);
  if (e != cudaSuccess) return e;
  const int groups = (glen[1] + kF5Warps - 1) / kF5Warps;
  F5PassArgs a = pass_args(L, glen, n_rec, cost1, ws, 2, k0_begin, k0_end);
  a.out_idx = out_idx;
  a.out_cost = out_cost;
  a.out_rec = out_rec;
  a.out_count = out_count;
  a.out_cap = out_cap;
  a.ties = reinterpret_cast<unsigned long long*>(ws + L.offTies);
  a.min_index = reinterpret_cast<unsigned long long*>(ws + L.offMinIdx);
  if (k0_end > k0_begin)
    f5_pass_kernel<<<(unsigned)((k0_end - k0_begin) * groups), kF5Warps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace gs

// ------------------------------------------------------------------ C ABI --
using namespace gs;

extern "C" int gs_front5_plan(int64_t n_rec, const int32_t* grid_len, gs_front5_info* info) {
  GS_REQUIRE(grid_len && info && n_rec >= 1);
  if (!f5_supported(n_rec, grid_len)) return GS_EUNSUPPORTED;
  const F5Layout L = f5_layout(grid_len, n_rec);
  info->n_configs = (int64_t)grid_len[0] * grid_len[1] * grid_len[2] * grid_len[3];
  info->workspace_bytes = L.bytes;
  info->mincost_offset = L.offMin;
  info->front_offset = L.offFront;
  info->ties_offset = L.offTies;
  info->min_index_offset = L.offMinIdx;
  info->k0_count = grid_len[0];
  info->bucket_shift = L.bucket_shift;
  return GS_OK;
}

extern "C" int gs_front5_prepare(const double* certainty, const uint8_t* correct, int64_t n_rec,
                                 const double* grids, const int32_t* grid_len, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  GS_REQUIRE(certainty && correct && grids && grid_len && n_rec >= 1);
  if (!f5_supported(n_rec, grid_len)) return GS_EUNSUPPORTED;
  if (!workspace || workspace_bytes < f5_layout(grid_len, n_rec).bytes) return GS_EWORKSPACE;
  GS_CUDA_TRY(f5_prepare(certainty, correct, n_rec, grids, grid_len, static_cast<uint8_t*>(workspace),
                         static_cast<cudaStream_t>(stream)));
  return GS_OK;
}

extern "C" int gs_front5_pass1(int64_t n_rec, const int32_t* grid_len, const double* cost1,
                               int32_t k0_begin, int32_t k0_end, void* workspace, size_t workspace_bytes,
                               void* stream) {
  GS_REQUIRE(grid_len && cost1 && n_rec >= 1);
  if (!f5_supported(n_rec, grid_len)) return GS_EUNSUPPORTED;
  GS_REQUIRE(0 <= k0_begin && k0_begin <= k0_end && k0_end <= grid_len[0]);
  if (!workspace || workspace_bytes < f5_layout(grid_len, n_rec).bytes) return GS_EWORKSPACE;
  GS_CUDA_TRY(f5_pass1(grid_len, n_rec, cost1, static_cast<uint8_t*>(workspace), k0_begin, k0_end,
                       static_cast<cudaStream_t>(stream)));
  return GS_OK;
}

extern "C" int gs_front5_select(int64_t n_rec, const int32_t* grid_len, void* workspace,
                                size_t workspace_bytes, unsigned long long* n_front, void* stream) {
  GS_REQUIRE(grid_len && n_front && n_rec >= 1);
  if (!f5_supported(n_rec, grid_len)) return GS_EUNSUPPORTED;
  if (!workspace || workspace_bytes < f5_layout(grid_len, n_rec).bytes) return GS_EWORKSPACE;
  GS_CUDA_TRY(f5_select(grid_len, n_rec, static_cast<uint8_t*>(workspace), n_front,
                        static_cast<cudaStream_t>(stream)));
  return GS_OK;
}

extern "C" int gs_front5_pass2(int64_t n_rec, const int32_t* grid_len, const double* cost1,
                               int32_t k0_begin, int32_t k0_end, void* workspace, size_t workspace_bytes,
                               unsigned long long* out_index, double* out_cost, uint32_t* out_counts,
                               unsigned long long* out_n, int64_t out_cap, void* stream) {
  GS_REQUIRE(grid_len && cost1 && out_index && out_cost && out_counts && out_n && out_cap >= 0);
  if (!f5_supported(n_rec, grid_len)) return GS_EUNSUPPORTED;
  GS_REQUIRE(0 <= k0_begin && k0_begin <= k0_end && k0_end <= grid_len[0]);
  if (!workspace || workspace_bytes < f5_layout(grid_len, n_rec).bytes) return GS_EWORKSPACE;
  GS_CUDA_TRY(f5_pass2(grid_len, n_rec, cost1, static_cast<uint8_t*>(workspace), k0_begin, k0_end, out_index,
                       out_cost, out_counts, out_n, out_cap, static_cast<cudaStream_t>(stream)));
  return GS_OK;
}
