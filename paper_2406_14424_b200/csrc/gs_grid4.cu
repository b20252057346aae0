// gs_grid4.cu — grid sweep, four-model fast path (the headline workload:
// BASELINE configs[1], a 4-stage cascade over 1M records).
//
// Same algorithm and outputs as the general path in gs_sweep.cu (dominance
// counting over the bins b_j of the threshold grids, scored exactly like
// _evaluate_numba, /root/reference/pkg/src/gearserve/kernels.py:39-62), laid
// out so a whole sweep is three launches and every config is written by the
// kernel that finishes its table slab:
//
//   g4_hist      one pass over the records.  Per record ONE packed 64-bit
//                reduction into the main table H[b0][b1][b2] = {cnt, c3, c2}
//                (21-bit fields: exact for n_rec < 2^21, no carry possible,
//                so no overflow check or fallback pass) and one into the
//                small table H2[b0][b1] = {c1, c0} (32-bit fields).  A correct
//                count c_j is only ever read where the dims after j are at
//                "any", so c1 and c0 need only (b0, b1).
//   g4_prefix0   inclusive prefix of H and H2 along b0 (strided dim): thread
//                per (column, row segment), all loads of a segment in flight,
//                segment carries through shared memory; re-zeroes H / H2.
//   g4_eval      one CTA per (b0 slab k0, column part): the slab arrives by
//                one TMA bulk copy, is row-prefixed along b2 in shared memory
//                (a warp per row) and column-walked along b1 (thread per
//                (b2 column, row segment)).  Each position (k1, k2) of slab k0
//                is the table cell of the full cascade's config (k0, k1, k2);
//                the same walk also scores every other structure that starts
//                with model 0 at threshold k0 (their cells are the slab's
//                last row / last column), and the "any" slab k0 = g0 scores
//                every structure without model 0.  No face table, no second
//                eval launch; the outputs of a slab are contiguous runs.
//
// Channels at a position (p0, p1, p2), "g" meaning any:
//   cnt(p)  records with b0 <= p0, b1 <= p1, b2 <= p2
//   C3, C2  the same restricted to model 3 / model 2 correct
//   C1(p0, p1) = C1 at (p0, p1, g2),  C0(p0) = C0 at (p0, g1, g2)
// Full cascade (k0, k1, k2):
//   reach = n, cnt(k0,g,g), cnt(k0,k1,g), cnt(k0,k1,k2)
//   correct = C0(g) - C0(k0) + C1(k0,g) - C1(k0,k1)
//             + C2(k0,k1,g) - C2(k0,k1,k2) + C3(k0,k1,k2)
// and likewise for the shorter structures.
#include <algorithm>
#include <atomic>

#include "gs_grid4.cuh"
#include "gs_grid_lut.cuh"

namespace gs {
namespace {

constexpr uint64_t kF21 = (1ull << 21) - 1;
constexpr int kHist4Threads = 1024;
constexpr int kHist4Unroll = 4;

__device__ __forceinline__ void red_add_u64(unsigned long long* addr, unsigned long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(addr), "l"(v) : "memory");
}

// ------------------------------------------------------------------ hist --
struct G4HistArgs {
  const double* cert;
  const uint8_t* corr;
  int32_t n_rec;
  int32_t vec_ok;
  const double* grids;
  int32_t goff[GS_MAX_MODELS];
  int32_t glen[GS_MAX_MODELS];
  int32_t n_grid;  // doubles of grids 0..2
  int32_t d1, d2p, d1p;
  unsigned long long* H;   // [d0][d1][d2p] {cnt, c3, c2}
  unsigned long long* H2;  // [d0][d1p] {c1, c0}
};

struct Rec4 {
  double x0, x1, x2;
  uint32_t k;  // correct bytes of models 0..3
};

__device__ __forceinline__ Rec4 load_rec4(const G4HistArgs& a, int r) {
  Rec4 v;
  const double* row = a.cert + (int64_t)r * 4;
  if (a.vec_ok) {
    const double2 p = __ldg(reinterpret_cast<const double2*>(row));
    v.x0 = p.x;
    v.x1 = p.y;
    v.x2 = __ldg(row + 2);
    v.k = __ldg(reinterpret_cast<const uint32_t*>(a.corr) + r);
  } else {
    v.x0 = __ldg(row);
    v.x1 = __ldg(row + 1);
    v.x2 = __ldg(row + 2);
    const uint8_t* c = a.corr + (int64_t)r * 4;
    v.k = (uint32_t)__ldg(c) | ((uint32_t)__ldg(c + 1) << 8) | ((uint32_t)__ldg(c + 2) << 16) |
          ((uint32_t)__ldg(c + 3) << 24);
  }
  return v;
}

__global__ void __launch_bounds__(kHist4Threads, 1) g4_hist_kernel(const __grid_constant__ G4HistArgs a) {
  extern __shared__ __align__(16) double s_grid[];
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(s_grid + a.n_grid);
  __shared__ double s_par[3 * GS_MAX_MODELS];
  const int stride = gridDim.x * kHist4Threads;
  int r0 = blockIdx.x * kHist4Threads + threadIdx.x;
  // the first batch of records is in flight while the bin tables are built
  Rec4 v[kHist4Unroll];
#pragma unroll
  for (int u = 0; u < kHist4Unroll; ++u) {
    const int r = r0 + u * stride;
    if (r < a.n_rec) v[u] = load_rec4(a, r);
  }
  const BinTables bt =
      build_bin_tables<kHist4Threads>(a.grids, a.goff, a.glen, 3, a.n_grid, s_grid, s_lut, s_par);
  const int d1 = a.d1, d2p = a.d2p, d1p = a.d1p;
  while (r0 < a.n_rec) {
#pragma unroll
    for (int u = 0; u < kHist4Unroll; ++u) {
      if (r0 + u * stride >= a.n_rec) break;
      const int b0 = bt.bin(0, v[u].x0);
      const int b1 = bt.bin(1, v[u].x1);
      const int b2 = bt.bin(2, v[u].x2);
      const uint32_t k = v[u].k;
      const unsigned long long k0 = (k & 0xffu) != 0, k1 = (k & 0xff00u) != 0;
      const unsigned long long k2 = (k & 0xff0000u) != 0, k3 = (k & 0xff000000u) != 0;
      const int row = b0 * d1 + b1;
      red_add_u64(a.H + (int64_t)row * d2p + b2, 1ull | (k3 << 21) | (k2 << 42));
      if (k0 | k1) red_add_u64(a.H2 + b0 * d1p + b1, k1 | (k0 << 32));
    }
    r0 += kHist4Unroll * stride;
#pragma unroll
    for (int u = 0; u < kHist4Unroll; ++u) {
      const int r = r0 + u * stride;
      if (r < a.n_rec) v[u] = load_rec4(a, r);
    }
  }
}

// --------------------------------------------------------------- prefix0 --
constexpr int kPre4Threads = 256;
constexpr int kPre4MaxSeg = 16;  // rows per thread

struct G4PrefixArgs {
  unsigned long long* H;   // [d0][cols]
  unsigned long long* S;
  unsigned long long* H2;  // [d0][cols2]
  unsigned long long* S2;
  int32_t d0, cols, cols2;
  int32_t nseg, seg_len, cpc;  // segments per column, rows per segment, columns per CTA
};

__global__ void __launch_bounds__(kPre4Threads) g4_prefix0_kernel(const __grid_constant__ G4PrefixArgs a) {
  __shared__ unsigned long long s_tot[kPre4Threads];
  const int cl = threadIdx.x % a.cpc, seg = threadIdx.x / a.cpc;
  const int c = blockIdx.x * a.cpc + cl;
  const bool main = c < a.cols;
  const bool live = c < a.cols + a.cols2 && seg < a.nseg;
  unsigned long long* src = main ? a.H + c : a.H2 + (c - a.cols);
  unsigned long long* dst = main ? a.S + c : a.S2 + (c - a.cols);
  const uint32_t pitch = main ? a.cols : a.cols2;
  const int r0 = seg * a.seg_len;
  const int len = live ? max(0, min(a.seg_len, a.d0 - r0)) : 0;
  src += (size_t)r0 * pitch;
  dst += (size_t)r0 * pitch;
  unsigned long long v[kPre4MaxSeg];
  unsigned long long sum = 0;
#pragma unroll
  for (int i = 0; i < kPre4MaxSeg; ++i) v[i] = i < len ? src[i * pitch] : 0ull;
#pragma unroll
  for (int i = 0; i < kPre4MaxSeg; ++i) sum += v[i];
  s_tot[threadIdx.x] = sum;
  __syncthreads();
  unsigned long long run = 0;
  for (int s = 0; s < seg; ++s) run += s_tot[s * a.cpc + cl];
#pragma unroll
  for (int i = 0; i < kPre4MaxSeg; ++i) {
    if (i < len) {
      run += v[i];
      dst[i * pitch] = run;
      src[i * pitch] = 0ull;  // the next build starts from zero
    }
  }
}

// ------------------------------------------------------------------ eval --
constexpr int kEval4Threads = 512;
constexpr int kEval4MaxRowCells = 8;  // cells per lane in the row prefix (d2 <= 256)

struct G4EvalArgs {
  int32_t d0, d1, d2, d2p, d1p;
  int32_t parts, width, nseg, seg_len;  // column parts per slab, columns per part, row segments
  int64_t sb[16];                       // first config of the structure with model mask m
  int64_t cfg_begin, cfg_count;
  int64_t n_rec;
  double rcp_n;
  const double* cost1;
  const unsigned long long* S;   // b0-prefixed main table
  const unsigned long long* S2;  // b0-prefixed {c1, c0}
  double* acc;
  double* cost;
  double* frac;
  uint32_t* n_correct;
};

struct Cell3 {
  uint32_t cnt, c3, c2;
};
__device__ __forceinline__ Cell3 unpack3(unsigned long long v) {
  return {(uint32_t)(v & kF21), (uint32_t)((v >> 21) & kF21), (uint32_t)(v >> 42)};
}

// One config's outputs: frac row [1, f[0..K-2], 0 pad], mean built stage by
// stage in the reference's order (src/kernels.py:57-60), acc = correct / n.
template <int K>
__device__ __forceinline__ void put4(const G4EvalArgs& a, int64_t cfg, const uint32_t* reach,
                                     const double* cst, uint32_t correct, double n, double rcp,
                                     double one) {
  const int64_t i = cfg - a.cfg_begin;
  if (i < 0 || i >= a.cfg_count) return;
  double fr[4] = {one, 0.0, 0.0, 0.0};
  double mean = dadd(0.0, dmul(one, cst[0]));
#pragma unroll
  for (int t = 1; t < K; ++t) {
    fr[t] = div_count((double)reach[t - 1], n, rcp);
    mean = dadd(mean, dmul(fr[t], cst[t]));
  }
  if (a.frac) {
    double2* row = reinterpret_cast<double2*>(a.frac + i * 4);
    row[0] = make_double2(fr[0], fr[1]);
    row[1] = make_double2(fr[2], fr[3]);
  }
  if (a.cost) a.cost[i] = mean;
  if (a.acc) a.acc[i] = div_count((double)correct, n, rcp);
  if (a.n_correct) a.n_correct[i] = correct;
}

__global__ void __launch_bounds__(kEval4Threads, 2) g4_eval_kernel(const __grid_constant__ G4EvalArgs a) {
  extern __shared__ __align__(16) unsigned long long s_slab[];  // [d1][d2p]
  __shared__ __align__(8) uint64_t bar;
  __shared__ unsigned long long s_colg[1024];  // prefix along b1 of column g2 (= row totals)
  __shared__ uint32_t s_c1[1024];              // C1(k0, b1) prefix along b1
  __shared__ unsigned long long s_seg[kEval4Threads];
  __shared__ uint32_t s_c0[2];                 // C0(k0), C0(g0)
  const int d0 = a.d0, d1 = a.d1, d2 = a.d2, d2p = a.d2p;
  const int g0 = d0 - 1, g1 = d1 - 1, g2 = d2 - 1;
  const int k0 = blockIdx.x / a.parts, part = blockIdx.x - k0 * a.parts;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kEval4Threads / 32;
  const bool any0 = k0 == g0;  // the "any" slab: structures without model 0
  // skip a slab none of whose configs is in the requested range: a slab
  // k0 < g0 scores structures (0,1) .. (0,1,2,3), the first starting at
  // sb[3] + k0 and the last ending at sb[15] + (k0 + 1) g1 g2; the any slab
  // scores the singletons (from config 0) through (1,2,3)
  {
    const int64_t lo = any0 ? 0 : a.sb[3] + k0;
    const int64_t hi = any0 ? a.sb[14] + (int64_t)g1 * g2 : a.sb[15] + (int64_t)(k0 + 1) * g1 * g2;
    if (hi <= a.cfg_begin || lo >= a.cfg_begin + a.cfg_count) return;
  }
  const uint32_t slab_bytes = (uint32_t)((int64_t)d1 * d2p * 8);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar, slab_bytes);
    const unsigned long long* src = a.S + (int64_t)k0 * d1 * d2p;
    constexpr uint32_t kChunk = 32768;
    for (uint32_t off = 0; off < slab_bytes; off += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_slab) + off, reinterpret_cast<const uint8_t*>(src) + off,
               min(kChunk, slab_bytes - off), &bar);
  }
  // side channels while the slab is in flight: warp 1 -> C1 prefix and C0(k0),
  // warp 2 -> C0(g0)
  if (warp == 1 || warp == 2) {
    const unsigned long long* row = a.S2 + (int64_t)(warp == 1 ? k0 : g0) * a.d1p;
    uint32_t carry = 0, c0 = 0;
    for (int b = 0; b < d1; b += 32) {
      const int b1 = b + lane;
      const unsigned long long w = b1 < d1 ? row[b1] : 0ull;
      c0 += (uint32_t)(w >> 32);
      if (warp == 1) {
        uint32_t x = (uint32_t)w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        x += carry;
        if (b1 < d1) s_c1[b1] = x;
        carry = __shfl_sync(0xffffffffu, x, 31);
      }
    }
    c0 = warp_sum(c0);
    if (lane == 0) s_c0[warp - 1] = c0;
  }
  mbar_wait(&bar, 0);
  // row prefix along b2, a warp per row, J consecutive cells per lane
  {
    const int J = (d2 + 31) / 32;
    for (int r = warp; r < d1; r += nwarps) {
      unsigned long long* row = s_slab + (int64_t)r * d2p;
      unsigned long long e[kEval4MaxRowCells];
      unsigned long long tot = 0;
#pragma unroll
      for (int j = 0; j < kEval4MaxRowCells; ++j) {
        const int c = lane * J + j;
        e[j] = (j < J && c < d2) ? row[c] : 0ull;
        tot += e[j];
        e[j] = tot;
      }
      unsigned long long incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned long long excl = incl - tot;
#pragma unroll
      for (int j = 0; j < kEval4MaxRowCells; ++j) {
        const int c = lane * J + j;
        if (j < J && c < d2) row[c] = e[j] + excl;
      }
    }
  }
  __syncthreads();
  // column g2 (row totals) prefix along b1 -> s_colg (warp 0); segment sums
  // of the walked columns (every thread)
  const int kc = tid % a.width, seg = tid / a.width;
  const int k2 = part * a.width + kc;
  const bool walker = kc < a.width && k2 < d2 && seg < a.nseg;
  const int r_lo = seg * a.seg_len, r_hi = min(d1, r_lo + a.seg_len);
  if (warp == 0) {
    unsigned long long carry = 0;
    for (int b = 0; b < d1; b += 32) {
      const int b1 = b + lane;
      unsigned long long x = b1 < d1 ? s_slab[(int64_t)b1 * d2p + g2] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      x += carry;
      if (b1 < d1) s_colg[b1] = x;
      carry = __shfl_sync(0xffffffffu, x, 31);
    }
  }
  unsigned long long ssum = 0;
  if (walker)
    for (int r = r_lo; r < r_hi; ++r) ssum += s_slab[(int64_t)r * d2p + k2];
  s_seg[tid] = ssum;
  __syncthreads();
  if (!walker) return;
  unsigned long long P = 0;
  for (int s = 0; s < seg; ++s) P += s_seg[s * a.width + kc];

  const double n = (double)a.n_rec, rcp = a.rcp_n;
  const double one = div_count(n, n, rcp);
  const double c0c = __ldg(a.cost1 + 0), c1c = __ldg(a.cost1 + 1), c2c = __ldg(a.cost1 + 2),
               c3c = __ldg(a.cost1 + 3);
  const Cell3 tot = unpack3(s_colg[g1]);
  const uint32_t C1g = s_c1[g1];
  if (!any0) {
    const uint32_t base0 = s_c0[1] - s_c0[0];  // model 0 completes b0 > k0
    for (int k1 = r_lo; k1 < r_hi; ++k1) {
      P += s_slab[(int64_t)k1 * d2p + k2];
      const Cell3 p = unpack3(P);
      if (k1 < g1) {
        const Cell3 rg = unpack3(s_colg[k1]);
        const uint32_t c01 = base0 + (C1g - s_c1[k1]);
        if (k2 < g2) {  // (0,1,2,3)
          const uint32_t reach[3] = {tot.cnt, rg.cnt, p.cnt};
          const double cst[4] = {c0c, c1c, c2c, c3c};
          put4<4>(a, a.sb[15] + ((int64_t)k0 * g1 + k1) * g2 + k2, reach, cst,
                  c01 + (rg.c2 - p.c2) + p.c3, n, rcp, one);
        } else {  // (0,1,2) and (0,1,3) at (k0, k1)
          const uint32_t reach[2] = {tot.cnt, rg.cnt};
          const double cst2[3] = {c0c, c1c, c2c}, cst3[3] = {c0c, c1c, c3c};
          put4<3>(a, a.sb[7] + (int64_t)k0 * g1 + k1, reach, cst2, c01 + rg.c2, n, rcp, one);
          put4<3>(a, a.sb[11] + (int64_t)k0 * g1 + k1, reach, cst3, c01 + rg.c3, n, rcp, one);
        }
      } else if (k2 < g2) {  // (0,2,3) at (k0, k2)
        const uint32_t reach[2] = {tot.cnt, p.cnt};
        const double cst[3] = {c0c, c2c, c3c};
        put4<3>(a, a.sb[13] + (int64_t)k0 * g2 + k2, reach, cst,
                base0 + (tot.c2 - p.c2) + p.c3, n, rcp, one);
      } else {  // (0,1), (0,2), (0,3) at k0
        const uint32_t reach[1] = {tot.cnt};
        const double cA[2] = {c0c, c1c}, cB[2] = {c0c, c2c}, cC[2] = {c0c, c3c};
        put4<2>(a, a.sb[3] + k0, reach, cA, base0 + C1g, n, rcp, one);
        put4<2>(a, a.sb[5] + k0, reach, cB, base0 + tot.c2, n, rcp, one);
        put4<2>(a, a.sb[9] + k0, reach, cC, base0 + tot.c3, n, rcp, one);
      }
    }
  } else {
    for (int k1 = r_lo; k1 < r_hi; ++k1) {
      P += s_slab[(int64_t)k1 * d2p + k2];
      const Cell3 p = unpack3(P);
      if (k1 < g1) {
        const Cell3 rg = unpack3(s_colg[k1]);
        const uint32_t c1 = C1g - s_c1[k1];  // model 1 completes b1 > k1
        if (k2 < g2) {  // (1,2,3) at (k1, k2)
          const uint32_t reach[2] = {rg.cnt, p.cnt};
          const double cst[3] = {c1c, c2c, c3c};
          put4<3>(a, a.sb[14] + (int64_t)k1 * g2 + k2, reach, cst, c1 + (rg.c2 - p.c2) + p.c3, n,
                  rcp, one);
        } else {  // (1,2), (1,3) at k1
          const uint32_t reach[1] = {rg.cnt};
          const double cA[2] = {c1c, c2c}, cB[2] = {c1c, c3c};
          put4<2>(a, a.sb[6] + k1, reach, cA, c1 + rg.c2, n, rcp, one);
          put4<2>(a, a.sb[10] + k1, reach, cB, c1 + rg.c3, n, rcp, one);
        }
      } else if (k2 < g2) {  // (2,3) at k2
        const uint32_t reach[1] = {p.cnt};
        const double cst[2] = {c2c, c3c};
        put4<2>(a, a.sb[12] + k2, reach, cst, (tot.c2 - p.c2) + p.c3, n, rcp, one);
      } else {  // singletons
        const uint32_t* none = nullptr;
        const double cA[1] = {c0c}, cB[1] = {c1c}, cC[1] = {c2c}, cD[1] = {c3c};
        put4<1>(a, a.sb[1], none, cA, s_c0[1], n, rcp, one);
        put4<1>(a, a.sb[2], none, cB, C1g, n, rcp, one);
        put4<1>(a, a.sb[4], none, cC, tot.c2, n, rcp, one);
        put4<1>(a, a.sb[8], none, cD, tot.c3, n, rcp, one);
      }
    }
  }
}

template <typename Kernel>
cudaError_t ensure_smem4(Kernel k, std::atomic<int>& done, size_t bytes) {
  if ((int)bytes <= done.load(std::memory_order_acquire)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.store((int)bytes, std::memory_order_release);
  return e;
}

}  // namespace

// ------------------------------------------------------------ host side --
bool grid4_supported(int64_t n_rec, int32_t M, const int32_t* glen) {
  if (M != 4 || n_rec < 1 || n_rec >= kGrid4MaxRec) return false;
  const int64_t d0 = glen[0] + 1, d1 = glen[1] + 1, d2 = glen[2] + 1;
  const int64_t d2p = (d2 + 1) & ~1ll;
  return d0 <= kPre4Threads && d1 <= 1024 && d2 <= 32 * kEval4MaxRowCells &&
         d1 * d2p * 8 <= kGrid4SlabMax;
}

Grid4Layout grid4_layout(const int32_t* glen) {
  Grid4Layout L{};
  L.d0 = glen[0] + 1;
  L.d1 = glen[1] + 1;
  L.d2 = glen[2] + 1;
  L.d2p = (L.d2 + 1) & ~1;
  L.d1p = (L.d1 + 1) & ~1;
  const size_t bH = round_up((size_t)L.d0 * L.d1 * L.d2p * 8, 256);
  const size_t bH2 = round_up((size_t)L.d0 * L.d1p * 8, 256);
  L.offH = 0;
  L.offH2 = bH;
  L.offS = bH + bH2;
  L.offS2 = 2 * bH + bH2;
  L.bytes = 2 * bH + 2 * bH2;
  return L;
}

cudaError_t grid4_build(const double* cert, const uint8_t* corr, int64_t n_rec, const double* grids,
                        const int32_t* glen, uint8_t* ws, bool dirty, cudaStream_t st) {
  const Grid4Layout L = grid4_layout(glen);
  auto* H = reinterpret_cast<unsigned long long*>(ws + L.offH);
  auto* H2 = reinterpret_cast<unsigned long long*>(ws + L.offH2);
  if (dirty) {
    cudaError_t e = cudaMemsetAsync(ws, 0, L.offS, st);  // H and H2
    if (e != cudaSuccess) return e;
  }
  G4HistArgs h{};
  h.cert = cert;
  h.corr = corr;
  h.n_rec = (int32_t)n_rec;
  h.vec_ok = aligned16(cert) && ((reinterpret_cast<uintptr_t>(corr) & 3u) == 0);
  h.grids = grids;
  int off = 0;
  for (int j = 0; j < 3; ++j) {
    h.goff[j] = off;
    h.glen[j] = glen[j];
    off += glen[j];
  }
  h.n_grid = off;
  h.d1 = L.d1;
  h.d2p = L.d2p;
  h.d1p = L.d1p;
  h.H = H;
  h.H2 = H2;
  const size_t smem = (size_t)h.n_grid * sizeof(double) + 3 * kLutBuckets * sizeof(uint32_t);
  static std::atomic<int> smem_set{0};
  cudaError_t e = ensure_smem4(g4_hist_kernel, smem_set, smem);
  if (e != cudaSuccess) return e;
  int64_t blocks = (n_rec + kHist4Threads * kHist4Unroll - 1) / (kHist4Threads * kHist4Unroll);
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, sm_count()));
  g4_hist_kernel<<<(unsigned)blocks, kHist4Threads, smem, st>>>(h);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  G4PrefixArgs p{};
  p.H = H;
  p.S = reinterpret_cast<unsigned long long*>(ws + L.offS);
  p.H2 = H2;
  p.S2 = reinterpret_cast<unsigned long long*>(ws + L.offS2);
  p.d0 = L.d0;
  p.cols = L.d1 * L.d2p;
  p.cols2 = L.d1p;
  int nseg = 1;
  while (nseg * kPre4MaxSeg < L.d0) nseg *= 2;
  p.nseg = nseg;
  p.seg_len = (L.d0 + nseg - 1) / nseg;
  p.cpc = kPre4Threads / nseg;
  const int64_t cols = (int64_t)p.cols + p.cols2;
  g4_prefix0_kernel<<<(unsigned)((cols + p.cpc - 1) / p.cpc), kPre4Threads, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t grid4_eval(int64_t n_rec, const int32_t* glen, const int64_t* struct_begin,
                       const uint32_t* struct_mask, int n_struct, const double* cost1,
                       int64_t cfg_begin, int64_t cfg_count, double* acc, double* cost,
                       double* frac, uint32_t* n_correct, const uint8_t* ws, cudaStream_t st) {
  const Grid4Layout L = grid4_layout(glen);
  G4EvalArgs a{};
  a.d0 = L.d0;
  a.d1 = L.d1;
  a.d2 = L.d2;
  a.d2p = L.d2p;
  a.d1p = L.d1p;
  for (int s = 0; s < n_struct; ++s) a.sb[struct_mask[s] & 15u] = struct_begin[s];
  a.cfg_begin = cfg_begin;
  a.cfg_count = cfg_count;
  a.n_rec = n_rec;
  a.rcp_n = 1.0 / (double)n_rec;
  a.cost1 = cost1;
  a.S = reinterpret_cast<const unsigned long long*>(ws + L.offS);
  a.S2 = reinterpret_cast<const unsigned long long*>(ws + L.offS2);
  a.acc = acc;
  a.cost = cost;
  a.frac = frac;
  a.n_correct = n_correct;
  // column parts so that every slab's walk spreads over >= 2 CTAs when the
  // slabs alone cannot fill the GPU; row segments fill the CTA
  a.parts = (L.d0 < 2 * sm_count() && L.d2 >= 16) ? 2 : 1;
  a.width = (L.d2 + a.parts - 1) / a.parts;
  a.nseg = std::max(1, std::min(kEval4Threads / a.width, L.d1));
  a.seg_len = (L.d1 + a.nseg - 1) / a.nseg;
  a.nseg = (L.d1 + a.seg_len - 1) / a.seg_len;
  const size_t smem = (size_t)L.d1 * L.d2p * 8;
  static std::atomic<int> smem_set{0};
  cudaError_t e = ensure_smem4(g4_eval_kernel, smem_set, (size_t)kGrid4SlabMax);
  if (e != cudaSuccess) return e;
  g4_eval_kernel<<<(unsigned)(L.d0 * a.parts), kEval4Threads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace gs
