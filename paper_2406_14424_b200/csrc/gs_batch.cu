// gs_batch.cu — many small three-model sweeps in one launch (SURVEY §8d,
// config 1: the reference's CPU default, 10k records x 3 models x 100-level
// grids, C = 10,303 configs, is launch-bound on its own: ~0.7 MB of
// traffic; stacking R validation sets per launch amortises the launch).
//
// Same algorithm and outputs as the grid path (gs_sweep.cu; dominance
// counting over the bins b_j = #{g in G_j : g <= cert}, scored like
// _evaluate_numba, /root/reference/pkg/src/gearserve/kernels.py:39-62), for
// M = 3: the table is two-dimensional over (b0, b1) and fits one CTA's
// shared memory, so a CTA does a whole sweep: bins by binary search in the
// set's grids, a shared-memory histogram of {records, c0, c1, c2}, the 2-D
// inclusive prefix, and every config of the enumeration (structures by size,
// then lexicographic; inside a structure the threshold tuple lexicographic).
#include <atomic>
#include <climits>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kBatchThreads = 1024;
constexpr int kBatchMaxCells = 12800;  // (g0 + 1)(g1 + 1) uint4 cells: 200 KB

struct BatchArgs {
  const double* cert;  // [sets][n][3]
  const uint8_t* corr; // [sets][n][3]
  int64_t n_rec;
  const double* grids;  // [sets][g0 + g1 + g2]
  int32_t g0, g1, g2;
  double rcp_n;
  const double* cost1;  // [3]
  int64_t n_cfg;
  double* acc;   // [sets][n_cfg]
  double* cost;  // [sets][n_cfg]
  double* frac;  // [sets][n_cfg][3]
};

// #{g[i] <= x} for strictly increasing g (n >= 1), branch-free
__device__ __forceinline__ int count_le(const double* g, int n, double x) {
  int base = 0, len = n;
  while (len > 1) {
    const int half = len >> 1;
    base = (g[base + half - 1] <= x) ? base + half : base;
    len -= half;
  }
  return base + (g[base] <= x ? 1 : 0);
}

__device__ __forceinline__ uint4 add4u(uint4 a, uint4 b) {
  return make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ uint4 shfl_up4u(uint4 v, int o) {
  return make_uint4(__shfl_up_sync(0xffffffffu, v.x, o), __shfl_up_sync(0xffffffffu, v.y, o),
                    __shfl_up_sync(0xffffffffu, v.z, o), __shfl_up_sync(0xffffffffu, v.w, o));
}

// A table cell: {records, c0, c1, c2} as four 32-bit counts, or (PACKED,
// fewer than 2^16 records: no field of any prefix sum can carry) as two
// words {records | c0 << 16, c1 | c2 << 16}: half the shared memory (two
// CTAs per SM) and half the atomics.
template <bool PACKED>
struct BCell;
template <>
struct BCell<false> {
  using T = uint4;
  __device__ static T zero() { return make_uint4(0, 0, 0, 0); }
  __device__ static T add(T a, T b) { return add4u(a, b); }
  __device__ static T shfl_up(T v, int o) { return shfl_up4u(v, o); }
  __device__ static T shfl(T v, int l) {
    return make_uint4(__shfl_sync(0xffffffffu, v.x, l), __shfl_sync(0xffffffffu, v.y, l),
                      __shfl_sync(0xffffffffu, v.z, l), __shfl_sync(0xffffffffu, v.w, l));
  }
  __device__ static void count(T* tab, int cell, bool k0, bool k1, bool k2) {
    uint32_t* w = reinterpret_cast<uint32_t*>(tab + cell);
    atomicAdd(w, 1u);
    if (k0) atomicAdd(w + 1, 1u);
    if (k1) atomicAdd(w + 2, 1u);
    if (k2) atomicAdd(w + 3, 1u);
  }
  __device__ static uint4 unpack(T v) { return v; }
};
template <>
struct BCell<true> {
  using T = uint2;
  __device__ static T zero() { return make_uint2(0, 0); }
  __device__ static T add(T a, T b) { return make_uint2(a.x + b.x, a.y + b.y); }
  __device__ static T shfl_up(T v, int o) {
    return make_uint2(__shfl_up_sync(0xffffffffu, v.x, o), __shfl_up_sync(0xffffffffu, v.y, o));
  }
  __device__ static T shfl(T v, int l) {
    return make_uint2(__shfl_sync(0xffffffffu, v.x, l), __shfl_sync(0xffffffffu, v.y, l));
  }
  __device__ static void count(T* tab, int cell, bool k0, bool k1, bool k2) {
    uint32_t* w = reinterpret_cast<uint32_t*>(tab + cell);
    atomicAdd(w, 1u | (k0 ? 1u << 16 : 0u));
    const uint32_t hi = (k1 ? 1u : 0u) | (k2 ? 1u << 16 : 0u);
    if (hi) atomicAdd(w + 1, hi);
  }
  __device__ static uint4 unpack(T v) {
    return make_uint4(v.x & 0xffffu, v.x >> 16, v.y & 0xffffu, v.y >> 16);
  }
};

template <bool PACKED>
__global__ void __launch_bounds__(kBatchThreads, PACKED ? 2 : 1) batch3_kernel(const __grid_constant__ BatchArgs a) {
  using CT = BCell<PACKED>;
  using Cell = typename CT::T;
  extern __shared__ __align__(16) uint8_t s_raw[];
  Cell* s_tab = reinterpret_cast<Cell*>(s_raw);  // [d0][d1], then grids
  const int64_t set = blockIdx.x;
  const int g0 = a.g0, g1 = a.g1, g2 = a.g2, d0 = g0 + 1, d1 = g1 + 1;
  const int cells = d0 * d1;
  double* s_grid = reinterpret_cast<double*>(s_tab + cells);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = kBatchThreads / 32;
  const double* grid = a.grids + set * (int64_t)(g0 + g1 + g2);
  for (int i = tid; i < g0 + g1; i += kBatchThreads) s_grid[i] = __ldg(grid + i);
  for (int i = tid; i < cells; i += kBatchThreads) s_tab[i] = CT::zero();
  __syncthreads();
  // histogram over (b0, b1): model 2 never forwards, so its bin is not needed
  const double* cert = a.cert + set * a.n_rec * 3;
  const uint8_t* corr = a.corr + set * a.n_rec * 3;
  for (int64_t r = tid; r < a.n_rec; r += kBatchThreads) {
    const double x0 = __ldg(cert + 3 * r), x1 = __ldg(cert + 3 * r + 1);
    const uint8_t k0 = __ldg(corr + 3 * r), k1 = __ldg(corr + 3 * r + 1), k2 = __ldg(corr + 3 * r + 2);
    const int cell = count_le(s_grid, g0, x0) * d1 + count_le(s_grid + g0, g1, x1);
    CT::count(s_tab, cell, k0 != 0, k1 != 0, k2 != 0);
  }
  __syncthreads();
  // inclusive prefix along b1 (a warp per row) then along b0 (a warp per column)
  for (int row = warp; row < d0; row += nwarps) {
    Cell carry = CT::zero();
    for (int b = 0; b < d1; b += 32) {
      const int c = b + lane;
      Cell v = c < d1 ? s_tab[row * d1 + c] : CT::zero();
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const Cell y = CT::shfl_up(v, o);
        if (lane >= o) v = CT::add(v, y);
      }
      v = CT::add(v, carry);
      if (c < d1) s_tab[row * d1 + c] = v;
      carry = CT::shfl(v, 31);
    }
  }
  __syncthreads();
  for (int col = warp; col < d1; col += nwarps) {
    Cell carry = CT::zero();
    for (int b = 0; b < d0; b += 32) {
      const int r = b + lane;
      Cell v = r < d0 ? s_tab[r * d1 + col] : CT::zero();
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const Cell y = CT::shfl_up(v, o);
        if (lane >= o) v = CT::add(v, y);
      }
      v = CT::add(v, carry);
      if (r < d0) s_tab[r * d1 + col] = v;
      carry = CT::shfl(v, 31);
    }
  }
  __syncthreads();
  // configs: (0), (1), (2), (0,1) x g0, (0,2) x g0, (1,2) x g1, (0,1,2) x g0 g1
  const double n = (double)a.n_rec, rcp = a.rcp_n;
  const double one = div_count(n, n, rcp);
  const double c0c = __ldg(a.cost1), c1c = __ldg(a.cost1 + 1), c2c = __ldg(a.cost1 + 2);
  const uint4 gg = CT::unpack(s_tab[g0 * d1 + g1]);  // (any, any): all records
  double* acc = a.acc + set * a.n_cfg;
  double* cost = a.cost + set * a.n_cfg;
  double* frac = a.frac + set * a.n_cfg * 3;
  for (int64_t c = tid; c < a.n_cfg; c += kBatchThreads) {
    double f1 = 0.0, f2 = 0.0, mean;
    uint32_t correct;
    if (c < 3) {  // singletons
      const double cc = c == 0 ? c0c : (c == 1 ? c1c : c2c);
      mean = dadd(0.0, dmul(one, cc));
      correct = c == 0 ? gg.y : (c == 1 ? gg.z : gg.w);
    } else if (c < 3 + 2 * (int64_t)g0) {  // (0,1) and (0,2) at k0
      const bool second = c >= 3 + g0;
      const int k0 = (int)(c - 3 - (second ? g0 : 0));
      const uint4 p = CT::unpack(s_tab[k0 * d1 + g1]);  // (k0, any)
      f1 = div_count((double)p.x, n, rcp);
      mean = dadd(dadd(0.0, dmul(one, c0c)), dmul(f1, second ? c2c : c1c));
      correct = (gg.y - p.y) + (second ? p.w : p.z);
    } else if (c < 3 + 2 * (int64_t)g0 + g1) {  // (1,2) at k1
      const int k1 = (int)(c - 3 - 2 * (int64_t)g0);
      const uint4 p = CT::unpack(s_tab[g0 * d1 + k1]);  // (any, k1)
      f1 = div_count((double)p.x, n, rcp);
      mean = dadd(dadd(0.0, dmul(one, c1c)), dmul(f1, c2c));
      correct = (gg.z - p.z) + p.w;
    } else {  // (0,1,2) at (k0, k1)
      const int64_t q = c - 3 - 2 * (int64_t)g0 - g1;
      const int k0 = (int)(q / g1), k1 = (int)(q - (int64_t)k0 * g1);
      const uint4 pa = CT::unpack(s_tab[k0 * d1 + g1]), pb = CT::unpack(s_tab[k0 * d1 + k1]);
      f1 = div_count((double)pa.x, n, rcp);
      f2 = div_count((double)pb.x, n, rcp);
      mean = dadd(dadd(dadd(0.0, dmul(one, c0c)), dmul(f1, c1c)), dmul(f2, c2c));
      correct = (gg.y - pa.y) + (pa.z - pb.z) + pb.w;
    }
    cost[c] = mean;
    acc[c] = div_count((double)correct, n, rcp);
    frac[3 * c] = one;
    frac[3 * c + 1] = f1;
    frac[3 * c + 2] = f2;
  }
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" int gs_grid_sweep_batched(const double* certainty, const uint8_t* correct,
                                     int64_t n_sets, int64_t n_rec, int32_t n_models,
                                     const double* grids, const int32_t* grid_len,
                                     const double* cost1, double* accuracy, double* mean_cost,
                                     double* forward_frac, void* stream) {
  GS_REQUIRE(certainty && correct && grids && grid_len && cost1 && accuracy && mean_cost &&
             forward_frac && n_sets >= 0 && n_rec >= 1);
  if (n_models != 3) return GS_EUNSUPPORTED;
  for (int j = 0; j < 3; ++j) GS_REQUIRE(grid_len[j] >= 1);
  const int g0 = grid_len[0], g1 = grid_len[1], g2 = grid_len[2];
  const int64_t cells = (int64_t)(g0 + 1) * (g1 + 1);
  if (cells > kBatchMaxCells || n_rec >= ((int64_t)1 << 31) || n_sets > INT32_MAX)
    return GS_EUNSUPPORTED;
  if (n_sets == 0) return GS_OK;
  BatchArgs a{};
  a.cert = certainty;
  a.corr = correct;
  a.n_rec = n_rec;
  a.grids = grids;
  a.g0 = g0;
  a.g1 = g1;
  a.g2 = g2;
  a.rcp_n = 1.0 / (double)n_rec;
  a.cost1 = cost1;
  a.n_cfg = 3 + 2 * (int64_t)g0 + g1 + (int64_t)g0 * g1;
  a.acc = accuracy;
  a.cost = mean_cost;
  a.frac = forward_frac;
  if (g0 + g1 > 2 * 1024) return GS_EUNSUPPORTED;
  const bool packed = n_rec < 65536;
  const size_t smem = (size_t)cells * (packed ? 8 : 16) + (size_t)(g0 + g1) * 8;
  static SmemAttr attr_wide, attr_packed;
  GS_CUDA_TRY(ensure_smem(batch3_kernel<false>, attr_wide, (size_t)(kBatchMaxCells * 16 + 2 * 1024 * 8)));
  GS_CUDA_TRY(ensure_smem(batch3_kernel<true>, attr_packed, (size_t)(kBatchMaxCells * 8 + 2 * 1024 * 8)));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (packed)
    batch3_kernel<true><<<(unsigned)n_sets, kBatchThreads, smem, st>>>(a);
  else
    batch3_kernel<false><<<(unsigned)n_sets, kBatchThreads, smem, st>>>(a);
  GS_LAUNCH_CHECK();
  return GS_OK;
}
