// gs_grid4.cu — grid sweep, four-model fast path (the headline workload:
// BASELINE configs[1], a 4-stage cascade over 1M records).
//
// Same algorithm and outputs as the general path in gs_sweep.cu (dominance
// counting over the bins b_j of the threshold grids, scored exactly like
// _evaluate_numba, /root/reference/pkg/src/gearserve/kernels.py:39-62), laid
// out as three launches.  A one-shot build (gs_grid_build):
//
//   g4_sort    one pass over the records (148 CTAs, a contiguous range each,
//              streamed through a cp.async shared-memory ring): bins by
//              per-CTA bucket tables, each record a 4-byte key {b0, b2, k1,
//              k2, k3, b1, k0}, counting-sorted by b1 in shared memory; one
//              bulk copy of the range's keys and its bucket offsets out.
//   g4_gather  one CTA per b1: the bucket's key segments of every range,
//              counted into the (b0, b2) plane in shared memory (16-bit
//              packed counters, 32-bit atomics), prefixed along b2 and b0 and
//              written as packed u64 {cnt, c3, c2} (21-bit fields, exact for
//              n_rec < 2^21) plus R1[b0][b1] (the c1 channel at b2 = any) and
//              the prefix P0 of model 0's correct counts per b0.
//
// The streamed build (gs_grid_accumulate / gs_grid_finish, and shapes the
// sorted plan does not fit) uses g4_hist (one red.global.add.v4.f32 of
// {1, k3, k2, k1} per record into H[b1][b0][b2]) and g4_plane (the same
// plane prefix from H, re-zeroing it).  Both leave the same S / R1 / P0.
//
//   g4_eval    one CTA per SM (four 256-thread groups); a unit is a block
//              of W columns (b2) of one b0 slab k0, stored contiguously in
//              S's blocked layout and staged by bulk copies; a column walk
//              along b1 finishes the prefix and scores each position
//              (k1, k2) as the full cascade's config (k0, k1, k2), with
//              row-shared terms (the stage-2 fraction, the partial mean cost,
//              the partial correct count) once per row.  Spare threads score
//              every structure that starts with model 0 at threshold k0
//              (their cells are the slab's last row / column), and the "any"
//              slab k0 = g0 scores every structure without model 0.
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

#include <cooperative_groups.h>

#include "gs_grid4.cuh"
#include "gs_grid_lut.cuh"

namespace gs {
namespace {

namespace cg = cooperative_groups;

// Phase stamps (GS_PHASE_TIMING builds only, tools/phase_probe.py): thread 0
// of each CTA records %globaltimer and clock64 at phase boundaries.
#ifdef GS_PHASE_TIMING
constexpr int kPhaseKernels = 3, kPhaseCtas = 1024, kPhaseSlots = 8;
__device__ unsigned long long g_phase[kPhaseKernels * kPhaseCtas * kPhaseSlots * 2];
__device__ __forceinline__ void phase(int kernel, int slot) {
  if (threadIdx.x == 0 && blockIdx.x < kPhaseCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const size_t i = ((size_t)(kernel * kPhaseCtas + blockIdx.x) * kPhaseSlots + slot) * 2;
    g_phase[i] = t;
    g_phase[i + 1] = clock64();
    if (slot == 0) {  // the CTA's SM in the last slot
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      const size_t j = ((size_t)(kernel * kPhaseCtas + blockIdx.x) * kPhaseSlots + kPhaseSlots - 1) * 2;
      g_phase[j + 1] = smid;
    }
  }
}
#else
__device__ __forceinline__ void phase(int, int) {}
#endif

constexpr uint64_t kF21 = (1ull << 21) - 1;

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// Programmatic dependent launch: the plane and eval kernels are launched
// with programmatic stream serialization, so their CTAs can be scheduled
// (and run their prologue: barrier init, zero buffers, range checks) while
// the previous kernel drains; griddepcontrol.wait then blocks until the
// previous grid has completed and its writes are visible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename Kernel, typename Args>
cudaError_t launch_pdl(Kernel k, unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       const Args& args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args);
}


// ------------------------------------------------------------------ hist --
constexpr int kHist4Threads = 1024;
constexpr int kHist4Unroll = 1;                          // records per thread per chunk
constexpr int kHist4Chunk = kHist4Threads * kHist4Unroll;  // records per chunk
constexpr int kMaxDim4 = 256;  // d0, d2 bound of this path

struct G4HistArgs {
  const double* cert;
  const uint8_t* corr;
  int32_t n_rec;
  int32_t vec_ok;
  const double* grids;
  int32_t glen[3];
  int32_t d0, hp;
  float* H;      // [d1][d0][hp] float4 {cnt, c3, c2, c1}
  uint32_t* G0;  // [d0] model-0 correct counts per b0
  uint32_t* counters;  // [0] chunks handed out, [1] CTAs done (both 0 between launches)
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

// Records are taken in chunks of kHist4Chunk: a CTA's first chunk is its
// block index (its loads go out before the bin tables are built), later ones
// come from a global counter, one chunk ahead, so CTAs on slower SMs simply
// take fewer chunks.  The last CTA to finish resets the counters.
__global__ void __launch_bounds__(kHist4Threads, 1) g4_hist_kernel(const __grid_constant__ G4HistArgs a) {
  extern __shared__ __align__(16) double s_grid[];  // grids 0..2, then the bucket tables
  __shared__ uint32_t s_c0[kMaxDim4];
  __shared__ int s_next[2];
  const int n_grid = a.glen[0] + a.glen[1] + a.glen[2];
  void* s_lut = s_grid + n_grid;  // [3][kLutBuckets] entries
  const int tid = threadIdx.x;
  phase(0, 0);
  // grid values first, then the first chunk's records: the records stream
  // in while the bin tables are built, and the grid loads are not queued
  // behind them
  constexpr int kGridRegs = 5;  // n_grid <= 5 * 1024 on this path
  double gv[kGridRegs];
#pragma unroll
  for (int q = 0; q < kGridRegs; ++q) {
    const int i = tid + q * kHist4Threads;
    gv[q] = i < n_grid ? __ldg(a.grids + i) : 0.0;
  }
  int c = blockIdx.x;
  Rec4 v[kHist4Unroll];
#pragma unroll
  for (int u = 0; u < kHist4Unroll; ++u) {
    const int r = c * kHist4Chunk + u * kHist4Threads + tid;
    if (r < a.n_rec) v[u] = load_rec4(a, r);
  }
  if (tid == 0) s_next[0] = gridDim.x + (int)atomicAdd(a.counters, 1u);
#pragma unroll
  for (int q = 0; q < kGridRegs; ++q) {
    const int i = tid + q * kHist4Threads;
    if (i < n_grid) s_grid[i] = gv[q];
  }
  for (int i = tid; i < a.d0; i += kHist4Threads) s_c0[i] = 0u;
  __syncthreads();
  const BinTables<3> bt = build_bin_tables<3, kHist4Threads>(a.glen, s_grid, s_lut);
  phase(0, 1);
  const int d0 = a.d0, hp = a.hp;
  int slot = 0;
  while (c * kHist4Chunk < a.n_rec) {
    const int cn = s_next[slot];
    Rec4 nv[kHist4Unroll];
#pragma unroll
    for (int u = 0; u < kHist4Unroll; ++u) {
      const int r = cn * kHist4Chunk + u * kHist4Threads + tid;
      if (r < a.n_rec) nv[u] = load_rec4(a, r);
    }
    if (tid == 0) s_next[slot ^ 1] = gridDim.x + (int)atomicAdd(a.counters, 1u);
#pragma unroll
    for (int u = 0; u < kHist4Unroll; ++u) {
      if (c * kHist4Chunk + u * kHist4Threads + tid >= a.n_rec) break;
      const int b0 = bt.bin(0, v[u].x0);
      const int b1 = bt.bin(1, v[u].x1);
      const int b2 = bt.bin(2, v[u].x2);
      const uint32_t k = v[u].k;
      const float k1 = (k & 0xff00u) ? 1.f : 0.f, k2 = (k & 0xff0000u) ? 1.f : 0.f;
      const float k3 = (k & 0xff000000u) ? 1.f : 0.f;
      const uint32_t cell = (uint32_t)(b1 * d0 + b0) * (uint32_t)hp + (uint32_t)b2;
      red_add_v4(a.H + 4ull * cell, 1.f, k3, k2, k1);
      if (k & 0xffu) atomicAdd(s_c0 + b0, 1u);
    }
    __syncthreads();  // s_next[slot ^ 1] visible; s_next[slot] free for reuse
#pragma unroll
    for (int u = 0; u < kHist4Unroll; ++u) v[u] = nv[u];
    c = cn;
    slot ^= 1;
  }
  phase(0, 2);
  pdl_release();
  phase(0, 3);
  for (int i = tid; i < a.d0; i += kHist4Threads)
    if (s_c0[i]) atomicAdd(a.G0 + i, s_c0[i]);
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.counters + 1, 1u) == gridDim.x - 1) {  // last CTA: reset for the next launch
      a.counters[0] = 0u;
      a.counters[1] = 0u;
    }
  }
  phase(0, 4);
}

// ----------------------------------------------------------------- plane --
constexpr int kPlaneThreads = 512;
constexpr int kZeroBytes = 16384;  // zero source of the bulk stores that re-zero H

struct G4PlaneArgs {
  float* H;                  // [d1][d0][hp] float4, re-zeroed here
  unsigned long long* S;     // [d0][nbk][d1][W] packed {cnt, c3, c2}, columns < d2 - 1
  unsigned long long* G;     // [d0][d1p] the same at column d2 - 1 (b2 = any)
  uint32_t* R1;              // [d0][d1p]
  uint32_t* G0;              // [d0] raw c0, re-zeroed here
  uint32_t* P0;              // [d0] inclusive prefix of G0
  int32_t d0, d1, d2, d2p, d1p;
  int32_t hp;                // histogram row pitch in cells (odd: conflict-free row walk)
  int32_t W, nbk;            // S column blocks (the eval's units)
  int32_t half;              // b0 rows of the cluster's first CTA
  int32_t ns2, seg2;         // b2 segments of the row walk
  int32_t ns0, seg0;         // b0 segments of the column walk
};

__device__ __forceinline__ float4 add4f(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
// exact f32 integer in [0, 2^23) -> u32 without the conversion unit
__device__ __forceinline__ uint32_t f2u_exact(float f) {
  return __float_as_uint(f + 8388608.f) - 0x4B000000u;
}

__device__ __forceinline__ void bulk_s2g(void* dst_gmem, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}

// Where column c of row b1 lives in the prefix tables, and the step
// between consecutive b0: columns < d2 - 1 in the eval's column blocks
// S[b0][c / W][b1][c % W], the last (b2 = any) in G[b0][b1].
__device__ __forceinline__ unsigned long long* table_column(unsigned long long* S, unsigned long long* G,
                                                            int W, int nbk, int d1, int d1p, int d2,
                                                            int b1, int c, int64_t& step) {
  if (c < d2 - 1) {
    const int blk = c / W;
    step = (int64_t)nbk * d1 * W;
    return S + ((int64_t)blk * d1 + b1) * W + (c - blk * W);
  }
  step = d1p;
  return G + b1;
}

// The (b0, b2) plane of one b1 is contiguous in H ([b1][b0][hp]).  A
// cluster of two CTAs owns it, split along b0: each CTA bulk-copies its half
// of the rows, re-zeroes them with bulk stores from a zeroed shared buffer,
// walks its rows along b2 and its columns along b0; the first CTA hands its
// column totals to the second through distributed shared memory as the b0
// carry.  The counts stay f32 through both walks (exact below 2^24) and are
// packed once.  Both walks are serial (one add per cell and channel, no
// shuffles) and two-level so that the whole CTA shares them.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPlaneThreads, 2)
    g4_plane_kernel(const __grid_constant__ G4PlaneArgs a) {
  extern __shared__ __align__(16) float4 s_tile[];  // [rows][hp], seg sums, carry, zeros
  __shared__ __align__(8) uint64_t bar;
  cg::cluster_group cluster = cg::this_cluster();
  const int h = (int)cluster.block_rank();
  const int b1 = blockIdx.x >> 1;
  const int d0 = a.d0, d2 = a.d2, hp = a.hp;
  const int r_beg = h ? a.half : 0, r_end = h ? d0 : a.half, nr = r_end - r_beg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = kPlaneThreads / 32;
  float4* s_seg = s_tile + (size_t)a.half * hp;
  float4* s_carry = s_seg + kPlaneThreads;  // [d2] column totals of the first half (rank 1)
  float4* s_zero = s_carry + d2;            // kZeroBytes of zeros
  const uint32_t tile_bytes = (uint32_t)(nr * hp * sizeof(float4));
  float4* H = reinterpret_cast<float4*>(a.H) + ((int64_t)b1 * d0 + r_beg) * hp;
  phase(1, 0);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < kZeroBytes / 16; i += kPlaneThreads) s_zero[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  fence_proxy_async();  // the zero buffer is read by the async proxy (bulk stores)
  __syncthreads();
  pdl_wait();  // the histogram is complete
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar, tile_bytes);
    constexpr uint32_t kChunk = 32768;
    for (uint32_t off = 0; off < tile_bytes; off += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_tile) + off, reinterpret_cast<const uint8_t*>(H) + off,
               min(kChunk, tile_bytes - off), &bar);
  }
  if (b1 == 0 && h == 0 && warp == nwarps - 1) {  // c0: inclusive prefix over b0, re-zero
    uint32_t carry = 0;
    for (int b = 0; b < d0; b += 32) {
      const int i = b + lane;
      uint32_t x = i < d0 ? a.G0[i] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      x += carry;
      if (i < d0) {
        a.P0[i] = x;
        a.G0[i] = 0u;
      }
      carry = __shfl_sync(0xffffffffu, x, 31);
    }
  }
  mbar_wait(&bar, 0);
  phase(1, 1);
  // re-zero the histogram rows just read (the next build starts from zero):
  // bulk stores from the zero buffer, issued by one thread, asynchronous
  if (tid == 0) {
    for (uint32_t off = 0; off < tile_bytes; off += kZeroBytes)
      bulk_s2g(reinterpret_cast<uint8_t*>(H) + off, s_zero, min((uint32_t)kZeroBytes, tile_bytes - off));
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  phase(1, 2);
  // row walk along b2
  {
    const int r = tid % nr, s = tid / nr;
    const bool live = s < a.ns2;
    const int c_lo = s * a.seg2, c_hi = min(d2, c_lo + a.seg2);
    float4* row = s_tile + (size_t)r * hp;
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live)
      for (int c = c_lo; c < c_hi; ++c) sum = add4f(sum, row[c]);
    if (live) s_seg[s * nr + r] = sum;
    __syncthreads();
    if (live) {
      float4 run = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = 0; q < s; ++q) run = add4f(run, s_seg[q * nr + r]);
      for (int c = c_lo; c < c_hi; ++c) {
        run = add4f(run, row[c]);
        row[c] = run;
      }
    }
    __syncthreads();
  }
  phase(1, 3);
  // column walk along b0; the first half's column totals are the second's carry
  const int c = tid % d2, s = tid / d2;
  const bool live = s < a.ns0;
  const int r_lo = s * a.seg0, r_hi = min(nr, r_lo + a.seg0);
  float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
  if (live)
    for (int r = r_lo; r < r_hi; ++r) sum = add4f(sum, s_tile[(size_t)r * hp + c]);
  if (live) s_seg[s * d2 + c] = sum;
  __syncthreads();
  if (h == 0 && s == 0) {
    float4 tot = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < a.ns0; ++q) tot = add4f(tot, s_seg[q * d2 + c]);
    *cluster.map_shared_rank(s_carry + c, 1) = tot;
  }
  cluster.sync();
  phase(1, 4);
  if (live) {
    float4 P = h ? s_carry[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < s; ++q) P = add4f(P, s_seg[q * d2 + c]);
    int64_t step;
    unsigned long long* S = table_column(a.S, a.G, a.W, a.nbk, a.d1, a.d1p, d2, b1, c, step);
    for (int r = r_lo; r < r_hi; ++r) {
      P = add4f(P, s_tile[(size_t)r * hp + c]);
      const int64_t b0 = r_beg + r;
      S[b0 * step] = (unsigned long long)f2u_exact(P.x) |
                     ((unsigned long long)f2u_exact(P.y) << 21) |
                     ((unsigned long long)f2u_exact(P.z) << 42);
      if (c == d2 - 1) a.R1[b0 * a.d1p + b1] = f2u_exact(P.w);
    }
  }
  pdl_release();
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  phase(1, 5);
}

// ------------------------------------------------------ sorted build --
// One-shot builds skip the global histogram: the reduction into a 16.5 MB
// table is what held g4_hist above the streaming rate (one L2 reduction per
// record, then a plane pass that re-reads and re-zeroes the table).  Here
// g4_sort streams the records once and writes each as a 4-byte key
// {b0, b2, k1, k2, k3, b1}, counting-sorted in shared memory by b1 within
// the CTA's record range, plus the range's bucket offsets; g4_gather then
// builds each b1's (b0, b2) plane in shared memory from its bucket's keys
// (32-bit shared atomics on 16-bit packed counters), prefixes it along b2
// and b0 and writes the same S / R1 / P0 tables as g4_plane.  Keys are
// 4 MB per 1M records and stay in L2.
constexpr int kSortThreads = 1024;
constexpr int kGatherThreads = 1024;
constexpr int kSortMaxD1 = 1024;  // b1 takes 10 key bits
constexpr int kSortSmemMax = 227 * 1024 - 4096;  // opt-in limit less the static arrays

struct G4SortArgs {
  const double* cert;
  const uint8_t* corr;
  int32_t n_rec;
  int32_t vec_ok;
  const double* grids;
  int32_t glen[3];
  int32_t d0, nb, per;         // buckets (one per b1), records per CTA
  int32_t off_ring;            // byte offset of the cp.async record ring (RING variant)
  uint32_t* keys;              // [n_rec] sorted by bucket within each CTA's range
  uint32_t* off;               // [parts][nb + 1] absolute key offsets of each bucket
  uint32_t* G0;                // [d0] model-0 correct counts per b0
};


constexpr int kRing = 3;  // records per thread in flight through the shared-memory ring

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// RING: each thread keeps kRing records in flight through a shared-memory
// ring filled by cp.async (no registers held), from before the bin tables
// are built until the range ends, so the records stream at the HBM rate
// while the tables are built; else (unaligned inputs, or no room) a
// rotation of register sets, two records ahead.
template <bool VEC, bool RING>
__global__ void __launch_bounds__(kSortThreads, 1) g4_sort_kernel(const __grid_constant__ G4SortArgs a) {
  extern __shared__ __align__(16) double s_grid[];  // grids, bucket tables, counts, keys
  __shared__ uint32_t s_c0[kMaxDim4];
  __shared__ uint32_t s_wsum[32];
  const int n_grid = a.glen[0] + a.glen[1] + a.glen[2];
  void* s_lut = s_grid + ((n_grid + 1) & ~1);           // [3][kLutBuckets] entries (16 B aligned)
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(s_lut) + 3 * kLutBuckets * kLutEntryBytes);  // [nb]
  uint32_t* s_key = s_cnt + ((a.nb + 3) & ~3);        // [per]
  uint32_t* s_sorted = s_key + a.per;                 // [per]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = blockIdx.x * a.per;
  const int cnt = min(a.n_rec - r0, a.per);
  phase(0, 0);
  constexpr int kGridRegs = 5;
  double gv[kGridRegs];
#pragma unroll
  for (int q = 0; q < kGridRegs; ++q) {
    const int i = tid + q * kSortThreads;
    gv[q] = i < n_grid ? __ldg(a.grids + i) : 0.0;
  }
  G4HistArgs ha{};
  ha.cert = a.cert;
  ha.corr = a.corr;
  ha.vec_ok = VEC ? 1 : 0;  // a compile-time branch in load_rec4
  constexpr int T = kSortThreads;
  double* s_rc = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(s_grid) + a.off_ring);  // [kRing][T][4]
  uint32_t* s_rk = reinterpret_cast<uint32_t*>(s_rc + (size_t)kRing * T * 4);                 // [kRing][T]
  auto issue = [&](int slot, int i) {  // record i of the range into this thread's slot
    if (i < cnt) {
      const double* src = a.cert + (int64_t)(r0 + i) * 4;
      double* dst = s_rc + ((size_t)slot * T + tid) * 4;
      cp_async16(dst, src);
      cp_async16(dst + 2, src + 2);
      cp_async4(s_rk + slot * T + tid, a.corr + (int64_t)(r0 + i) * 4);
    }
    cp_async_commit();  // one group per record, empty past the range
  };
  Rec4 v, w;  // register variant: two records per thread in flight from the start
  if (!RING) {
    if (tid < cnt) v = load_rec4(ha, r0 + tid);
    if (tid + kSortThreads < cnt) w = load_rec4(ha, r0 + tid + kSortThreads);
  }
#pragma unroll
  for (int q = 0; q < kGridRegs; ++q) {
    const int i = tid + q * kSortThreads;
    if (i < n_grid) s_grid[i] = gv[q];
  }
  for (int i = tid; i < a.d0; i += kSortThreads) s_c0[i] = 0u;
  for (int i = tid; i < a.nb; i += kSortThreads) s_cnt[i] = 0u;
  __syncthreads();
  phase(0, 1);
  // the ring fills while the tables are built (issued only now: queued
  // behind the records of every SM, the grid values would arrive late)
  if (RING) {
#pragma unroll
    for (int q = 0; q < kRing; ++q) issue(q, tid + q * T);
  }
  const BinTables<3> bt = build_bin_tables<3, kSortThreads>(a.glen, s_grid, s_lut);
  phase(0, 2);
  auto put = [&](int i, double x0, double x1, double x2, uint32_t k) {
    const uint32_t b0 = (uint32_t)bt.bin(0, x0);
    const uint32_t b1 = (uint32_t)bt.bin(1, x1);
    const uint32_t b2 = (uint32_t)bt.bin(2, x2);
    // bit 29: model 0's correct bit, counted per b0 in the scatter (one
    // shared atomic less in the streaming loop); the gather ignores it
    const uint32_t key = b0 | (b2 << 8) | ((k & 0xff00u) ? 1u << 16 : 0u) |
                         ((k & 0xff0000u) ? 1u << 17 : 0u) | ((k & 0xff000000u) ? 1u << 18 : 0u) |
                         (b1 << 19) | ((k & 0xffu) ? 1u << 29 : 0u);
    atomicAdd(s_cnt + b1, 1u);  // count only: the rank is taken in the scatter
    s_key[i] = key;
  };
  if (RING) {
    int slot = 0;
    for (int i = tid; i < cnt; i += T) {
      cp_async_wait<kRing - 1>();  // this record's group is complete
      const double* rc = s_rc + ((size_t)slot * T + tid) * 4;
      const double2 p = *reinterpret_cast<const double2*>(rc);
      const double x2 = rc[2];
      const uint32_t k = s_rk[slot * T + tid];
      issue(slot, i + kRing * T);
      put(i, p.x, p.y, x2, k);
      slot = slot == kRing - 1 ? 0 : slot + 1;
    }
    cp_async_wait<0>();
  } else
  // three records per trip in a rotation of three registers sets, each
  // loaded two records ahead (no register moves)
  for (int i = tid; i < cnt; i += 3 * T) {
    Rec4 x;
    if (i + 2 * T < cnt) x = load_rec4(ha, r0 + i + 2 * T);
    put(i, v.x0, v.x1, v.x2, v.k);
    if (i + 3 * T < cnt) v = load_rec4(ha, r0 + i + 3 * T);
    if (i + T >= cnt) break;
    put(i + T, w.x0, w.x1, w.x2, w.k);
    if (i + 4 * T < cnt) w = load_rec4(ha, r0 + i + 4 * T);
    if (i + 2 * T >= cnt) break;
    put(i + 2 * T, x.x0, x.x1, x.x2, x.k);
  }
  phase(0, 3);
  pdl_release();
  __syncthreads();
  // exclusive scan of the bucket counts (two per thread, nb <= 2 * kSortThreads)
  {
    const int i0 = 2 * tid, i1 = 2 * tid + 1;
    const uint32_t t0 = i0 < a.nb ? s_cnt[i0] : 0u, t1 = i1 < a.nb ? s_cnt[i1] : 0u;
    uint32_t x = t0 + t1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = s_wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_wsum[lane] = w;
    }
    __syncthreads();
    const uint32_t excl = x - (t0 + t1) + (warp ? s_wsum[warp - 1] : 0u);
    uint32_t* off = a.off + (int64_t)blockIdx.x * (a.nb + 1);
    if (i0 < a.nb) {
      s_cnt[i0] = excl;
      off[i0] = (uint32_t)r0 + excl;
    }
    if (i1 < a.nb) {
      s_cnt[i1] = excl + t0;
      off[i1] = (uint32_t)r0 + excl + t0;
    }
    if (tid == 0) off[a.nb] = (uint32_t)(r0 + cnt);
  }
  __syncthreads();
  phase(0, 4);
  for (int i = tid; i < cnt; i += kSortThreads) {
    const uint32_t key = s_key[i];
    s_sorted[atomicAdd(s_cnt + ((key >> 19) & 1023u), 1u)] = key;
    if (key & (1u << 29)) atomicAdd(s_c0 + (key & 255u), 1u);
  }
  fence_proxy_async();  // the scattered keys are read next by the async proxy
  __syncthreads();
  // the range's keys leave by one bulk copy (16-byte multiple) plus a tail
  const int bulk = cnt & ~3;
  if (tid == 0 && bulk > 0) {
    bulk_s2g(a.keys + r0, s_sorted, (uint32_t)bulk * 4u);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  for (int i = bulk + tid; i < cnt; i += kSortThreads) a.keys[r0 + i] = s_sorted[i];
  for (int i = tid; i < a.d0; i += kSortThreads)
    if (s_c0[i]) atomicAdd(a.G0 + i, s_c0[i]);
  if (tid == 0 && bulk > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  phase(0, 5);
}

struct G4GatherArgs {
  const uint32_t* keys;
  const uint32_t* off;        // [parts][nb + 1]
  int32_t n_parts, nb;
  unsigned long long* S;      // [d0][nbk][d1][W] packed {cnt, c3, c2}, columns < d2 - 1
  unsigned long long* G;      // [d0][d1p] the same at column d2 - 1 (b2 = any)
  uint32_t* R1;               // [d0][d1p]
  uint32_t* G0;               // [d0] raw c0, re-zeroed here
  uint32_t* P0;               // [d0] inclusive prefix of G0
  int32_t d0, d1, d2, d2p, d1p;
  int32_t hp;                 // plane row pitch in cells (odd: conflict-free row walk)
  int32_t W, nbk;             // S column blocks (the eval's units)
  int32_t ns2, seg2;          // b2 segments of the row walk
  int32_t ns0, seg0;          // b0 segments of the column walk
};

// One CTA per b1 builds the whole (b0, b2) plane (b1's bin holds ~1/d1 of
// the records by construction of the quantile grids, so the CTAs are
// balanced).  A warp takes one record range's segment of the bucket at a
// time, a key per lane.
__global__ void __launch_bounds__(kGatherThreads, 1) g4_gather_kernel(const __grid_constant__ G4GatherArgs a) {
  extern __shared__ __align__(16) unsigned long long s_pl[];  // [d0][hp], then tables
  __shared__ uint32_t s_total;
  const int b1 = blockIdx.x;
  const int d0 = a.d0, d2 = a.d2, hp = a.hp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = kGatherThreads / 32;
  const int cells = d0 * hp;
  uint32_t* s_w = reinterpret_cast<uint32_t*>(s_pl);                  // [cells] x 2 words
  uint32_t* s_c2 = s_w + 2 * (size_t)cells;                           // [cells]
  uint32_t* s_c1 = s_c2 + cells;                                      // [d0]
  unsigned long long* s_seg = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(s_c1 + d0) + 15) & ~(uintptr_t)15);  // [kGatherThreads]
  uint32_t* s_beg = reinterpret_cast<uint32_t*>(s_seg + kGatherThreads);  // [parts] first key
  uint32_t* s_end = s_beg + a.n_parts;                                // [parts] end key
  phase(1, 0);
  for (int i = tid; i < cells; i += kGatherThreads) {
    s_pl[i] = 0ull;
    s_c2[i] = 0u;
  }
  for (int i = tid; i < d0; i += kGatherThreads) s_c1[i] = 0u;
  // the eval's CTAs (one per SM, pinned by their register file) take the
  // SMs this kernel leaves idle and wait there in griddepcontrol.wait
  pdl_release();
  pdl_wait();  // keys, offsets and G0 are complete
  if (b1 == 0 && warp == nwarps - 1) {  // c0: inclusive prefix over b0, re-zero
    uint32_t carry = 0;
    for (int b = 0; b < d0; b += 32) {
      const int i = b + lane;
      uint32_t x = i < d0 ? a.G0[i] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      x += carry;
      if (i < d0) {
        a.P0[i] = x;
        a.G0[i] = 0u;
      }
      carry = __shfl_sync(0xffffffffu, x, 31);
    }
  }
  // this bucket's key segment in every record range
  uint32_t len = 0;
  if (tid < a.n_parts) {
    const uint32_t* o = a.off + (int64_t)tid * (a.nb + 1) + b1;
    const uint32_t b = o[0], e = o[1];
    s_beg[tid] = b;
    s_end[tid] = e;
    len = e - b;
  }
  if (tid == 0) s_total = 0u;
  __syncthreads();
  const uint32_t wl = __reduce_add_sync(0xffffffffu, len);
  if (lane == 0 && wl) atomicAdd(&s_total, wl);
  __syncthreads();
  phase(1, 1);
  const uint32_t total = s_total;
  const int n_parts = a.n_parts;
  // shared 64-bit adds are CAS loops on sm_100: count in 32-bit words
  // instead, {cnt | c3 << 16, c2 | c1 << 16} while no field can reach 2^16
  // (fewer than 2^16 keys in the bucket), else {cnt, c3} with c2 per cell
  // and c1 per row apart; then pack once
  const bool narrow = total < 65536u;
  auto count = [&](uint32_t key) {
    const int r = (int)(key & 255u);
    const int cell = r * hp + (int)((key >> 8) & 255u);
    const uint32_t k3 = (key >> 18) & 1u;
    if (narrow) {
      atomicAdd(s_w + 2 * cell, 1u + (k3 << 16));
      const uint32_t w1 = ((key >> 17) & 1u) | (key & (1u << 16));
      if (w1) atomicAdd(s_w + 2 * cell + 1, w1);
    } else {
      atomicAdd(s_w + 2 * cell, 1u);
      if (k3) atomicAdd(s_w + 2 * cell + 1, 1u);
      if (key & (1u << 17)) atomicAdd(s_c2 + cell, 1u);
      if (key & (1u << 16)) atomicAdd(s_c1 + r, 1u);
    }
  };
  // a warp per record range: the first kHead x 32 keys of the segments of
  // kBatch ranges are loaded at once (kHead * kBatch coalesced loads in
  // flight per lane, one latency for the whole batch), the rest of a long
  // segment inline
  constexpr int kHead = 3, kBatch = 5;
  constexpr uint32_t kNone = 0xffffffffu;
  for (int p0 = warp; p0 < n_parts; p0 += nwarps * kBatch) {
    uint32_t k[kBatch][kHead];
#pragma unroll
    for (int m = 0; m < kBatch; ++m) {
      const int p = p0 + m * nwarps;
      const uint32_t b = p < n_parts ? s_beg[p] : 0u, e = p < n_parts ? s_end[p] : 0u;
#pragma unroll
      for (int j = 0; j < kHead; ++j) {
        const uint32_t i = b + 32u * j + lane;
        k[m][j] = i < e ? __ldg(a.keys + i) : kNone;
      }
    }
#pragma unroll
    for (int m = 0; m < kBatch; ++m)
#pragma unroll
      for (int j = 0; j < kHead; ++j)
        if (k[m][j] != kNone) count(k[m][j]);
#pragma unroll 1
    for (int m = 0; m < kBatch; ++m) {
      const int p = p0 + m * nwarps;
      if (p >= n_parts) break;
      const uint32_t e = s_end[p];
      for (uint32_t i = s_beg[p] + 32u * kHead + lane; i < e; i += 32u) count(__ldg(a.keys + i));
    }
  }
  __syncthreads();
  phase(1, 2);
  // row walk along b2, packing each cell to {cnt, c3, c2} (21-bit fields)
  // as its prefix is stored.  Narrow: the 16-bit fields of the two words
  // are prefixed by plain 64-bit adds (no field's sum reaches 2^16), and
  // the row total's c1 field is the row's C1 count.
  {
    const int r = tid % d0, s = tid / d0;
    const bool live = s < a.ns2;
    const int c_lo = s * a.seg2, c_hi = min(d2, c_lo + a.seg2);
    const int rb = r * hp;
    unsigned long long sum = 0;
    if (live) {
      if (narrow)
        for (int c = c_lo; c < c_hi; ++c) sum += s_pl[rb + c];
      else
        for (int c = c_lo; c < c_hi; ++c) {
          const int cell = rb + c;
          sum += (unsigned long long)s_w[2 * cell] | ((unsigned long long)s_w[2 * cell + 1] << 21) |
                 ((unsigned long long)s_c2[cell] << 42);
        }
      s_seg[s * d0 + r] = sum;
    }
    __syncthreads();
    if (live) {
      unsigned long long run = 0;
      for (int p = 0; p < s; ++p) run += s_seg[p * d0 + r];
      if (narrow) {
        for (int c = c_lo; c < c_hi; ++c) {
          run += s_pl[rb + c];
          s_pl[rb + c] = (run & 0xffffull) | (((run >> 16) & 0xffffull) << 21) |
                         (((run >> 32) & 0xffffull) << 42);
        }
        if (c_hi == d2) s_c1[r] = (uint32_t)(run >> 48);
      } else {
        for (int c = c_lo; c < c_hi; ++c) {
          const int cell = rb + c;
          run += (unsigned long long)s_w[2 * cell] | ((unsigned long long)s_w[2 * cell + 1] << 21) |
                 ((unsigned long long)s_c2[cell] << 42);
          s_pl[cell] = run;  // the cell's two words, read just above
        }
      }
    }
    __syncthreads();
  }
  phase(1, 3);
  // column walk along b0 (prefix along b2 already in place); c1 prefix over b0
  const int c = tid % d2, s = tid / d2;
  const bool live = s < a.ns0;
  const int r_lo = s * a.seg0, r_hi = min(d0, r_lo + a.seg0);
  unsigned long long sum = 0;
  if (live)
    for (int r = r_lo; r < r_hi; ++r) sum += s_pl[(size_t)r * hp + c];
  if (live) s_seg[s * d2 + c] = sum;
  if (warp == nwarps - 1) {
    uint32_t carry = 0;
    for (int b = 0; b < d0; b += 32) {
      const int r = b + lane;
      uint32_t v = r < d0 ? s_c1[r] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      v += carry;
      if (r < d0) a.R1[(int64_t)r * a.d1p + b1] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  phase(1, 4);
  if (live) {
    unsigned long long P = 0;
    for (int p = 0; p < s; ++p) P += s_seg[p * d2 + c];
    int64_t step;
    unsigned long long* dst = table_column(a.S, a.G, a.W, a.nbk, a.d1, a.d1p, d2, b1, c, step);
    dst += r_lo * step;
    const unsigned long long* src = s_pl + (size_t)r_lo * hp + c;
    for (int r = r_lo; r < r_hi; ++r) {  // pointers stepped, no per-row index math
      P += *src;
      *dst = P;
      src += hp;
      dst += step;
    }
  }
  phase(1, 5);
}

// ------------------------------------------------------------------ eval --
constexpr int kEvalThreads = 256;

struct G4EvalArgs {
  int32_t d0, d1, d2, d1p, d0p;
  int32_t W, Wp, nbk, nseg, seg_len;    // columns per unit, walker row pitch, column blocks per slab, row segments
  int32_t n_units;                      // d0 * nbk
  int64_t sb[16];                       // first config of the structure with model mask m
  int64_t cfg_begin, cfg_count;
  int64_t n_rec;
  double rcp_n;
  const double* cost1;
  const unsigned long long* S;  // [d0][nbk][d1][W] prefixed along b0 and b2, packed {cnt, c3, c2}
  const unsigned long long* G;  // [d0][d1p] the same at b2 = any (row totals)
  const uint32_t* R1;           // [d0][d1p] C1 over b0 <= k0, b1, any b2
  const uint32_t* P0;           // [d0p] C0(k0)
  int32_t group_smem;           // bytes of shared memory per group
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

// One config's outputs given its frac row and mean cost (the reference's
// epilogue, src/kernels.py:57-61: frac = count / n, mean += frac * cost1 in
// stage order, acc = correct / n).
__device__ __forceinline__ void st_v4_f64(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}

// ALL: accuracy, mean_cost and forward_frac all requested (the sweep's usual
// call) and forward_frac 32-byte aligned: the frac row is one 256-bit store
// (a warp writes 1 KB of whole lines; two 128-bit stores per row write every
// line twice, half each time: tools/micro_store.cu, 14.5 vs 10.4 us for the
// 52 B/config outputs of 1M configs).
template <bool ALL>
__device__ __forceinline__ void store4(const G4EvalArgs& a, int64_t i, double f0, double f1,
                                       double f2, double f3, double mean, uint32_t correct,
                                       double n, double rcp) {
  if (ALL) {
    st_v4_f64(a.frac + i * 4, f0, f1, f2, f3);
  } else if (a.frac) {
    double2* row = reinterpret_cast<double2*>(a.frac + i * 4);
    row[0] = make_double2(f0, f1);
    row[1] = make_double2(f2, f3);
  }
  if (ALL || a.cost) a.cost[i] = mean;
  if (ALL || a.acc) a.acc[i] = div_count((double)correct, n, rcp);
  if (a.n_correct) a.n_correct[i] = correct;
}

// A config of K stages with reach counts reach[0..K-2] (after stages
// 0..K-2) and stage costs cst[0..K-1], scored from scratch (edge cells).
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
  store4<false>(a, i, fr[0], fr[1], fr[2], fr[3], mean, correct, n, rcp);
}

// Scoring.  Units are (b0 slab k0, block of W columns k2); the gather left
// S prefixed along b0 and b2 in blocks [k0][block][b1][W] (plus the row
// totals G = the b2 = "any" column, and R1), so the b1 prefix of a column
// needs only that column: no exchange between CTAs (the previous design
// split a slab by rows over a four-CTA cluster and exchanged the b1 carry
// through distributed shared memory).  A unit is staged by three bulk
// copies and scored by a group of 256 threads:
//   1. walker (column c, row segment s) sums its segment; warps 0 / 1
//      prefix the row totals and C1 along b1;
//   2. row-shared terms of every row (the stage-2 fraction, the partial
//      mean cost and correct count of the longest structure); the edge
//      configs at k2 = any of this block's share of the rows;
//   3. the walk: carry = the segments before, then each row's prefix P
//      scores config (k0, k1, c); the last row (k1 = any) is the column
//      total and scores the structure that skips model 1 at (k0, c).
constexpr int kEvalGroups = 4;

// Named barrier of one 256-thread group (ids 1..kEvalGroups; 0 is __syncthreads).
__device__ __forceinline__ void group_sync(int grp) {
  asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "n"(kEvalThreads) : "memory");
}

template <bool ALL>
__device__ __forceinline__ void eval_unit(const G4EvalArgs& a, int u, const unsigned long long* s_col,
                                          unsigned long long* s_g, uint32_t* s_c1,
                                          const uint32_t* s_p0, unsigned long long* s_seg,
                                          double* s_rowf, double* s_rowm, uint32_t* s_rowc,
                                          int tid, int grp) {
  const int d0 = a.d0, d1 = a.d1, d2 = a.d2, W = a.W, nbk = a.nbk;
  const int g0 = d0 - 1, g1 = d1 - 1, g2 = d2 - 1;
  const int k0 = u / nbk, blk = u - k0 * nbk;
  const int c_lo = blk * W, nc = min(g2, c_lo + W) - c_lo;
  const int lane = tid & 31, warp = tid >> 5;
  const bool any0 = k0 == g0;
  // skip a slab none of whose configs is in the requested range: a slab
  // k0 < g0 scores structures (0,1) .. (0,1,2,3), the first starting at
  // sb[3] + k0 and the last ending at sb[15] + (k0 + 1) g1 g2; the any slab
  // scores the singletons (from config 0) through (1,2,3)
  const int64_t lo = any0 ? 0 : a.sb[3] + k0;
  const int64_t hi = any0 ? a.sb[14] + (int64_t)g1 * g2 : a.sb[15] + (int64_t)(k0 + 1) * g1 * g2;
  if (hi <= a.cfg_begin || lo >= a.cfg_begin + a.cfg_count) return;
  const bool full = lo >= a.cfg_begin && hi <= a.cfg_begin + a.cfg_count;
  // 1. segment sums; prefixes of the row totals and of C1 along b1
  const int wc = tid % a.Wp, ws = tid / a.Wp;
  const bool walker = ws < a.nseg && wc < nc;
  const int r_lo = ws * a.seg_len, r_hi = min(d1, r_lo + a.seg_len);
  if (walker) {
    unsigned long long t = 0;
    for (int r = r_lo; r < r_hi; ++r) t += s_col[r * W + wc];
    s_seg[ws * W + wc] = t;
  }
  if (warp == 0) {
    unsigned long long carry = 0;
    for (int b = 0; b < d1; b += 32) {
      const int r = b + lane;
      unsigned long long x = r < d1 ? s_g[r] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      x += carry;
      if (r < d1) s_g[r] = x;
      carry = __shfl_sync(0xffffffffu, x, 31);
    }
  } else if (warp == 1) {
    uint32_t carry = 0;
    for (int b = 0; b < d1; b += 32) {
      const int r = b + lane;
      uint32_t x = r < d1 ? s_c1[r] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      x += carry;
      if (r < d1) s_c1[r] = x;
      carry = __shfl_sync(0xffffffffu, x, 31);
    }
  }
  group_sync(grp);
  const double n = (double)a.n_rec, rcp = a.rcp_n;
  const double one = div_count(n, n, rcp);
  const double c0c = __ldg(a.cost1 + 0), c1c = __ldg(a.cost1 + 1), c2c = __ldg(a.cost1 + 2),
               c3c = __ldg(a.cost1 + 3);
  const Cell3 tot = unpack3(s_g[g1]);  // slab total: (k0, g1, g2)
  const uint32_t C1g = s_c1[g1];
  const uint32_t base0 = s_p0[g0] - s_p0[k0];  // slab k0: model 0 completes b0 > k0
  const double f1 = div_count((double)tot.cnt, n, rcp);
  const double m1 = dadd(dadd(0.0, dmul(one, c0c)), dmul(f1, c1c));
  // 2. row-shared terms of the longest structure:
  //   slab k0: (0,1,2,3) -> frac[2] = cnt(k0,k1,g)/n, mean through stage 2,
  //            correct through stage 1 plus C2(k0,k1,g)
  //   any:     (1,2,3)   -> frac[1] = cnt(g,k1,g)/n, mean through stage 1,
  //            correct of stage 0 (model 1) plus C2(g,k1,g)
  for (int r = tid; r < g1; r += kEvalThreads) {
    const Cell3 rg = unpack3(s_g[r]);
    const double fr = div_count((double)rg.cnt, n, rcp);
    s_rowf[r] = fr;
    if (!any0) {
      s_rowm[r] = dadd(m1, dmul(fr, c2c));
      s_rowc[r] = base0 + (C1g - s_c1[r]) + rg.c2;
    } else {
      s_rowm[r] = dadd(dadd(0.0, dmul(one, c1c)), dmul(fr, c2c));
      s_rowc[r] = (C1g - s_c1[r]) + rg.c2;
    }
  }
  // edge configs at k2 = any for this block's share of the rows, and (block
  // 0) the slab's corner structures
  {
    const int per = (g1 + nbk - 1) / nbk;
    const int e_lo = min(g1, blk * per), e_hi = min(g1, e_lo + per);
    const int n_items = (e_hi - e_lo) + (blk == 0 ? 1 : 0);
    for (int e = tid; e < n_items; e += kEvalThreads) {
      if (e < e_hi - e_lo) {
        const int k1 = e_lo + e;
        const Cell3 p = unpack3(s_g[k1]);
        if (!any0) {  // (0,1,2) and (0,1,3) at (k0, k1)
          const uint32_t reach[2] = {tot.cnt, p.cnt};
          const uint32_t c01 = base0 + (C1g - s_c1[k1]);
          const double cst2[3] = {c0c, c1c, c2c}, cst3[3] = {c0c, c1c, c3c};
          put4<3>(a, a.sb[7] + (int64_t)k0 * g1 + k1, reach, cst2, c01 + p.c2, n, rcp, one);
          put4<3>(a, a.sb[11] + (int64_t)k0 * g1 + k1, reach, cst3, c01 + p.c3, n, rcp, one);
        } else {  // (1,2), (1,3) at k1
          const uint32_t reach[1] = {p.cnt};
          const uint32_t c1 = C1g - s_c1[k1];
          const double cA[2] = {c1c, c2c}, cB[2] = {c1c, c3c};
          put4<2>(a, a.sb[6] + k1, reach, cA, c1 + p.c2, n, rcp, one);
          put4<2>(a, a.sb[10] + k1, reach, cB, c1 + p.c3, n, rcp, one);
        }
      } else if (!any0) {  // (0,1), (0,2), (0,3) at k0
        const uint32_t reach[1] = {tot.cnt};
        const double cA[2] = {c0c, c1c}, cB[2] = {c0c, c2c}, cC[2] = {c0c, c3c};
        put4<2>(a, a.sb[3] + k0, reach, cA, base0 + C1g, n, rcp, one);
        put4<2>(a, a.sb[5] + k0, reach, cB, base0 + tot.c2, n, rcp, one);
        put4<2>(a, a.sb[9] + k0, reach, cC, base0 + tot.c3, n, rcp, one);
      } else {  // singletons
        const uint32_t* none = nullptr;
        const double cA[1] = {c0c}, cB[1] = {c1c}, cC[1] = {c2c}, cD[1] = {c3c};
        put4<1>(a, a.sb[1], none, cA, s_p0[g0], n, rcp, one);
        put4<1>(a, a.sb[2], none, cB, C1g, n, rcp, one);
        put4<1>(a, a.sb[4], none, cC, tot.c2, n, rcp, one);
        put4<1>(a, a.sb[8], none, cD, tot.c3, n, rcp, one);
      }
    }
  }
  group_sync(grp);
  if (!walker) return;
  // 3. the walk
  const int col = c_lo + wc;
  unsigned long long P = 0;
  for (int q = 0; q < ws; ++q) P += s_seg[q * W + wc];
  const int64_t row_base = (any0 ? a.sb[14] : a.sb[15] + (int64_t)k0 * g1 * g2) + col - a.cfg_begin;
  const int r_end = min(r_hi, g1);
  if (ALL && full && !a.n_correct) {
    // the usual sweep: every output of the slab requested, the configs of
    // consecutive rows g2 apart -- walk three output pointers
    const int64_t i0 = row_base + (int64_t)r_lo * g2;
    double* pf = a.frac + i0 * 4;
    double* pc = a.cost + i0;
    double* pa = a.acc + i0;
    for (int r = r_lo; r < r_end; ++r) {
      P += s_col[r * W + wc];
      const Cell3 p = unpack3(P);
      const double f3 = div_count((double)p.cnt, n, rcp);
      const double rf = s_rowf[r];
      const double mean = dadd(s_rowm[r], dmul(f3, c3c));
      const uint32_t correct = s_rowc[r] - p.c2 + p.c3;
      if (!any0)
        st_v4_f64(pf, one, f1, rf, f3);
      else
        st_v4_f64(pf, one, rf, f3, 0.0);
      *pc = mean;
      *pa = div_count((double)correct, n, rcp);
      pf += 4 * (int64_t)g2;
      pc += g2;
      pa += g2;
    }
  } else {
    for (int r = r_lo; r < r_end; ++r) {
      P += s_col[r * W + wc];
      const int64_t i = row_base + (int64_t)r * g2;
      if (!full && (i < 0 || i >= a.cfg_count)) continue;
      const Cell3 p = unpack3(P);
      const double f3 = div_count((double)p.cnt, n, rcp);
      const double rf = s_rowf[r];
      const double mean = dadd(s_rowm[r], dmul(f3, c3c));
      const uint32_t correct = s_rowc[r] - p.c2 + p.c3;
      if (!any0)
        store4<ALL>(a, i, one, f1, rf, f3, mean, correct, n, rcp);
      else
        store4<ALL>(a, i, one, rf, f3, 0.0, mean, correct, n, rcp);
    }
  }
  if (r_hi == d1) {  // the last segment: P is the column total (k0, g1, col)
    P += s_col[g1 * W + wc];
    const Cell3 p = unpack3(P);
    if (!any0) {  // (0,2,3) at (k0, col)
      const uint32_t reach[2] = {tot.cnt, p.cnt};
      const double cst[3] = {c0c, c2c, c3c};
      put4<3>(a, a.sb[13] + (int64_t)k0 * g2 + col, reach, cst, base0 + (tot.c2 - p.c2) + p.c3, n,
              rcp, one);
    } else {  // (2,3) at col
      const uint32_t reach[1] = {p.cnt};
      const double cst[2] = {c2c, c3c};
      put4<2>(a, a.sb[12] + col, reach, cst, (tot.c2 - p.c2) + p.c3, n, rcp, one);
    }
  }
}

// One CTA of kEvalGroups x 256 threads per SM (its 64-register threads
// fill the register file, so the CTAs cannot pile onto the SMs the gather
// frees first, which the launch-early programmatic dependency would do with
// small CTAs: 118 SMs hosting four and 17 none).  Group g of CTA c scores
// units u = c + (g + kEvalGroups * k) * gridDim.x: every SM gets
// n_units / #SMs units, within one.  A group syncs on its own named barrier
// and stages each unit with three bulk copies on its own mbarrier.
template <bool ALL>
__global__ void __launch_bounds__(kEvalGroups * kEvalThreads, 1) g4_eval_kernel(const __grid_constant__ G4EvalArgs a) {
  extern __shared__ __align__(16) unsigned char s_raw[];  // per group: unit buffer, P0, tables
  __shared__ __align__(8) uint64_t bar[kEvalGroups];
  const int d1 = a.d1, W = a.W, nbk = a.nbk;
  const int grp = threadIdx.x / kEvalThreads, tid = threadIdx.x % kEvalThreads;
  const uint32_t col_bytes = (uint32_t)d1 * W * 8, g_bytes = (uint32_t)a.d1p * 8,
                 r_bytes = (uint32_t)a.d1p * 4, p0_bytes = (uint32_t)a.d0p * 4;
  const uint32_t buf_bytes = col_bytes + g_bytes + r_bytes;
  unsigned char* buf = s_raw + (size_t)grp * a.group_smem;
  uint32_t* s_p0 = reinterpret_cast<uint32_t*>(buf + buf_bytes);
  unsigned long long* s_seg = reinterpret_cast<unsigned long long*>(s_p0 + a.d0p);  // [nseg][W]
  double* s_rowf = reinterpret_cast<double*>(s_seg + (size_t)a.nseg * W);             // [d1]
  double* s_rowm = s_rowf + d1;                                                        // [d1]
  uint32_t* s_rowc = reinterpret_cast<uint32_t*>(s_rowm + d1);                         // [d1]
  phase(2, 0);
  if (tid == 0) {
    mbar_init(&bar[grp], 1);
    fence_mbar_init();
  }
  group_sync(grp);
  pdl_wait();  // the prefix tables are complete
  uint32_t parity = 0;
  bool first = true;
  for (int u = blockIdx.x + grp * gridDim.x; u < a.n_units; u += kEvalGroups * gridDim.x) {
    if (tid == 0) {
      const int k0 = u / nbk, blk = u - k0 * nbk;
      fence_proxy_async();  // the generic reads of the buffer (previous unit) come first
      mbar_arrive_expect_tx(&bar[grp], buf_bytes + (first ? p0_bytes : 0u));
      bulk_g2s(buf, a.S + ((int64_t)k0 * nbk + blk) * d1 * W, col_bytes, &bar[grp]);
      bulk_g2s(buf + col_bytes, a.G + (int64_t)k0 * a.d1p, g_bytes, &bar[grp]);
      bulk_g2s(buf + col_bytes + g_bytes, a.R1 + (int64_t)k0 * a.d1p, r_bytes, &bar[grp]);
      if (first) bulk_g2s(s_p0, a.P0, p0_bytes, &bar[grp]);
    }
    first = false;
    mbar_wait(&bar[grp], parity);
    parity ^= 1u;
    phase(2, 1);
    eval_unit<ALL>(a, u, reinterpret_cast<const unsigned long long*>(buf),
                   reinterpret_cast<unsigned long long*>(buf + col_bytes),
                   reinterpret_cast<uint32_t*>(buf + col_bytes + g_bytes), s_p0, s_seg, s_rowf, s_rowm,
                   s_rowc, tid, grp);
    group_sync(grp);  // the buffer is free again
  }
  phase(2, 5);
}

}  // namespace

// ------------------------------------------------------------ host side --
#ifndef GS_G4_EVAL_W
#define GS_G4_EVAL_W 20  // columns per eval unit (config 2: five blocks of 20 per slab)
#endif

// Eval unit shape: W columns (even: the unit's block is a 16-byte multiple
// for the bulk copy), row segments for 256 threads, and the shared memory
// of two unit buffers plus the tables.
#ifndef GS_G4_EVAL_WARP_ROWS
#define GS_G4_EVAL_WARP_ROWS 1  // walkers of a row segment padded to whole warps
#endif

struct EvalShape {
  int W, Wp, nbk, nseg, seg_len;
  size_t smem;
};

EvalShape eval_shape(int64_t d0, int64_t d1, int64_t d2) {
  const int64_t d1p = (d1 + 3) & ~3ll, d0p = (d0 + 3) & ~3ll, g2 = d2 - 1;
  EvalShape e{};
  for (e.W = (int)std::min<int64_t>(GS_G4_EVAL_W, (g2 + 1) & ~1ll); e.W >= 2; e.W -= 2) {
    e.Wp = GS_G4_EVAL_WARP_ROWS && e.W <= 32 ? 32 : e.W;
    e.nseg = (int)std::max<int64_t>(1, std::min<int64_t>(kEvalThreads / e.Wp, d1));
    e.seg_len = (int)((d1 + e.nseg - 1) / e.nseg);
    e.nseg = (int)((d1 + e.seg_len - 1) / e.seg_len);
    e.smem = round_up((size_t)(d1 * e.W * 8 + d1p * 12) + (size_t)d0p * 4 + (size_t)e.nseg * e.W * 8 +
                          (size_t)d1 * 20, 128);  // per group
    if (e.smem * kEvalGroups <= kGrid4SlabMax) break;
  }
  e.nbk = e.W >= 2 ? (int)((g2 + e.W - 1) / e.W) : 0;
  return e;
}

bool grid4_supported(int64_t n_rec, int32_t M, const int32_t* glen) {
  if (M != 4 || n_rec < 1 || n_rec >= kGrid4MaxRec) return false;
  const int64_t d0 = glen[0] + 1, d1 = glen[1] + 1, d2 = glen[2] + 1;
  const int64_t grid_bytes = (int64_t)(glen[0] + glen[1] + glen[2]) * 8 + 3 * kLutBuckets * kLutEntryBytes;
  if (glen[0] + glen[1] + glen[2] > 5 * kHist4Threads) return false;
  // plane tile [d0][d2p] x 16 B plus segment sums
  const int64_t plane_smem = ((d0 + 1) / 2 * (d2 | 1) + kPlaneThreads + d2) * 16 + kZeroBytes;
  return d0 <= kMaxDim4 && d2 <= kMaxDim4 && d1 <= 4096 && grid_bytes <= 96 * 1024 &&
         d2 <= kPlaneThreads && plane_smem <= (int64_t)kGrid4SlabMax && d1 >= 2 &&
         eval_shape(d0, d1, d2).W >= 2;
}

// Shared memory of the sorted build's two kernels (0 when it does not apply).
struct SortPlan {
  int parts, per, off_ring;
  bool ring;
  size_t sort_smem, gather_smem;
};

SortPlan sort_plan(const Grid4Layout& L, const int32_t* glen, int64_t n_rec) {
  SortPlan sp{};
  if (L.d1 > kSortMaxD1 || n_rec < 1) return sp;
  sp.parts = (int)std::max<int64_t>(1, std::min<int64_t>(sm_count(), (n_rec + kSortThreads - 1) / kSortThreads));
  sp.per = (int)(((n_rec + sp.parts - 1) / sp.parts + 31) & ~31ll);
  sp.parts = (int)((n_rec + sp.per - 1) / sp.per);
  sp.sort_smem = (size_t)((glen[0] + glen[1] + glen[2] + 1) & ~1) * 8 + 3 * kLutBuckets * kLutEntryBytes +
                 (size_t)((L.nb + 3) & ~3) * 4 + (size_t)sp.per * 8;
  sp.off_ring = (int)round_up(sp.sort_smem, 128);
  const size_t ring_bytes = (size_t)kRing * kSortThreads * 36;
  sp.ring = sp.off_ring + ring_bytes <= (size_t)kSortSmemMax;
  if (sp.ring) sp.sort_smem = sp.off_ring + ring_bytes;
  sp.gather_smem = (size_t)L.d0 * L.hp * 12 + (size_t)L.d0 * 4 + 16 + kGatherThreads * 8 +
                   (size_t)sp.parts * 12 + 4;
  if (sp.sort_smem > (size_t)kSortSmemMax || sp.gather_smem > kGrid4SlabMax || sp.parts > kGatherThreads ||
      L.d2 > kGatherThreads)
    sp.sort_smem = sp.gather_smem = 0;
  return sp;
}

Grid4Layout grid4_layout(const int32_t* glen, int64_t n_rec) {
  Grid4Layout L{};
  L.d0 = glen[0] + 1;
  L.d1 = glen[1] + 1;
  L.d2 = glen[2] + 1;
  L.d2p = (L.d2 + 1) & ~1;
  L.d1p = (L.d1 + 3) & ~3;
  L.hp = L.d2 | 1;
  L.nb = L.d1;
  L.max_parts = sm_count();
  const EvalShape es = eval_shape(L.d0, L.d1, L.d2);
  L.W = es.W;
  L.nbk = es.nbk;
  const size_t bH = round_up((size_t)L.d0 * L.d1 * L.hp * 16, 256);
  const size_t bS = round_up((size_t)L.d0 * L.nbk * L.d1 * L.W * 8, 256);
  const size_t bGt = round_up((size_t)L.d0 * L.d1p * 8, 256);
  const size_t bR1 = round_up((size_t)L.d0 * L.d1p * 4, 256);
  const size_t bG = round_up((size_t)L.d0 * 4, 256);
  L.offH = 0;
  L.offG0 = bH;
  L.offS = bH + bG;
  L.offGt = L.offS + bS;
  L.offR1 = L.offGt + bGt;
  L.offP0 = L.offR1 + bR1;
  L.offCnt = L.offP0 + bG;
  L.offKeys = L.offCnt + 256;
  L.offOff = L.offKeys + round_up((size_t)std::max<int64_t>(n_rec, 1) * 4, 256);
  L.bytes = L.offOff + round_up((size_t)L.max_parts * (L.nb + 1) * 4, 256);
  L.sorted = sort_plan(L, glen, n_rec).sort_smem != 0;
  return L;
}

cudaError_t grid4_accumulate(const double* cert, const uint8_t* corr, int64_t n_chunk,
                             const double* grids, const int32_t* glen, uint8_t* ws, bool dirty,
                             cudaStream_t st) {
  const Grid4Layout L = grid4_layout(glen, n_chunk);
  float* H = reinterpret_cast<float*>(ws + L.offH);
  uint32_t* G0 = reinterpret_cast<uint32_t*>(ws + L.offG0);
  if (dirty) {
    cudaError_t e = cudaMemsetAsync(ws, 0, L.offS, st);  // H and G0
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(ws + L.offCnt, 0, 256, st);
    if (e != cudaSuccess) return e;
  }
  G4HistArgs h{};
  h.cert = cert;
  h.corr = corr;
  h.n_rec = (int32_t)n_chunk;
  h.vec_ok = aligned16(cert) && ((reinterpret_cast<uintptr_t>(corr) & 3u) == 0);
  h.grids = grids;
  for (int j = 0; j < 3; ++j) h.glen[j] = glen[j];
  h.d0 = L.d0;
  h.hp = L.hp;
  h.H = H;
  h.G0 = G0;
  h.counters = reinterpret_cast<uint32_t*>(ws + L.offCnt);
  const size_t smem =
      (size_t)(glen[0] + glen[1] + glen[2]) * sizeof(double) + 3 * kLutBuckets * kLutEntryBytes;
  static SmemAttr smem_hist;
  cudaError_t e = ensure_smem(g4_hist_kernel, smem_hist, smem);
  if (e != cudaSuccess) return e;
  if (n_chunk == 0) return cudaSuccess;
  int64_t blocks = (n_chunk + kHist4Chunk - 1) / kHist4Chunk;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, sm_count()));
  g4_hist_kernel<<<(unsigned)blocks, kHist4Threads, smem, st>>>(h);
  return cudaGetLastError();
}

cudaError_t grid4_finish(const int32_t* glen, uint8_t* ws, cudaStream_t st) {
  const Grid4Layout L = grid4_layout(glen, 1);  // the table offsets do not depend on n_rec
  float* H = reinterpret_cast<float*>(ws + L.offH);
  uint32_t* G0 = reinterpret_cast<uint32_t*>(ws + L.offG0);
  cudaError_t e = cudaSuccess;

  G4PlaneArgs p{};
  p.H = H;
  p.S = reinterpret_cast<unsigned long long*>(ws + L.offS);
  p.G = reinterpret_cast<unsigned long long*>(ws + L.offGt);
  p.W = L.W;
  p.nbk = L.nbk;
  p.R1 = reinterpret_cast<uint32_t*>(ws + L.offR1);
  p.G0 = G0;
  p.P0 = reinterpret_cast<uint32_t*>(ws + L.offP0);
  p.d0 = L.d0;
  p.d1 = L.d1;
  p.d2 = L.d2;
  p.d2p = L.d2p;
  p.d1p = L.d1p;
  p.hp = L.hp;
  p.half = (L.d0 + 1) / 2;
  p.ns2 = std::max(1, std::min(kPlaneThreads / p.half, L.d2));
  p.seg2 = (L.d2 + p.ns2 - 1) / p.ns2;
  p.ns2 = (L.d2 + p.seg2 - 1) / p.seg2;
  p.ns0 = std::max(1, std::min(kPlaneThreads / L.d2, p.half));
  p.seg0 = (p.half + p.ns0 - 1) / p.ns0;
  p.ns0 = (p.half + p.seg0 - 1) / p.seg0;
  const size_t psmem = ((size_t)p.half * p.hp + kPlaneThreads + L.d2) * 16 + kZeroBytes;
  static SmemAttr smem_plane;
  e = ensure_smem(g4_plane_kernel, smem_plane, (size_t)kGrid4SlabMax);
  if (e != cudaSuccess) return e;
  return launch_pdl(g4_plane_kernel, (unsigned)(2 * L.d1), kPlaneThreads, psmem, st, p);
}

// One-shot build: the bucket-sorted kernels when their shared-memory plan
// fits (the headline shapes), else histogram + plane.  Either way the
// workspace is left as the streamed path expects it (H and G0 zero).
cudaError_t grid4_build(const double* cert, const uint8_t* corr, int64_t n_rec, const double* grids,
                        const int32_t* glen, uint8_t* ws, bool dirty, int passes, cudaStream_t st) {
  const Grid4Layout L = grid4_layout(glen, n_rec);
  const SortPlan sp = sort_plan(L, glen, n_rec);
  cudaError_t e = cudaSuccess;
  if (!L.sorted || sp.sort_smem == 0 || sp.parts > L.max_parts) {
    if (passes & 1) e = grid4_accumulate(cert, corr, n_rec, grids, glen, ws, dirty, st);
    if (e != cudaSuccess || !(passes & 2)) return e;
    return grid4_finish(glen, ws, st);
  }
  if (dirty && (passes & 1)) {
    if ((e = cudaMemsetAsync(ws, 0, L.offS, st)) != cudaSuccess) return e;  // H and G0
    if ((e = cudaMemsetAsync(ws + L.offCnt, 0, 256, st)) != cudaSuccess) return e;
  }
  uint32_t* keys = reinterpret_cast<uint32_t*>(ws + L.offKeys);
  uint32_t* off = reinterpret_cast<uint32_t*>(ws + L.offOff);
  uint32_t* G0 = reinterpret_cast<uint32_t*>(ws + L.offG0);
  G4SortArgs a{};
  a.cert = cert;
  a.corr = corr;
  a.n_rec = (int32_t)n_rec;
  a.vec_ok = aligned16(cert) && ((reinterpret_cast<uintptr_t>(corr) & 3u) == 0);
  a.grids = grids;
  for (int j = 0; j < 3; ++j) a.glen[j] = glen[j];
  a.d0 = L.d0;
  a.nb = L.nb;
  a.per = sp.per;
  a.keys = keys;
  a.off = off;
  a.G0 = G0;
  static SmemAttr smem_sort, smem_sort_r, smem_sort_s, smem_gather;
  a.off_ring = sp.off_ring;
  // the ring's cp.async copies want 16-byte aligned rows and 4-byte correct words
  const bool ring = sp.ring && a.vec_ok;
  const size_t smem = ring ? sp.sort_smem : (size_t)sp.off_ring;
  if (!(passes & 1)) {
  } else if (ring) {
    if ((e = ensure_smem(g4_sort_kernel<true, true>, smem_sort_r, kSortSmemMax)) != cudaSuccess) return e;
    g4_sort_kernel<true, true><<<(unsigned)sp.parts, kSortThreads, smem, st>>>(a);
  } else if (a.vec_ok) {
    if ((e = ensure_smem(g4_sort_kernel<true, false>, smem_sort, kSortSmemMax)) != cudaSuccess) return e;
    g4_sort_kernel<true, false><<<(unsigned)sp.parts, kSortThreads, smem, st>>>(a);
  } else {
    if ((e = ensure_smem(g4_sort_kernel<false, false>, smem_sort_s, kSortSmemMax)) != cudaSuccess) return e;
    g4_sort_kernel<false, false><<<(unsigned)sp.parts, kSortThreads, smem, st>>>(a);
  }
  if ((e = cudaGetLastError()) != cudaSuccess || !(passes & 2)) return e;

  G4GatherArgs g{};
  g.keys = keys;
  g.off = off;
  g.n_parts = sp.parts;
  g.nb = L.nb;
  g.S = reinterpret_cast<unsigned long long*>(ws + L.offS);
  g.G = reinterpret_cast<unsigned long long*>(ws + L.offGt);
  g.W = L.W;
  g.nbk = L.nbk;
  g.R1 = reinterpret_cast<uint32_t*>(ws + L.offR1);
  g.G0 = G0;
  g.P0 = reinterpret_cast<uint32_t*>(ws + L.offP0);
  g.d0 = L.d0;
  g.d1 = L.d1;
  g.d2 = L.d2;
  g.d2p = L.d2p;
  g.d1p = L.d1p;
  g.hp = L.hp;
  g.ns2 = std::max(1, std::min(kGatherThreads / L.d0, L.d2));
  g.seg2 = (L.d2 + g.ns2 - 1) / g.ns2;
  g.ns2 = (L.d2 + g.seg2 - 1) / g.seg2;
  g.ns0 = std::max(1, std::min(kGatherThreads / L.d2, L.d0));
  g.seg0 = (L.d0 + g.ns0 - 1) / g.ns0;
  g.ns0 = (L.d0 + g.seg0 - 1) / g.seg0;
  if ((e = ensure_smem(g4_gather_kernel, smem_gather, (size_t)kGrid4SlabMax)) != cudaSuccess) return e;
  return launch_pdl(g4_gather_kernel, (unsigned)L.d1, kGatherThreads, sp.gather_smem, st, g);
}

template <bool ALL>
cudaError_t launch_eval(const G4EvalArgs& a, cudaStream_t st) {
  static SmemAttr done;
  const size_t smem = (size_t)kEvalGroups * a.group_smem;
  cudaError_t e = ensure_smem(g4_eval_kernel<ALL>, done, smem);
  if (e != cudaSuccess) return e;
  const int grid = std::max(1, std::min(a.n_units, sm_count()));
  return launch_pdl(g4_eval_kernel<ALL>, (unsigned)grid, kEvalGroups * kEvalThreads, smem, st, a);
}

cudaError_t grid4_eval(int64_t n_rec, const int32_t* glen, const int64_t* struct_begin,
                       const uint32_t* struct_mask, int n_struct, const double* cost1,
                       int64_t cfg_begin, int64_t cfg_count, double* acc, double* cost,
                       double* frac, uint32_t* n_correct, const uint8_t* ws, cudaStream_t st) {
  const Grid4Layout L = grid4_layout(glen, n_rec);
  G4EvalArgs a{};
  const EvalShape es = eval_shape(L.d0, L.d1, L.d2);
  a.d0 = L.d0;
  a.d1 = L.d1;
  a.d2 = L.d2;
  a.d1p = L.d1p;
  a.d0p = (L.d0 + 3) & ~3;
  a.W = es.W;
  a.Wp = es.Wp;
  a.nbk = es.nbk;
  a.nseg = es.nseg;
  a.seg_len = es.seg_len;
  a.n_units = L.d0 * es.nbk;
  for (int s = 0; s < n_struct; ++s) a.sb[struct_mask[s] & 15u] = struct_begin[s];
  a.cfg_begin = cfg_begin;
  a.cfg_count = cfg_count;
  a.n_rec = n_rec;
  a.rcp_n = 1.0 / (double)n_rec;
  a.cost1 = cost1;
  a.S = reinterpret_cast<const unsigned long long*>(ws + L.offS);
  a.G = reinterpret_cast<const unsigned long long*>(ws + L.offGt);
  a.R1 = reinterpret_cast<const uint32_t*>(ws + L.offR1);
  a.P0 = reinterpret_cast<const uint32_t*>(ws + L.offP0);
  a.group_smem = (int32_t)es.smem;
  a.acc = acc;
  a.cost = cost;
  a.frac = frac;
  a.n_correct = n_correct;
  const bool all = acc && cost && frac && (reinterpret_cast<uintptr_t>(frac) & 31u) == 0;
  return all ? launch_eval<true>(a, st) : launch_eval<false>(a, st);
}

}  // namespace gs

#ifdef GS_PHASE_TIMING
// phase-timing builds only: copy the stamps [kernel][cta][slot][globaltimer,
// clock64] to host memory (kPhaseKernels * kPhaseCtas * kPhaseSlots * 2 u64)
extern "C" int gs_debug_phases(unsigned long long* host) {
  if (cudaMemcpyFromSymbol(host, gs::g_phase, sizeof(gs::g_phase)) != cudaSuccess) return GS_ECUDA;
  return GS_OK;
}
#endif
