// gs_common.cuh — shared device/host helpers for the gearserve B200 kernels.
//
// Contents: error plumbing for the C ABI, f64 arithmetic that never contracts
// into FMA (the reference's numba loop does separate multiply and add,
// src/kernels.py:57-61), the 1-D TMA bulk-copy + mbarrier primitives used to
// stage record tiles in shared memory, and a decoupled look-back block scan
// that gives order-preserving (stable) stream compaction in one pass.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/gearserve_b200.h"

namespace gs {

// ---------------------------------------------------------------- errors --
void set_cuda_error(cudaError_t e);

#define GS_CUDA_TRY(expr)                  \
  do {                                     \
    cudaError_t _e = (expr);               \
    if (_e != cudaSuccess) {               \
      ::gs::set_cuda_error(_e);            \
      return GS_ECUDA;                     \
    }                                      \
  } while (0)

#define GS_LAUNCH_CHECK() GS_CUDA_TRY(cudaGetLastError())

#define GS_REQUIRE(cond)      \
  do {                        \
    if (!(cond)) return GS_EINVAL; \
  } while (0)

__host__ __device__ inline bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Devices a process can drive through this library (one process may use
// several GPUs, e.g. one executor thread per device: src/serving.py:121-139).
constexpr int kMaxDevices = 64;

// Ordinal of the calling thread's current device (0 if it cannot be read).
int current_device();

// Number of SMs of the current device (cached per device; safe to call from
// any thread).
int sm_count();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the current
// device only, so the "already set" high-water mark is kept per device: a
// kernel first launched on device 1 gets its attribute there too.  Once set
// for a size, later calls (e.g. inside a CUDA-graph capture) issue nothing.
struct SmemAttr {
  std::atomic<int> bytes[kMaxDevices];  // zero-initialised (static storage)
};

template <typename Kernel>
cudaError_t ensure_smem(Kernel k, SmemAttr& attr, size_t bytes) {
  const int dev = current_device();
  std::atomic<int>& slot = attr.bytes[(dev >= 0 && dev < kMaxDevices) ? dev : 0];
  if ((int)bytes <= slot.load(std::memory_order_acquire) && dev < kMaxDevices) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && dev < kMaxDevices) {
    int cur = slot.load(std::memory_order_relaxed);
    while ((int)bytes > cur && !slot.compare_exchange_weak(cur, (int)bytes)) {
    }
  }
  return e;
}

// ------------------------------------------------------------ f64 epilogue --
// Explicit round-to-nearest intrinsics so nvcc cannot fuse a*b+c into a DFMA.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// x / n for integer counts 0 <= x <= n < 2^26, correctly rounded, in three
// FP64 ops instead of a full division: with rcp = RN(1/n) (IEEE division on
// the host), q0 = RN(x * rcp) is within one ulp of x/n, the remainder
// x - q0*n is exact in one FMA, and one FMA correction yields the correctly
// rounded quotient (Markstein's theorem).  Counts never produce the
// subnormal/overflow cases a general division has to check for.
// tests/test_gpu_grid.py checks it exhaustively against __ddiv_rn.
__device__ __forceinline__ double div_count(double x, double n, double rcp) {
  const double q0 = __dmul_rn(x, rcp);
  const double e = __fma_rn(-q0, n, x);
  return __fma_rn(e, rcp, q0);
}

// ------------------------------------------------------- TMA bulk (1-D) --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ----------------------------------------------------------- warp helpers --
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------- decoupled look-back scan ----
// A tile publishes one u64: bits 62-63 status, bits 0-61 a packed pair of
// 31-bit counts (field A in bits 0-30, field B in bits 31-61).  Sums of
// packed pairs never carry between fields because every count is < 2^31.
constexpr uint64_t kLbAggregate = 1ull << 62;
constexpr uint64_t kLbInclusive = 2ull << 62;
constexpr uint64_t kLbValueMask = (1ull << 62) - 1;
constexpr uint64_t kLbFieldMask = (1ull << 31) - 1;

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Warp 0 of the block: given this tile's packed aggregate, publish it, walk
// back over predecessors 32 at a time and return the exclusive prefix
// (packed).  Must be called by all 32 lanes of one warp.
__device__ __forceinline__ uint64_t lookback_exclusive(uint64_t* states, int64_t tile,
                                                       uint64_t aggregate) {
  const uint32_t lane = lane_id();
  if (tile == 0) {
    if (lane == 0) st_volatile_u64(&states[0], kLbInclusive | aggregate);
    return 0;
  }
  if (lane == 0) st_volatile_u64(&states[tile], kLbAggregate | aggregate);
  uint64_t excl = 0;
  int64_t pred = tile - 1;
  while (true) {
    const int64_t t = pred - (int64_t)lane;
    uint64_t s = (t >= 0) ? ld_volatile_u64(&states[t]) : kLbInclusive;
    while (__any_sync(0xffffffffu, (s >> 62) == 0)) {
      if ((s >> 62) == 0) s = ld_volatile_u64(&states[t]);
    }
    const uint32_t incl = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    if (incl) {
      const int first = __ffs(incl) - 1;
      uint64_t v = ((int)lane <= first) ? (s & kLbValueMask) : 0;
      excl += warp_sum(v);
      break;
    }
    excl += warp_sum(s & kLbValueMask);
    pred -= 32;
  }
  if (lane == 0) st_volatile_u64(&states[tile], kLbInclusive | (excl + aggregate));
  return excl;
}

// Block-wide stable compaction offsets for two predicates (a, b) of the
// element this thread owns.  Returns global exclusive offsets and, for the
// whole tile, the inclusive totals (valid in every thread).  smem must hold
// 2*32 u32 + 4 u64.  blockDim.x must be a multiple of 32.
struct PairScan {
  uint32_t a_off, b_off;    // this element's output positions
  uint64_t a_total, b_total;  // inclusive totals through this tile
};

__device__ __forceinline__ PairScan block_pair_scan(bool a, bool b, uint64_t* states, int64_t tile,
                                                    uint32_t* s_warp /*[64]*/,
                                                    uint64_t* s_misc /*[4]*/) {
  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t nwarps = blockDim.x >> 5;
  const uint32_t ma = __ballot_sync(0xffffffffu, a);
  const uint32_t mb = __ballot_sync(0xffffffffu, b);
  if (lane == 0) {
    s_warp[warp] = __popc(ma);
    s_warp[32 + warp] = __popc(mb);
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t ca = lane < nwarps ? s_warp[lane] : 0;
    uint32_t cb = lane < nwarps ? s_warp[32 + lane] : 0;
    // inclusive warp scan over per-warp counts
    uint32_t ia = ca, ib = cb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t xa = __shfl_up_sync(0xffffffffu, ia, o);
      uint32_t xb = __shfl_up_sync(0xffffffffu, ib, o);
      if ((int)lane >= o) {
        ia += xa;
        ib += xb;
      }
    }
    const uint32_t ta = __shfl_sync(0xffffffffu, ia, 31);
    const uint32_t tb = __shfl_sync(0xffffffffu, ib, 31);
    if (lane < nwarps) {
      s_warp[lane] = ia - ca;  // exclusive per-warp offsets
      s_warp[32 + lane] = ib - cb;
    }
    const uint64_t agg = (uint64_t)ta | ((uint64_t)tb << 31);
    // states == nullptr: a single-tile launch, nothing before it
    const uint64_t excl = states ? lookback_exclusive(states, tile, agg) : 0;
    if (lane == 0) {
      s_misc[0] = excl & kLbFieldMask;
      s_misc[1] = (excl >> 31) & kLbFieldMask;
      s_misc[2] = (excl & kLbFieldMask) + ta;
      s_misc[3] = ((excl >> 31) & kLbFieldMask) + tb;
    }
  }
  __syncthreads();
  PairScan r;
  const uint32_t lt = lanemask_lt();
  r.a_off = (uint32_t)s_misc[0] + s_warp[warp] + __popc(ma & lt);
  r.b_off = (uint32_t)s_misc[1] + s_warp[32 + warp] + __popc(mb & lt);
  r.a_total = s_misc[2];
  r.b_total = s_misc[3];
  return r;
}

// Dynamic tile id (guarantees every predecessor tile has started, so the
// look-back cannot deadlock).  One thread takes it, the block reads it.
// counter == nullptr: a single-tile launch (tile 0, no workspace).
__device__ __forceinline__ int64_t next_tile_id(unsigned long long* counter, int64_t* s_tile) {
  if (counter == nullptr) return 0;
  if (threadIdx.x == 0) *s_tile = (int64_t)atomicAdd(counter, 1ull);
  __syncthreads();
  return *s_tile;
}

}  // namespace gs
