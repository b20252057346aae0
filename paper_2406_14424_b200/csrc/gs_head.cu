// gs_head.cu — a cascade stage's classifier head on the 5th-generation tensor
// cores, fused with the stage step's certainty (north_star: "Tensor cores are
// used only for the dense classifier GEMMs inside each cascade model").
//
// The reference has no GPU model code: its stage runs a model and then
// cascades.certainty over the scores (src/serving.py:79-97 mock_execute,
// src/cascades.py:20-28).  Here one kernel takes the stage's features
// [B, K] (bf16) and the head's weight [N, K] (bf16, nn.Linear layout) and
// returns each row's certainty without writing the logits to HBM:
//
//   logits = features @ weight^T (+ bias)     tcgen05.mma kind::f16, f32 in TMEM
//   certainty per row over the N classes      online in the epilogue:
//     MARGIN       top1 - top2 of the logits (the reference's Eq. 5 on scores)
//     MAX_SOFTMAX  max_i softmax(x)_i = 1 / sum_i exp(x_i - max)
//     ENTROPY      1 - H(softmax(x)) / ln N
//
// A persistent CTA per SM takes 128-row tiles in turn and walks each tile's
// classes in chunks of 256 (UMMA M = 128, N = 256, K = 16): warp 0 streams
// 128 x 64 feature tiles and 256 x 64 weight tiles through a 4-stage
// shared-memory ring with TMA (128-byte swizzle, the layout the UMMA
// descriptors name); one thread of warp 1 issues the MMAs into one of two
// 256-column TMEM accumulators, alternating across chunks and tiles; eight
// epilogue warps (two per TMEM lane quadrant, a row per thread, half of a
// chunk's columns each) read the other accumulator with tcgen05.ld while the
// next chunk is multiplied, and fold its logits into the row's running max /
// sum of 2^(y - max) / entropy sum (ex2 on the MUFU, base-2 domain); the two
// halves of a row meet in shared memory at the end of its tile.
// Logits can optionally be stored (f32) for checking.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kHM = 128, kHN = 256, kHK = 64, kHUK = 16;
constexpr int kHStages = 4;
constexpr int kHEpiWarps = 8;   // two per TMEM lane quadrant, each half of a chunk's columns
constexpr int kHThreads = 64 + 32 * kHEpiWarps;  // warp 0 TMA, warp 1 MMA (+ TMEM owner), then the epilogue
constexpr uint32_t kHABytes = kHM * kHK * 2, kHBBytes = kHN * kHK * 2;
constexpr int kHBiasSmem = 4096;  // bias staged in shared memory up to this many classes
constexpr size_t kHSmem = 1024 + (size_t)kHStages * (kHABytes + kHBBytes) + kHBiasSmem * 4;  // + 1 KB alignment slack

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// K-major operand tile, 128-byte swizzle: rows of 64 bf16 (128 B), 8-row
// groups 1024 B apart (SBO), LBO unused (1), descriptor version 1.
__device__ __forceinline__ uint64_t smem_desc(const void* tile) {
  const uint64_t addr = (smem_u32(tile) & 0x3FFFFu) >> 4;
  return addr | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// kind::f16 instruction descriptor: f32 accumulate, bf16 A and B, both
// K-major, N >> 3 at bit 17, M >> 4 at bit 24.
constexpr uint32_t kHIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kHN >> 3) << 17) |
                             ((uint32_t)(kHM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kHIdesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 32 consecutive f32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t addr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
      "[%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct HeadArgs {
  int64_t B;
  int32_t N, K, kind;
  const float* bias;  // [N] or null
  double* cert;       // [B]
  float* logits;      // [B, N] or null
};

// Running certainty state of one row (half of its columns), in base 2:
// y = x log2(e), m = max y, s = sum 2^(y - m), t = sum (y - m) 2^(y - m).
struct RowStats {
  float m, s, t;
  float top1, top2;  // margin: the two largest logits
};
constexpr float kLog2e = 1.4426950408889634f;
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// fold (m2, s2, t2) into (m, s, t): both rescaled to the larger max
__device__ __forceinline__ void merge_stats(RowStats& a, const RowStats& b) {
  const float m = fmaxf(a.m, b.m);
  float s = 0.f, t = 0.f;
  if (a.s > 0.f) {
    const float d = a.m - m, e = ex2(d);
    s += e * a.s;
    t += e * fmaf(d, a.s, a.t);
  }
  if (b.s > 0.f) {
    const float d = b.m - m, e = ex2(d);
    s += e * b.s;
    t += e * fmaf(d, b.s, b.t);
  }
  a.m = m;
  a.s = s;
  a.t = t;
  const float hi = fmaxf(a.top1, b.top1), lo = fminf(a.top1, b.top1);
  a.top2 = fmaxf(lo, fmaxf(a.top2, b.top2));
  a.top1 = hi;
}

__global__ void __launch_bounds__(kHThreads, 1) head_certainty_kernel(const __grid_constant__ CUtensorMap map_a,
                                                                       const __grid_constant__ CUtensorMap map_b,
                                                                       const __grid_constant__ HeadArgs a) {
  extern __shared__ uint8_t s_raw[];
  __shared__ __align__(8) uint64_t full[kHStages], empty[kHStages], tfull[2], tempty[2];
  __shared__ uint32_t s_tmem;
  __shared__ RowStats s_half[2][kHM];  // the second column half's row stats, merged per tile
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(s_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* s_a = base;                                // [stages][128 x 64] bf16, swizzled
  uint8_t* s_b = base + (size_t)kHStages * kHABytes;  // [stages][256 x 64] bf16, swizzled
  float* s_bias = reinterpret_cast<float*>(s_b + (size_t)kHStages * kHBBytes);  // [N] when N <= kHBiasSmem
  const bool bias_smem = a.bias && a.N <= kHBiasSmem;
  if (bias_smem)
    for (int i = threadIdx.x; i < a.N; i += blockDim.x) s_bias[i] = a.bias[i];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = (a.B + kHM - 1) / kHM;  // persistent: tiles blockIdx.x, += gridDim.x
  const int n_chunks = (a.N + kHN - 1) / kHN, n_k = a.K / kHK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kHStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kHEpiWarps);  // one arrival per epilogue warp
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
  }
  if (warp == 1) {  // 512 columns: two 256-column accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
      for (int c = 0; c < n_chunks; ++c)
        for (int kb = 0; kb < n_k; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], kHABytes + kHBBytes);
          tma_load_2d(s_a + (size_t)s * kHABytes, &map_a, kb * kHK, (int)(tile * kHM), &full[s]);
          tma_load_2d(s_b + (size_t)s * kHBBytes, &map_b, kb * kHK, c * kHN, &full[s]);
          if (++s == kHStages) {
            s = 0;
            ph ^= 1;
          }
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int s = 0;
      uint32_t ph = 0;
      uint32_t it = 0;  // accumulator uses, across tiles
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
      for (int c = 0; c < n_chunks; ++c, ++it) {
        const int buf = it & 1;
        mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);  // the epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * kHN);
        for (int kb = 0; kb < n_k; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t da = smem_desc(s_a + (size_t)s * kHABytes);
          const uint64_t db = smem_desc(s_b + (size_t)s * kHBBytes);
#pragma unroll
          for (int k = 0; k < kHK / kHUK; ++k)  // +32 bytes along K inside the swizzled rows
            mma_bf16(d, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), (kb | k) != 0);
          mma_commit(&empty[s]);  // the smem slot is free once these MMAs have read it
          if (++s == kHStages) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(&tfull[buf]);  // the accumulator is complete
      }
    }
  } else {  // epilogue: TMEM lane quadrant warp % 4 (a row per thread), column half h
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t r = tile * kHM + row;
    RowStats st{-INFINITY, 0.f, 0.f, -INFINITY, -INFINITY};
    for (int c = 0; c < n_chunks; ++c, ++it) {
      const int buf = it & 1;
      mbar_wait(&tfull[buf], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int g = h * (kHN / 64); g < (h + 1) * (kHN / 64); ++g) {
        const int col0 = c * kHN + g * 32;
        if (col0 >= a.N) break;  // warp-uniform
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kHN + g * 32), v);
        const bool full = col0 + 32 <= a.N;  // warp-uniform: only the last group is ragged
        if (a.bias) {
          if (bias_smem) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              if (full || col0 + i + 3 < a.N) {
                const float4 b4 = *reinterpret_cast<const float4*>(s_bias + col0 + i);
                v[i] += b4.x;
                v[i + 1] += b4.y;
                v[i + 2] += b4.z;
                v[i + 3] += b4.w;
              } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  if (col0 + i + j < a.N) v[i + j] += s_bias[col0 + i + j];
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < a.N) v[i] += __ldg(a.bias + col0 + i);
          }
        }
        if (!full) {  // padding classes never count
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (col0 + i >= a.N) v[i] = -INFINITY;
        }
        if (a.logits && r < a.B) {
          float* out = a.logits + r * (int64_t)a.N + col0;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (col0 + i < a.N) out[i] = v[i];
        }
        if (a.kind == GS_CERT_MARGIN) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = v[i];
            const float lo = fminf(x, st.top1);
            st.top1 = fmaxf(x, st.top1);
            st.top2 = fmaxf(st.top2, lo);
          }
          continue;
        }
        // max by a tree, then four independent (s, t) chains: the FADD / FFMA
        // latencies of one row's 32 terms overlap instead of queueing
        float mx[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) mx[j] = fmaxf(fmaxf(v[j], v[j + 8]), fmaxf(v[j + 16], v[j + 24]));
#pragma unroll
        for (int j = 0; j < 4; ++j) mx[j] = fmaxf(mx[j], mx[j + 4]);
        const float ly = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * kLog2e;
        if (ly > st.m) {  // rescale the running sums to the new max
          if (st.s > 0.f) {
            const float d = st.m - ly, e = ex2(d);
            st.t = e * fmaf(d, st.s, st.t);
            st.s = e * st.s;
          }
          st.m = ly;
        }
        float ps[4] = {0.f, 0.f, 0.f, 0.f}, pt[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float d = fmaf(v[i], kLog2e, -st.m), e = ex2(d);  // -inf padding: e = 0
          ps[i & 3] += e;
          pt[i & 3] = fmaf(e > 0.f ? d : 0.f, e, pt[i & 3]);
        }
        st.s += (ps[0] + ps[1]) + (ps[2] + ps[3]);
        st.t += (pt[0] + pt[1]) + (pt[2] + pt[3]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
    // the two column halves of each row meet in shared memory (double
    // buffered by tile: the halves pass this barrier once per tile together)
    RowStats* half = s_half[((tile - blockIdx.x) / gridDim.x) & 1];
    if (h == 1) half[row] = st;
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kHEpiWarps) : "memory");
    if (h == 0 && r < a.B) {
      merge_stats(st, half[row]);
      double cert;
      if (a.kind == GS_CERT_MARGIN) {
        cert = a.N > 1 ? (double)st.top1 - (double)st.top2 : (double)st.top1;
      } else if (a.kind == GS_CERT_MAX_SOFTMAX) {
        cert = 1.0 / (double)st.s;
      } else {  // 1 - H / ln N, H = ln S - T / S = ln 2 (log2 s - t / s)
        const double H = 0.6931471805599453 * (log2((double)st.s) - (double)st.t / (double)st.s);
        cert = a.N > 1 ? 1.0 - H / log((double)a.N) : 1.0;
      }
      a.cert[r] = cert;
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Row-major [rows, K] bf16 tensor map with a 64 x box_rows box, 128-byte swizzle.
int make_map(CUtensorMap* map, const void* ptr, int64_t rows, int32_t K, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return GS_ECUDA;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kHK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return rc == CUDA_SUCCESS ? GS_OK : GS_EINVAL;
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" int gs_head_certainty(const void* features, const void* weight, const float* bias, int64_t n_rows,
                                 int32_t n_cls, int32_t n_feat, int32_t kind, double* cert_out,
                                 float* logits_out, void* stream) {
  GS_REQUIRE(features && weight && cert_out && n_rows >= 0 && n_cls >= 1 && n_feat >= kHK);
  GS_REQUIRE(kind == GS_CERT_MARGIN || kind == GS_CERT_MAX_SOFTMAX || kind == GS_CERT_ENTROPY);
  if (n_feat % kHK != 0 || n_rows >= (1ll << 31) || n_cls > (1 << 20)) return GS_EUNSUPPORTED;
  // TMA: 16-byte aligned bases (row pitch 2 K bytes is a multiple of 128)
  if ((reinterpret_cast<uintptr_t>(features) & 15u) || (reinterpret_cast<uintptr_t>(weight) & 15u))
    return GS_EINVAL;
  if (n_rows == 0) return GS_OK;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, features, n_rows, n_feat, kHM);
  if (rc != GS_OK) return rc;
  if ((rc = make_map(&mb, weight, n_cls, n_feat, kHN)) != GS_OK) return rc;
  HeadArgs a{};
  a.B = n_rows;
  a.N = n_cls;
  a.K = n_feat;
  a.kind = kind;
  a.bias = bias;
  a.cert = cert_out;
  a.logits = logits_out;
  static SmemAttr attr;
  GS_CUDA_TRY(ensure_smem(head_certainty_kernel, attr, kHSmem));
  const unsigned grid = (unsigned)std::min<int64_t>((n_rows + kHM - 1) / kHM, sm_count());
  head_certainty_kernel<<<grid, kHThreads, kHSmem, static_cast<cudaStream_t>(stream)>>>(ma, mb, a);
  GS_LAUNCH_CHECK();
  return GS_OK;
}
