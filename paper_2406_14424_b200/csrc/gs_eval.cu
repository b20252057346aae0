// gs_eval.cu — list path: the drop-in for kernels.evaluate_encoded.
//
// Reference: /root/reference/pkg/src/gearserve/kernels.py:39-62
// (_evaluate_numba) and :93-108 (evaluate_encoded).  For every encoded
// cascade c and every record r the reference walks stages s = 0..ns-1,
// counts the visit (forward_frac[c, s] += 1) and stops at the first stage
// with s == ns-1 or certainty[r, m] >= thresholds[c, s], adding
// correct[r, m].  The epilogue divides the counts by n_rec and accumulates
// mean_cost in stage order without FMA.
//
// B200 mapping: one thread owns one cascade; a CTA owns 128 cascades and
// streams a contiguous range of records through shared memory in tiles
// staged by 1-D TMA bulk copies (cp.async.bulk + mbarrier, 3-stage ring).
// All threads of a CTA read the same record at the same time, so the tile
// reads are shared-memory broadcasts.  Counts are integers in registers and
// are merged across record splits with u32 atomics (exact, order-free); a
// finalize kernel does the f64 epilogue in the reference's order.
#include <algorithm>
#include <atomic>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int kEvalThreads = 128;
constexpr int kEvalStages = 3;
constexpr int kEvalStageBytes = 24 * 1024;  // cert+corr bytes per stage (max)

struct EvalArgs {
  const double* cert;
  const uint8_t* corr;
  int64_t n_rec;
  int32_t n_models;
  const int32_t* stage_model;
  const double* thr;
  const int32_t* n_stages;
  int64_t n_casc;
  int32_t max_len;
  uint32_t* counts;  // [n_casc][max_len + 1]: [s] reach of stage s (s>=1), [max_len] correct
  int64_t rec_per_split;
  int32_t tile;      // records per smem tile (multiple of 16)
  int32_t use_tma;
};

template <int MAXL>
__global__ void __launch_bounds__(kEvalThreads) eval_list_kernel(EvalArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kEvalStages];

  const int M = a.n_models;
  const int tile = a.tile;
  double* s_cert = reinterpret_cast<double*>(smem);  // [stages][tile*M]
  uint8_t* s_corr = smem + (size_t)kEvalStages * tile * M * sizeof(double);

  const int64_t c = (int64_t)blockIdx.x * kEvalThreads + threadIdx.x;
  const bool active = c < a.n_casc;

  int ns = 0;
  int sm[MAXL];
  double th[MAXL];
  uint32_t reach[MAXL];
#pragma unroll
  for (int s = 0; s < MAXL; ++s) {
    sm[s] = 0;
    th[s] = 0.0;
    reach[s] = 0;
  }
  if (active) {
    ns = a.n_stages[c];
    ns = ns < 0 ? 0 : (ns > a.max_len ? a.max_len : ns);
#pragma unroll
    for (int s = 0; s < MAXL; ++s) {
      if (s < ns) {
        int m = a.stage_model[c * a.max_len + s];
        if (m < 0 || m >= M) {  // malformed: host validates; never read OOB
          ns = s;
          break;
        }
        sm[s] = m;
        th[s] = a.thr[c * a.max_len + s];
      }
    }
  }
  uint32_t correct = 0;

  const int64_t r_begin = (int64_t)blockIdx.y * a.rec_per_split;
  const int64_t r_end = min(a.n_rec, r_begin + a.rec_per_split);
  if (r_begin >= r_end) return;
  const int ntiles = (int)((r_end - r_begin + tile - 1) / tile);

  auto tile_rows = [&](int i) -> int {
    int64_t r0 = r_begin + (int64_t)i * tile;
    return (int)min((int64_t)tile, r_end - r0);
  };
  auto tma_ok = [&](int i) -> bool {
    const int rows = tile_rows(i);
    return a.use_tma && ((rows * M) % 16 == 0);
  };
  auto issue = [&](int i) {
    const int st = i % kEvalStages;
    const int rows = tile_rows(i);
    const int64_t r0 = r_begin + (int64_t)i * tile;
    const uint32_t cb = (uint32_t)rows * M * sizeof(double);
    const uint32_t kb = (uint32_t)rows * M;
    fence_proxy_async();
    mbar_arrive_expect_tx(&bars[st], cb + kb);
    bulk_g2s(s_cert + (size_t)st * tile * M, a.cert + r0 * M, cb, &bars[st]);
    bulk_g2s(s_corr + (size_t)st * tile * M, a.corr + r0 * M, kb, &bars[st]);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kEvalStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kEvalStages && i < ntiles; ++i)
      if (tma_ok(i)) issue(i);
  }

  for (int i = 0; i < ntiles; ++i) {
    const int st = i % kEvalStages;
    const int rows = tile_rows(i);
    const double* tc = s_cert + (size_t)st * tile * M;
    const uint8_t* tk = s_corr + (size_t)st * tile * M;
    if (tma_ok(i)) {
      mbar_wait(&bars[st], (uint32_t)((i / kEvalStages) & 1));
    } else {
      // unaligned base or ragged last tile: cooperative copy
      const int64_t r0 = r_begin + (int64_t)i * tile;
      double* dc = s_cert + (size_t)st * tile * M;
      uint8_t* dk = s_corr + (size_t)st * tile * M;
      for (int j = threadIdx.x; j < rows * M; j += blockDim.x) {
        dc[j] = a.cert[r0 * M + j];
        dk[j] = a.corr[r0 * M + j];
      }
      __syncthreads();
    }
    if (active && ns > 0) {
      if (MAXL <= 4) {
        // branch-free: every stage's certainty is loaded at once (the loads
        // do not wait on the stop decisions) and the first stopping stage
        // picked by predicated selects; stages s >= ns - 1 compare against
        // NaN (never true: the last stage always stops).  The select picks
        // the stop stage's model and its count increment: the records
        // stopping at stage t >= 1 are counted in 10-bit field t - 1 of one
        // word (flushed to the reach counts per tile, <= 256 records) --
        // reach[s] is the suffix sum of those fields
        double tq[MAXL];
        uint32_t inc_s[MAXL];
#pragma unroll
        for (int s = 0; s < MAXL; ++s) {
          tq[s] = s < ns - 1 ? th[s] : __longlong_as_double(0x7ff8000000000000ll);
          inc_s[s] = s == 0 ? 0u : 1u << (10 * (s - 1));
        }
        uint32_t inc_last = inc_s[0], m_last = (uint32_t)sm[0];
#pragma unroll
        for (int s = 1; s < MAXL; ++s)
          if (s == ns - 1) {
            inc_last = inc_s[s];
            m_last = (uint32_t)sm[s];
          }
        uint32_t stops = 0;
#pragma unroll 4
        for (int r = 0; r < rows; ++r) {
          const double* crow = tc + r * M;
          const uint8_t* krow = tk + r * M;
          double v[MAXL];
#pragma unroll
          for (int s = 0; s < MAXL - 1; ++s) v[s] = crow[sm[s]];  // sm[s] = 0 past ns: a valid read
          uint32_t inc = inc_last, m = m_last;
#pragma unroll
          for (int s = MAXL - 2; s >= 0; --s)
            if (v[s] >= tq[s]) {
              inc = inc_s[s];
              m = (uint32_t)sm[s];
            }
          stops += inc;
          correct += krow[m];
        }
        uint32_t above = 0;
#pragma unroll
        for (int s = MAXL - 1; s >= 1; --s) {
          above += (stops >> (10 * (s - 1))) & 1023u;
          reach[s] += above;
        }
      } else if (MAXL <= 8) {
        // as above with per-stage counters (eight stages do not fit one word)
#pragma unroll 2
        for (int r = 0; r < rows; ++r) {
          const double* crow = tc + r * M;
          const uint8_t* krow = tk + r * M;
          double v[MAXL];
#pragma unroll
          for (int s = 0; s < MAXL; ++s) v[s] = crow[sm[s]];  // sm[s] = 0 past ns: a valid read
          int stop = ns - 1, m = sm[0];
#pragma unroll
          for (int s = MAXL - 2; s >= 0; --s)
            if (s < ns - 1 && v[s] >= th[s]) stop = s;
#pragma unroll
          for (int s = 1; s < MAXL; ++s) {
            reach[s] += s <= stop ? 1u : 0u;
            m = s == stop ? sm[s] : m;
          }
          correct += krow[m];
        }
      } else {
        for (int r = 0; r < rows; ++r) {
          const double* crow = tc + r * M;
          const uint8_t* krow = tk + r * M;
#pragma unroll
          for (int s = 0; s < MAXL; ++s) {
            if (s >= ns) break;
            const int m = sm[s];
            if (s == ns - 1 || crow[m] >= th[s]) {
              correct += krow[m];
              break;
            }
            if (s + 1 < MAXL) reach[s + 1] += 1;
          }
        }
      }
    }
    __syncthreads();  // every thread is done with stage st
    if (threadIdx.x == 0 && i + kEvalStages < ntiles && tma_ok(i + kEvalStages))
      issue(i + kEvalStages);
  }

  if (active) {
    uint32_t* out = a.counts + c * (a.max_len + 1);
#pragma unroll
    for (int s = 1; s < MAXL; ++s)
      if (s < ns - 0 && reach[s]) atomicAdd(out + s, reach[s]);
    if (correct) atomicAdd(out + a.max_len, correct);
  }
}

__global__ void eval_finalize_kernel(const uint32_t* counts, const int32_t* stage_model,
                                     const int32_t* n_stages, int64_t n_casc, int32_t max_len,
                                     int32_t n_models, int64_t n_rec, const double* cost1,
                                     double* accuracy, double* mean_cost, double* forward_frac) {
  const double n = (double)n_rec;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_casc;
       c += (int64_t)gridDim.x * blockDim.x) {
    int ns = n_stages[c];
    ns = ns < 0 ? 0 : (ns > max_len ? max_len : ns);
    const uint32_t* cnt = counts + c * (max_len + 1);
    double mean = 0.0;
    bool valid = true;
    for (int s = 0; s < max_len; ++s) {
      double frac = 0.0;
      if (s < ns && valid) {
        const int m = stage_model[c * max_len + s];
        if (m < 0 || m >= n_models) {
          valid = false;
        } else {
          const double visits = s == 0 ? n : (double)cnt[s];
          frac = ddiv(visits, n);
          mean = dadd(mean, dmul(frac, cost1[m]));
        }
      }
      forward_frac[c * max_len + s] = frac;
    }
    mean_cost[c] = mean;
    accuracy[c] = ddiv((double)cnt[max_len], n);
  }
}

template <int MAXL>
cudaError_t launch_eval(const EvalArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  auto k = eval_list_kernel<MAXL>;
  static SmemAttr smem_set;
  cudaError_t e = ensure_smem(k, smem_set, smem);
  if (e != cudaSuccess) return e;
  k<<<grid, kEvalThreads, smem, st>>>(a);
  return cudaGetLastError();
}

size_t eval_counts_bytes(int64_t n_casc, int32_t max_len) {
  return round_up((size_t)n_casc * (max_len + 1) * sizeof(uint32_t), 256);
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" int gs_eval_encoded_workspace(int64_t n_rec, int32_t n_models, int64_t n_casc,
                                         int32_t max_len, size_t* bytes) {
  GS_REQUIRE(bytes && n_rec >= 0 && n_models >= 1 && n_casc >= 0 && max_len >= 0);
  *bytes = eval_counts_bytes(n_casc, max_len);
  return GS_OK;
}

extern "C" int gs_eval_encoded(const double* certainty, const uint8_t* correct, int64_t n_rec,
                               int32_t n_models, const int32_t* stage_model,
                               const double* thresholds, const int32_t* n_stages, int64_t n_casc,
                               int32_t max_len, const double* cost1, double* accuracy,
                               double* mean_cost, double* forward_frac, void* workspace,
                               size_t workspace_bytes, void* stream) {
  GS_REQUIRE(n_models >= 1 && n_casc >= 0 && max_len >= 0);
  if (n_casc == 0) return GS_OK;
  GS_REQUIRE(n_rec >= 1 && max_len >= 1);
  if (max_len > GS_MAX_STAGES || n_rec >= (int64_t)UINT32_MAX) return GS_EUNSUPPORTED;
  GS_REQUIRE(certainty && correct && stage_model && thresholds && n_stages && cost1 && accuracy &&
             mean_cost && forward_frac);
  const size_t need = eval_counts_bytes(n_casc, max_len);
  if (!workspace || workspace_bytes < need) return GS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t* counts = static_cast<uint32_t*>(workspace);
  GS_CUDA_TRY(cudaMemsetAsync(counts, 0, need, st));

  // records per smem tile: multiple of 16, cert+corr bytes per stage bounded
  int tile = kEvalStageBytes / (9 * n_models);
  tile = std::max(16, std::min(256, tile / 16 * 16));
  const size_t smem = (size_t)kEvalStages * tile * n_models * 9;
  if (smem > 200 * 1024) return GS_EUNSUPPORTED;

  const int64_t blocks_x = (n_casc + kEvalThreads - 1) / kEvalThreads;
  if (blocks_x > 0x7fffffff) return GS_EUNSUPPORTED;
  const int64_t target = (int64_t)sm_count() * 8;
  const int64_t max_splits = (n_rec + tile - 1) / tile;
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>((target + blocks_x - 1) / blocks_x, max_splits));
  splits = std::min<int64_t>(splits, 65535);
  int64_t per = (n_rec + splits - 1) / splits;
  per = (per + tile - 1) / tile * tile;
  splits = (n_rec + per - 1) / per;

  EvalArgs a;
  a.cert = certainty;
  a.corr = correct;
  a.n_rec = n_rec;
  a.n_models = n_models;
  a.stage_model = stage_model;
  a.thr = thresholds;
  a.n_stages = n_stages;
  a.n_casc = n_casc;
  a.max_len = max_len;
  a.counts = counts;
  a.rec_per_split = per;
  a.tile = tile;
  a.use_tma = aligned16(certainty) && aligned16(correct);

  dim3 grid((unsigned)blocks_x, (unsigned)splits);
  cudaError_t e;
  if (max_len <= 2)
    e = launch_eval<2>(a, grid, smem, st);
  else if (max_len <= 4)
    e = launch_eval<4>(a, grid, smem, st);
  else if (max_len <= 8)
    e = launch_eval<8>(a, grid, smem, st);
  else if (max_len <= 16)
    e = launch_eval<16>(a, grid, smem, st);
  else if (max_len <= 32)
    e = launch_eval<32>(a, grid, smem, st);  // 17+ stage cascades: rare, per-thread arrays spill
  else
    e = launch_eval<64>(a, grid, smem, st);
  GS_CUDA_TRY(e);

  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n_casc + threads - 1) / threads, (int64_t)sm_count() * 16);
  eval_finalize_kernel<<<(unsigned)blocks, threads, 0, st>>>(counts, stage_model, n_stages, n_casc,
                                                             max_len, n_models, n_rec, cost1,
                                                             accuracy, mean_cost, forward_frac);
  GS_LAUNCH_CHECK();
  return GS_OK;
}
