// gs_sampler.cu — SP1's cascade sampler on the device.
//
// Reference: cascades.sample_cascades (src/cascades.py:166-193), called by
// planner.sp1_search_cascades with seed = seed + calls - 1
// (src/planner.py:374-375).  The sampler is one sequential stream of
// variable-length draws from numpy's default_rng(seed), so a job (one seed)
// is one thread; many seeds (SP1 calls, tenants) run per launch, one warp
// each.  The draws are numpy's, reproduced exactly (PCG64 + the bit
// generator's buffered 32-bit half, see gs_engine.cu):
//   k     = rng.integers(1, M + 1)                 Lemire on [0, M - 1]
//   pick  = rng.choice(M, size=k, replace=False)   Floyd's algorithm
//           (Lemire on [0, j] for j = M-k .. M-1) then a Fisher-Yates
//           shuffle of the k picks (Lemire on [0, i], i = k-1 .. 1)
//   thr_s = rng.choice(grid[m_s])                  Lemire on [0, len - 1]
// Stages are the picks sorted (cost ranks); duplicates are dropped in order
// against every cascade seen so far, singletons included (`seen`), with an
// open-addressing hash set of (stage mask, threshold grid indices).
// Outputs are the encoded cascades evaluate_encoded takes, plus each
// stage's grid index (a sampled cascade IS a grid-product config, so the
// full-grid sweep's outputs can be gathered for it instead of walking).
#include "gs_common.cuh"

namespace gs {
namespace {

struct Pcg64s {
  unsigned __int128 state, inc;
  uint32_t has32, u32;
  __device__ uint64_t next64() {
    const unsigned __int128 mult =
        ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    state = state * mult + inc;
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const uint32_t rot = (uint32_t)(state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t n = next64();
    has32 = 1;
    u32 = (uint32_t)(n >> 32);
    return (uint32_t)n;
  }
  // numpy buffered_bounded_lemire_uint32 on [0, rng]; rng == 0 draws nothing
  __device__ uint32_t bounded(uint32_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return next32();
    const uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)next32() * excl;
    if ((uint32_t)m < excl) {
      const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
      while ((uint32_t)m < thr) m = (uint64_t)next32() * excl;
    }
    return (uint32_t)(m >> 32);
  }
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// insert (lo, hi) into the set; true if it was not there.  lo != 0 always
// (the stage mask is in its low 16 bits and never empty).
__device__ bool set_insert(uint64_t* table, int64_t cap, uint64_t lo, uint64_t hi) {
  int64_t slot = (int64_t)(mix64(lo ^ mix64(hi)) & (uint64_t)(cap - 1));
  while (true) {
    uint64_t* e = table + 2 * slot;
    if (e[0] == 0) {
      e[0] = lo;
      e[1] = hi;
      return true;
    }
    if (e[0] == lo && e[1] == hi) return false;
    slot = (slot + 1) & (cap - 1);
  }
}

struct SamplerArgs {
  int32_t M;
  const int32_t* order;      // [M] model column of cost rank r
  const double* grid;        // concatenated grids, by model column
  const int32_t* grid_off;   // [M + 1]
};

__global__ void __launch_bounds__(32) sampler_kernel(SamplerArgs a, const gs_sampler_job* jobs, int n_jobs) {
  if (blockIdx.x >= (unsigned)n_jobs || threadIdx.x != 0) return;
  const gs_sampler_job job = jobs[blockIdx.x];
  const int M = a.M;
  Pcg64s rng;
  rng.state = ((unsigned __int128)job.rng_state_hi << 64) | job.rng_state_lo;
  rng.inc = ((unsigned __int128)job.rng_inc_hi << 64) | job.rng_inc_lo;
  rng.has32 = job.rng_has_uint32;
  rng.u32 = job.rng_uinteger;
  int64_t count = 0;
  auto emit = [&](uint32_t mask, const int32_t* ranks, int k, const uint32_t* gidx) {
    int32_t* sm = job.stage_model + count * M;
    double* th = job.thresholds + count * M;
    int32_t* gi = job.grid_index + count * M;
    for (int s = 0; s < M; ++s) {
      if (s < k) {
        const int col = a.order[ranks[s]];
        sm[s] = col;
        if (s < k - 1) {
          th[s] = a.grid[a.grid_off[col] + gidx[s]];
          gi[s] = (int32_t)gidx[s];
        } else {
          th[s] = 0.0;
          gi[s] = -1;
        }
      } else {
        sm[s] = -1;
        th[s] = 0.0;
        gi[s] = -1;
      }
    }
    job.n_stages[count] = k;
    count += 1;
    (void)mask;
  };
  // every singleton first, cheap to expensive (all distinct)
  for (int r = 0; r < M; ++r) {
    const int32_t ranks[1] = {r};
    const uint32_t none[1] = {0};
    set_insert(job.table, job.table_cap, 1ull << r, 0);
    emit(1u << r, ranks, 1, none);
  }
  int64_t pick[GS_MAX_MODELS];
  for (int64_t it = 0; it < job.n_samples; ++it) {
    const int k = 1 + (int)rng.bounded((uint32_t)(M - 1));
    // Floyd's algorithm over j = M-k .. M-1 (the hash set is tiny: bits)
    uint32_t taken = 0;
    for (int j = M - k; j < M; ++j) {
      const uint32_t v = rng.bounded((uint32_t)j);
      if (!(taken >> v & 1u)) {
        taken |= 1u << v;
        pick[j - (M - k)] = v;
      } else {
        taken |= 1u << j;
        pick[j - (M - k)] = j;
      }
    }
    for (int i = k - 1; i >= 1; --i) {  // the shuffle: consumes draws, order irrelevant after sort
      const uint32_t jj = rng.bounded((uint32_t)i);
      const int64_t t = pick[jj];
      pick[jj] = pick[i];
      pick[i] = t;
    }
    // stages = sorted picks (cost ranks ascending) = set bits of `taken`
    int32_t ranks[GS_MAX_MODELS];
    int n = 0;
    for (int r = 0; r < M; ++r)
      if (taken >> r & 1u) ranks[n++] = r;
    uint32_t gidx[GS_MAX_MODELS];
    uint64_t lo = taken, hi = 0;
    for (int s = 0; s < k - 1; ++s) {
      const int col = a.order[ranks[s]];
      const int32_t len = a.grid_off[col + 1] - a.grid_off[col];
      gidx[s] = rng.bounded((uint32_t)(len - 1));
      const uint64_t g = gidx[s];
      if (s < 3) lo |= g << (16 * (s + 1));
      else hi |= g << (16 * (s - 3));
    }
    if (set_insert(job.table, job.table_cap, lo, hi)) emit(taken, ranks, k, gidx);
  }
  job.result[0] = count;
  job.result[1] = (int64_t)(uint64_t)(rng.state >> 64);
  job.result[2] = (int64_t)(uint64_t)rng.state;
  job.result[3] = rng.has32;
  job.result[4] = rng.u32;
}

}  // namespace
}  // namespace gs

extern "C" int gs_sample_cascades(int32_t n_models, const int32_t* order, const double* grids,
                                  const int32_t* grid_off, const gs_sampler_job* jobs,
                                  int32_t n_jobs, void* stream) {
  GS_REQUIRE(n_models >= 1 && n_jobs >= 0);
  if (n_models > GS_MAX_MODELS) return GS_EUNSUPPORTED;
  if (n_jobs == 0) return GS_OK;
  GS_REQUIRE(order && grids && grid_off && jobs);
  gs::SamplerArgs a{n_models, order, grids, grid_off};
  gs::sampler_kernel<<<(unsigned)n_jobs, 32, 0, static_cast<cudaStream_t>(stream)>>>(a, jobs, n_jobs);
  GS_LAUNCH_CHECK();
  return GS_OK;
}
