// gs_engine.cu — the serving engine's virtual-clock event loop on the device.
//
// Reference: gearserve.engine.run (src/engine.py:452-520) driving
// EngineState (src/engine.py:267-449).  A run is inherently sequential (each
// event's outcome decides which batch starts next), so the device does not
// split one run; it runs MANY independent runs per launch — the replica
// groups of a bursty trace replay (config 5: one engine state per replica
// group), Monte-Carlo seeds, and the planner's simulator probes
// (_probe_range / _burst_throughput, src/planner.py:293-356), which call
// engine.run once per candidate.  One warp per run: the event loop's control
// flow is uniform across the warp (every lane reads the same shared-memory
// state and replays the same generator draws, so no lane waits for another),
// and the data-parallel parts go across lanes -- a finished batch's items
// (one lane each: queue entry, certainty, correct flag, record write), the
// dispatch scan over a device's replicas (one lane per replica, a warp
// min-reduction of (stage, -length, id rank)).
//
// Exactness.  Event order is the reference heap's (t, priority, seq) order:
// complete (0) < tick (1) < arrival (2) at equal t, pushes numbered in the
// reference's push order (all ticks first, then one pending arrival at a
// time and one completion per busy device).  Replica choice reproduces
// numpy's PCG64 generator (default_rng) draw for draw: rng.random() for a
// weighted draw (choose_weighted :238-245), rng.integers(n) through numpy's
// 32-bit Lemire bounded sampler with the bit generator's buffered upper half
// when a stage's weights sum to zero.  The gate is the reference's f64
// compare cert[row, m] >= thr.  Percentiles are nearest-rank (:111-120).
//
// State per run: every replica queue is a ring buffer in global memory
// (rings[R][ring_cap]) whose entries carry the request whole -- arrival index,
// stage, gear -- so a request moves between queues as one 8-byte store and a
// batch pop is a head advance; heads, tails, device state and counters live
// in shared memory.
#include <math.h>

#include "gs_common.cuh"

namespace gs {
namespace {

// ----------------------------------------------------------------- PCG64 --
// numpy's PCG64 (pcg_setseq_128_xsl_rr_64): state = state * M + inc, output
// the XSL-RR of the new state.  next_uint32 keeps the unused upper half of a
// 64-bit draw, exactly as numpy's bit generator does (has_uint32/uinteger).
struct Pcg64 {
  unsigned __int128 state, inc;
  uint32_t has32, u32;

  __device__ uint64_t next64() {
    const unsigned __int128 mult =
        ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    state = state * mult + inc;
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const uint32_t rot = (uint32_t)(state >> 122);
    const uint64_t x = hi ^ lo;
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
  // Generator.random(): 53 random bits scaled to [0, 1)
  __device__ double random() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
  // Generator.integers(0, n) for 1 <= n <= 2^32 (numpy: rng == 0 draws nothing;
  // else buffered_bounded_lemire_uint32 over [0, n - 1])
  __device__ uint32_t below(uint32_t n) {
    const uint32_t rng = n - 1;
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return next32();
    const uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
      while (left < thr) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

constexpr int kMaxR = GS_ENGINE_MAX_REPLICAS;
constexpr int kMaxD = GS_ENGINE_MAX_DEVICES;

struct RunSmem {
  uint32_t head[kMaxR], tail[kMaxR];  // ring positions (mod ring_cap): len = tail - head
  int64_t routed[kMaxR];
  int64_t t_done[kMaxD], seq_done[kMaxD];
  uint32_t batch_head[kMaxD];
  int32_t batch_r[kMaxD], batch_n[kMaxD];
  uint8_t busy[kMaxD];
};

// a queue entry: arrival index | stage << 32 | gear << 40
__device__ __forceinline__ uint64_t entry(uint32_t rid, uint32_t stage, uint32_t gear) {
  return (uint64_t)rid | ((uint64_t)stage << 32) | ((uint64_t)gear << 40);
}

// choose_weighted (src/engine.py:238-245) over one gear stage's CSR slice;
// every lane runs it alike (same generator state, same result)
__device__ int32_t choose_replica(const gs_engine_plan& p, int gear, int stage, Pcg64& rng) {
  const int32_t* off = p.gear_rep_off + (int64_t)gear * (p.max_stages + 1);
  const int32_t b = off[stage], e = off[stage + 1];
  const int32_t n = e - b;
  const double* cum = p.gear_cum + b;
  const double total = cum[n - 1];
  int32_t pos;
  if (total <= 0.0) {
    pos = (int32_t)rng.below((uint32_t)n);
  } else {
    const double x = rng.random() * total;
    // searchsorted(cum, x, side="right"), clipped to n - 1
    int32_t lo = 0, hi = n;
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (cum[mid] <= x) lo = mid + 1; else hi = mid;
    }
    pos = lo < n ? lo : n - 1;
  }
  return p.gear_rep[b + pos];
}

// k-th smallest (0-based) of a[0..n) by quickselect (the array is scratch)
__device__ int64_t select_kth(int64_t* a, int64_t n, int64_t k) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t pivot = a[lo + ((hi - lo) >> 1)];
    int64_t i = lo, j = hi;
    while (i <= j) {
      while (a[i] < pivot) ++i;
      while (a[j] > pivot) --j;
      if (i <= j) {
        const int64_t t = a[i];
        a[i] = a[j];
        a[j] = t;
        ++i;
        --j;
      }
    }
    if (k <= j) hi = j;
    else if (k >= i) lo = i;
    else return a[k];
  }
  return a[lo];
}

__global__ void __launch_bounds__(32) engine_kernel(const gs_engine_job* __restrict__ jobs, int n_jobs) {
  __shared__ RunSmem sm;
  __shared__ int64_t s_p95;
  if (blockIdx.x >= (unsigned)n_jobs) return;
  const gs_engine_job job = jobs[blockIdx.x];
  const gs_engine_plan p = *job.plan;
  const int R = p.n_replicas, D = p.n_devices, L = p.max_stages;
  const int lane = threadIdx.x;
  const uint32_t cap = (uint32_t)job.ring_cap;
  for (int i = lane; i < kMaxR; i += 32) {
    sm.head[i] = 0u;
    sm.tail[i] = 0u;
    sm.routed[i] = 0;
  }
  for (int i = lane; i < kMaxD; i += 32) {
    sm.busy[i] = 0;
    sm.batch_n[i] = 0;
  }
  const int64_t nb = (int64_t)p.n_cols * (p.batch_cap + 1);
  for (int64_t i = lane; i < nb; i += 32) job.model_batches[i] = 0;
  __syncwarp();

  Pcg64 rng;  // replicated in every lane
  rng.state = ((unsigned __int128)job.rng_state_hi << 64) | job.rng_state_lo;
  rng.inc = ((unsigned __int128)job.rng_inc_hi << 64) | job.rng_inc_lo;
  rng.has32 = job.rng_has_uint32;
  rng.u32 = job.rng_uinteger;

  const int64_t horizon = job.horizon_us;
  const int64_t period = job.measure_period_us;
  const int64_t n_ticks = (job.enable_ticks && period > 0) ? horizon / period : 0;
  int64_t seq = n_ticks;  // ticks took seq 0..n_ticks-1 (pushed first)
  int64_t tick_idx = 0;
  bool arr_pending = job.n_arrivals > 0;
  int64_t arr_idx = 0, arr_t = arr_pending ? job.arrivals[0] : 0;
  if (arr_pending) seq++;  // the pending arrival's push (it never ties another arrival)

  int gear_now = job.initial_gear;
  int64_t arrivals = 0, completed = 0, in_flight = 0, n_windows = 0;
  int64_t win_arrivals = 0, win_start = 0, win_correct = 0;
  const double period_s = (double)period / 1000000.0;

  while (true) {
    __syncwarp();
    // ---- pop the minimum (t, prio, seq) event (uniform: every lane alike)
    int kind = -1;  // 0 complete, 1 tick, 2 arrival
    int64_t bt = 0, bseq = 0;
    int bdev = -1;
    for (int d = 0; d < D; ++d) {
      if (!sm.busy[d]) continue;
      if (kind < 0 || sm.t_done[d] < bt || (sm.t_done[d] == bt && sm.seq_done[d] < bseq)) {
        kind = 0;
        bt = sm.t_done[d];
        bseq = sm.seq_done[d];
        bdev = d;
      }
    }
    if (tick_idx < n_ticks) {
      const int64_t tt = (tick_idx + 1) * period;
      if (kind < 0 || tt < bt) {
        kind = 1;
        bt = tt;
      }
    }
    if (arr_pending && (kind < 0 || arr_t < bt)) {
      kind = 2;
      bt = arr_t;
    }
    if (kind < 0 || bt > horizon) break;
    const int64_t now = bt;

    uint64_t touched = 0;
    if (kind == 2) {  // ---- EngineState.submit (:299-319)
      const int32_t ridx = choose_replica(p, gear_now, 0, rng);
      const uint32_t t = sm.tail[ridx];
      if (lane == 0) job.rings[(int64_t)ridx * cap + (t % cap)] = entry((uint32_t)arr_idx, 0u, (uint32_t)gear_now);
      __syncwarp();
      if (lane == 0) {
        sm.tail[ridx] = t + 1;
        sm.routed[ridx] += 1;
      }
      arrivals += 1;
      win_arrivals += 1;
      touched = 1ull << p.replica_device[ridx];
      arr_idx += 1;
      if (arr_idx < job.n_arrivals) {
        arr_t = job.arrivals[arr_idx];
        seq++;
      } else {
        arr_pending = false;
      }
    } else if (kind == 0) {  // ---- EngineState.finish_batch (:355-383)
      const int d = bdev;
      const int n = sm.batch_n[d];
      const int br = sm.batch_r[d];
      const uint32_t bh = sm.batch_head[d];
      __syncwarp();
      if (lane == 0) sm.busy[d] = 0;
      in_flight -= n;
      touched = 1ull << d;
      for (int c0 = 0; c0 < n; c0 += 32) {  // 32 items at a time, a lane each
        const int k = c0 + lane;
        const bool live = k < n;
        uint64_t e = 0;
        bool stop = false;
        uint8_t ok = 0;
        if (live) {
          e = job.rings[(int64_t)br * cap + ((bh + (uint32_t)k) % cap)];
          const uint32_t rid = (uint32_t)e, stage = (uint32_t)(e >> 32) & 0xFFu,
                         gear = (uint32_t)(e >> 40);
          const int m = p.gear_model[(int64_t)gear * L + stage];
          const bool last = (int)stage == p.gear_n_stages[gear] - 1;
          const int64_t cell = ((int64_t)rid % p.n_records) * p.n_cols + m;
          stop = last || p.cert[cell] >= p.gear_thr[(int64_t)gear * L + stage];
          if (stop) ok = p.corr[cell] ? 1 : 0;
        }
        const uint32_t smask = __ballot_sync(0xffffffffu, stop);
        const uint32_t cmask = __ballot_sync(0xffffffffu, stop && ok);
        if (stop) {
          gs_engine_record rec;
          rec.completion_us = now;
          rec.request_id = (int32_t)(uint32_t)e;
          rec.stages_executed = (uint8_t)(((e >> 32) & 0xFFu) + 1);
          rec.correct = ok;
          rec.gear_index = (uint16_t)(e >> 40);
          job.records[completed + __popc(smask & ((1u << lane) - 1u))] = rec;
        }
        completed += __popc(smask);
        win_correct += __popc(cmask);
        // forwarded items in batch order: one draw each, every lane alike
        uint32_t fmask = __ballot_sync(0xffffffffu, live && !stop);
        while (fmask) {
          const int src = __ffs(fmask) - 1;
          fmask &= fmask - 1;
          const uint64_t fe = __shfl_sync(0xffffffffu, e, src);
          const uint32_t stage = (uint32_t)(fe >> 32) & 0xFFu, gear = (uint32_t)(fe >> 40);
          const int32_t ridx = choose_replica(p, (int)gear, (int)stage + 1, rng);
          const uint32_t t = sm.tail[ridx];
          if (lane == 0) {
            job.rings[(int64_t)ridx * cap + (t % cap)] = entry((uint32_t)fe, stage + 1, gear);
            sm.tail[ridx] = t + 1;
          }
          __syncwarp();
          touched |= 1ull << p.replica_device[ridx];
        }
      }
    } else {  // ---- tick (:389-410) and maybe_switch_gear (:123-133)
      tick_idx += 1;
      const double qps = (double)win_arrivals / period_s;
      const int32_t* off = p.gear_rep_off + (int64_t)gear_now * (L + 1);
      int64_t q0 = 0;
      for (int e = off[0]; e < off[1]; ++e) {
        const int r = p.gear_rep[e];
        q0 += (int64_t)(sm.tail[r] - sm.head[r]);
      }
      const int n_ranges = p.n_gears;
      int64_t cand = (int64_t)floor(qps * (double)n_ranges / p.qps_max);
      if (cand > n_ranges - 1) cand = n_ranges - 1;
      int after = (int)cand;
      if (cand < gear_now && qps < job.alpha * (double)q0) after = gear_now;
      const int64_t nlat = completed - win_start;
      if (nlat > 0) {
        for (int64_t i = lane; i < nlat; i += 32) {  // latencies of the window, lane-parallel
          const gs_engine_record& r = job.records[win_start + i];
          job.scratch[i] = r.completion_us - job.arrivals[r.request_id];
        }
        __syncwarp();
        if (lane == 0) {
          int64_t k = (int64_t)ceil(95.0 / 100.0 * (double)nlat);
          if (k < 1) k = 1;
          s_p95 = select_kth(job.scratch, nlat, k - 1);
        }
        __syncwarp();
      }
      if (lane == 0) {
        gs_engine_window w;
        w.end_us = now;
        w.measured_qps = qps;
        w.first_stage_queue_len = (int32_t)q0;
        w.gear_before = gear_now;
        w.candidate_gear = (int32_t)cand;
        w.gear_after = after;
        w.completed = nlat;
        w.p95_us = nlat > 0 ? s_p95 : -1;
        w.accuracy = nlat > 0 ? (double)win_correct / (double)nlat
                              : __longlong_as_double(0x7ff8000000000000ll);
        if (n_windows < job.windows_cap) job.windows[n_windows] = w;
      }
      n_windows += 1;
      gear_now = after;
      win_arrivals = 0;
      win_start = completed;
      win_correct = 0;
      touched = (D >= 64) ? ~0ull : ((1ull << D) - 1);
    }

    __syncwarp();  // lane 0's shared-memory updates are seen by every lane
    // ---- scan_device for the touched devices in ascending order (:321-353)
    while (touched) {
      const int d = __ffsll((long long)touched) - 1;
      touched &= touched - 1;
      if (sm.busy[d]) continue;
      // a lane per replica: candidate key (stage, -len, id rank), warp minimum
      const int32_t* minq = p.gear_min_qlen + (int64_t)gear_now * R;
      uint64_t best = ~0ull;
      for (int r = lane; r < R; r += 32) {
        if (p.replica_device[r] != d) continue;
        const uint32_t len = sm.tail[r] - sm.head[r];
        if (len == 0 || (int)len < minq[r]) continue;
        const uint64_t e = job.rings[(int64_t)r * cap + (sm.head[r] % cap)];
        const uint64_t st = (e >> 32) & 0xFFu;
        const uint64_t key = (st << 56) | ((uint64_t)(0xFFFFFFFFu - len) << 16) |
                             ((uint64_t)p.replica_rank[r] << 8) | (uint64_t)r;
        best = key < best ? key : best;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y < best ? y : best;
      }
      if (best == ~0ull) continue;
      const int r = (int)(best & 0xFFu);
      const int m = p.replica_model[r];
      const uint32_t len = sm.tail[r] - sm.head[r];
      const int size = min((int)len, p.model_max_batch[m]);
      const uint32_t h = sm.head[r];
      __syncwarp();
      if (lane == 0) {
        sm.head[r] = h + (uint32_t)size;
        sm.busy[d] = 1;
        sm.batch_head[d] = h;
        sm.batch_r[d] = r;
        sm.batch_n[d] = size;
        sm.t_done[d] = now + p.model_runtime_us[(int64_t)m * (p.batch_cap + 1) + size];
        sm.seq_done[d] = seq;
        job.model_batches[(int64_t)m * (p.batch_cap + 1) + size] += 1;
      }
      __syncwarp();
      seq++;
      in_flight += size;
    }
  }

  __syncwarp();
  for (int r = lane; r < R; r += 32) {
    job.replica_counts[2 * r] = sm.routed[r];
    job.replica_counts[2 * r + 1] = (int64_t)(sm.tail[r] - sm.head[r]);
  }
  if (lane == 0) {
    job.result[0] = arrivals;
    job.result[1] = completed;
    job.result[2] = in_flight;
    job.result[3] = n_windows;
    job.result[4] = (int64_t)(uint64_t)(rng.state >> 64);
    job.result[5] = (int64_t)(uint64_t)rng.state;
    job.result[6] = rng.has32;
    job.result[7] = rng.u32;
  }
}

}  // namespace
}  // namespace gs

extern "C" int gs_engine_run(const gs_engine_job* jobs, int32_t n_jobs, void* stream) {
  GS_REQUIRE(n_jobs >= 0);
  if (n_jobs == 0) return GS_OK;
  GS_REQUIRE(jobs != nullptr);
  gs::engine_kernel<<<(unsigned)n_jobs, 32, 0, static_cast<cudaStream_t>(stream)>>>(jobs, n_jobs);
  GS_LAUNCH_CHECK();
  return GS_OK;
}
