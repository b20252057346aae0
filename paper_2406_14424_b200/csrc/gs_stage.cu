// gs_stage.cu — online cascade stage step.
//
// Reference: EngineState.finish_batch (/root/reference/pkg/src/gearserve/
// engine.py:355-383): item i stops when its stage is the cascade's last or
// cert[row, m] >= thr (inclusive, :366-367); otherwise it is forwarded and
// appended, in batch order, to a next-stage queue (:377-382).  Certainty is
// Eq. 5, top score minus second score, a singleton returning the score
// itself (cascades.certainty, src/cascades.py:20-28).
//
// B200 mapping.  One pass over the stage's score rows:
//   * wide rows (n_cls >= 32): one warp per row, 128-bit vector loads,
//     per-lane top-2 / max / exp-sums, warp-shuffle reductions;
//   * narrow rows (binary heads etc.): one thread per row;
//   * gate, then order-preserving compaction of the deferred rows with a
//     single-pass decoupled look-back scan (ballot + popc inside the block),
//     so deferred indices land in batch order without a second kernel;
//   * the deferred rows' payload is gathered into the next stage's
//     contiguous batch buffer by the same CTA.
// Margin certainty is bit-exact: the top two are found in the source dtype
// (exact) and subtracted in f64, like the reference on the same values
// promoted to f64.  Max-softmax / entropy are extensions (no reference
// oracle): exp in f32 (expf, <= 2 ulp), sums in f64.
#include <algorithm>
#include <cmath>

#include "gs_common.cuh"

namespace gs {
namespace {

struct bf16_t {
  uint16_t v;
};

__device__ __forceinline__ float to_float(float x) { return x; }
__device__ __forceinline__ double to_float(double x) { return x; }
__device__ __forceinline__ float to_float(bf16_t x) {
  return __uint_as_float((uint32_t)x.v << 16);
}

template <typename T>
struct Compute {
  using type = float;
};
template <>
struct Compute<double> {
  using type = double;
};

template <typename C>
__device__ __forceinline__ C neg_inf();
template <>
__device__ __forceinline__ float neg_inf<float>() {
  return __int_as_float(0xff800000);
}
template <>
__device__ __forceinline__ double neg_inf<double>() {
  return __longlong_as_double(0xfff0000000000000ll);
}

// top two so far (duplicates count twice, NaN never enters: the sorted()
// semantics of cascades.certainty on finite scores)
__device__ __forceinline__ void push_top2(float x, float& m1, float& m2) {
  m2 = fmaxf(m2, fminf(m1, x));  // three FMNMX, no branches
  m1 = fmaxf(m1, x);
}
template <typename C>
__device__ __forceinline__ void push_top2(C x, C& m1, C& m2) {
  if (x > m1) {
    m2 = m1;
    m1 = x;
  } else if (x > m2) {
    m2 = x;
  }
}

template <typename C>
__device__ __forceinline__ void merge_top2(C& m1, C& m2, C o1, C o2) {
  const C hi = m1 > o1 ? m1 : o1;
  const C lo = m1 > o1 ? o1 : m1;
  const C s = m2 > o2 ? m2 : o2;
  m1 = hi;
  m2 = lo > s ? lo : s;
}

__device__ __forceinline__ double exp_term(float d) { return (double)expf(d); }
__device__ __forceinline__ double exp_term(double d) { return exp(d); }

// streaming 16-byte load: read once, keep it out of L1
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// 16-byte vector of T
template <typename T>
struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
  T v[N];
};

template <typename T, typename F>
__device__ __forceinline__ void warp_for_each(const T* row, int n, bool vec_ok, F&& f) {
  const int lane = (int)lane_id();
  if (vec_ok) {
    constexpr int V = Vec16<T>::N;
    const int nv = n / V;
    const uint4* rv = reinterpret_cast<const uint4*>(row);
    int i = lane;
    // two 16-byte loads in flight per lane per iteration
    for (; i + 32 < nv; i += 64) {
      uint4 r0 = __ldg(rv + i);
      uint4 r1 = __ldg(rv + i + 32);
      const T* t0 = reinterpret_cast<const T*>(&r0);
      const T* t1 = reinterpret_cast<const T*>(&r1);
#pragma unroll
      for (int u = 0; u < V; ++u) f(t0[u]);
#pragma unroll
      for (int u = 0; u < V; ++u) f(t1[u]);
    }
    for (; i < nv; i += 32) {
      uint4 r0 = __ldg(rv + i);
      const T* t0 = reinterpret_cast<const T*>(&r0);
#pragma unroll
      for (int u = 0; u < V; ++u) f(t0[u]);
    }
    for (int j = nv * V + lane; j < n; j += 32) f(row[j]);
  } else {
    for (int j = lane; j < n; j += 32) f(row[j]);
  }
}

// The two reduced quantities a row's certainty is finished from (valid in
// all lanes): margin {top, second}; max-softmax {sum of exp(x - max), -};
// entropy {that sum, sum of exp(x - max) (x - max)}.  finish_cert turns
// them into the certainty; the stage step finishes 32 rows in one pass
// (lane k the warp's k-th row) instead of once per row: the f64 log and
// divisions of the entropy were a quarter of its instructions.
struct RowPair {
  double x, y;
};

template <int KIND>
__device__ __forceinline__ double finish_cert(RowPair p, int n, double log_n) {
  if (KIND == GS_CERT_MARGIN) return p.x - p.y;
  if (n == 1) return 1.0;
  if (KIND == GS_CERT_MAX_SOFTMAX) return 1.0 / p.x;
  const double H = log(p.x) - p.y / p.x;
  return 1.0 - H / (log_n > 0.0 ? log_n : log((double)n));
}

// Certainty pair of one row, computed by a full warp.
template <typename T, int KIND>
__device__ __forceinline__ RowPair warp_row_pair(const T* row, int n, bool vec_ok) {
  using C = typename Compute<T>::type;
  if (n == 1) {
    const double x0 = (double)to_float(row[0]);
    return {KIND == GS_CERT_MARGIN ? x0 : 1.0, 0.0};
  }
  constexpr int V = Vec16<T>::N;
  constexpr int RV = 8;  // 16-byte vectors per lane held in registers
  if (vec_ok && n / V <= 32 * RV) {
    // register-resident row: every 16-byte load of the row is issued up
    // front (8 per lane, 4 KB per warp in flight) and the row is read from
    // HBM exactly once, whatever the certainty kind
    const int lane = (int)lane_id();
    const int nv = n / V;
    const uint4* rv = reinterpret_cast<const uint4*>(row);
    uint4 buf[RV];
#pragma unroll
    for (int u = 0; u < RV; ++u) {
      const int i = lane + 32 * u;
      buf[u] = i < nv ? ldg_stream(rv + i) : make_uint4(0, 0, 0, 0);
    }
    const int tail = n - nv * V;
    const bool has_tail = lane < tail;
    const T tx = has_tail ? row[nv * V + lane] : row[0];
    auto each = [&](auto&& f) {
#pragma unroll
      for (int u = 0; u < RV; ++u) {
        if (lane + 32 * u < nv) {
          const T* t = reinterpret_cast<const T*>(&buf[u]);
#pragma unroll
          for (int q = 0; q < V; ++q) f(t[q]);
        }
      }
      if (has_tail) f(tx);
    };
    if (KIND == GS_CERT_MARGIN) {
      C m1 = neg_inf<C>(), m2 = neg_inf<C>();
      each([&](T x) { push_top2((C)to_float(x), m1, m2); });
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const C o1 = __shfl_xor_sync(0xffffffffu, m1, o);
        const C o2 = __shfl_xor_sync(0xffffffffu, m2, o);
        merge_top2<C>(m1, m2, o1, o2);
      }
      return {(double)m1, (double)m2};
    }
    C m = neg_inf<C>();
    if constexpr (sizeof(C) == 4) {  // a max per 16-byte vector, then two chains over them
      C ma = neg_inf<C>(), mb = neg_inf<C>();
#pragma unroll
      for (int u = 0; u < RV; ++u) {
        if (lane + 32 * u < nv) {
          const T* tv = reinterpret_cast<const T*>(&buf[u]);
          C vm = (C)to_float(tv[0]);
#pragma unroll
          for (int q = 1; q < V; ++q) vm = fmaxf(vm, (C)to_float(tv[q]));
          if (u & 1)
            mb = fmaxf(mb, vm);
          else
            ma = fmaxf(ma, vm);
        }
      }
      m = fmaxf(ma, mb);
      if (has_tail) m = fmaxf(m, (C)to_float(tx));
    } else {
      each([&](T x) {
        const C v = (C)to_float(x);
        m = v > m ? v : m;
      });
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const C y = __shfl_xor_sync(0xffffffffu, m, o);
      m = y > m ? y : m;
    }
    double s = 0.0, t = 0.0;
    if constexpr (sizeof(C) == 4) {
      // f32 rows: exp2 on the SFU, the terms of one 16-byte vector summed in
      // f32 (all of one sign, so each group sum is within 3 ulp), the group
      // sums accumulated in f64: half a conversion per element instead of
      // two, and |cert error| stays far below the 5e-7 the tests allow
      constexpr float kLog2e = 1.4426950408889634f;
      auto term = [&](float x, float& e, float& d) {
        d = x - m;
        float y;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(d * kLog2e));
        e = y;
      };
      double s_odd = 0.0, t_odd = 0.0;  // two f64 chains over the vectors
#pragma unroll
      for (int u = 0; u < RV; ++u) {
        if (lane + 32 * u < nv) {
          const T* tv = reinterpret_cast<const T*>(&buf[u]);
          float s4 = 0.f, t4 = 0.f;
#pragma unroll
          for (int q = 0; q < V; ++q) {
            float e, d;
            term((float)to_float(tv[q]), e, d);
            s4 += e;
            t4 = fmaf(e, d, t4);
          }
          if (u & 1) {
            s_odd += (double)s4;
            if (KIND == GS_CERT_ENTROPY) t_odd += (double)t4;
          } else {
            s += (double)s4;
            if (KIND == GS_CERT_ENTROPY) t += (double)t4;
          }
        }
      }
      s += s_odd;
      t += t_odd;
      if (has_tail) {
        float e, d;
        term((float)to_float(tx), e, d);
        s += (double)e;
        if (KIND == GS_CERT_ENTROPY) t += (double)e * (double)d;
      }
    } else {
      each([&](T x) {
        const C d = (C)to_float(x) - m;
        const double e = exp_term(d);
        s += e;
        if (KIND == GS_CERT_ENTROPY) t += e * (double)d;
      });
    }
    s = warp_sum(s);
    if (KIND == GS_CERT_ENTROPY) t = warp_sum(t);
    return {s, t};
  }
  if (KIND == GS_CERT_MARGIN) {
    C m1 = neg_inf<C>(), m2 = neg_inf<C>();
    warp_for_each<T>(row, n, vec_ok, [&](T x) { push_top2((C)to_float(x), m1, m2); });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const C o1 = __shfl_xor_sync(0xffffffffu, m1, o);
      const C o2 = __shfl_xor_sync(0xffffffffu, m2, o);
      merge_top2<C>(m1, m2, o1, o2);
    }
    return {(double)m1, (double)m2};
  } else {
    C m = neg_inf<C>();
    warp_for_each<T>(row, n, vec_ok, [&](T x) {
      const C v = (C)to_float(x);
      m = v > m ? v : m;
    });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const C y = __shfl_xor_sync(0xffffffffu, m, o);
      m = y > m ? y : m;
    }
    double s = 0.0, t = 0.0;
    warp_for_each<T>(row, n, vec_ok, [&](T x) {
      const C d = (C)to_float(x) - m;
      const double e = exp_term(d);
      s += e;
      if (KIND == GS_CERT_ENTROPY) t += e * (double)d;
    });
    s = warp_sum(s);
    if (KIND == GS_CERT_ENTROPY) t = warp_sum(t);
    return {s, t};
  }
}

// Certainty of one row, computed by a full warp; result valid in all lanes.
// log_n: ln(n) precomputed by the caller for the entropy kind (<= 0: compute)
template <typename T, int KIND>
__device__ __forceinline__ double warp_row_cert(const T* row, int n, bool vec_ok, double log_n = 0.0) {
  return finish_cert<KIND>(warp_row_pair<T, KIND>(row, n, vec_ok), n, log_n);
}

// Certainty of one row computed by one thread.
template <typename T, int KIND>
__device__ __forceinline__ double thread_row_cert(const T* row, int n) {
  using C = typename Compute<T>::type;
  if (n == 1) {
    const double x0 = (double)to_float(row[0]);
    return KIND == GS_CERT_MARGIN ? x0 : 1.0;
  }
  if (KIND == GS_CERT_MARGIN) {
    C m1 = neg_inf<C>(), m2 = neg_inf<C>();
    for (int j = 0; j < n; ++j) push_top2((C)to_float(row[j]), m1, m2);
    return (double)m1 - (double)m2;
  } else {
    C m = neg_inf<C>();
    for (int j = 0; j < n; ++j) {
      const C v = (C)to_float(row[j]);
      m = v > m ? v : m;
    }
    double s = 0.0, t = 0.0;
    for (int j = 0; j < n; ++j) {
      const C d = (C)to_float(row[j]) - m;
      const double e = exp_term(d);
      s += e;
      if (KIND == GS_CERT_ENTROPY) t += e * (double)d;
    }
    if (KIND == GS_CERT_MAX_SOFTMAX) return 1.0 / s;
    const double H = log(s) - t / s;
    return 1.0 - H / log((double)n);
  }
}

// --------------------------------------------------------- gs_certainty --
template <typename T, int KIND, bool WIDE>
__global__ void __launch_bounds__(256) certainty_kernel(const T* scores, int64_t n_rows, int n_cls,
                                                        int64_t stride, const int32_t* row_len,
                                                        bool vec_ok, double* out) {
  if (WIDE && KIND == GS_CERT_MARGIN) {  // nothing to finish: a row per warp trip
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nw) {
      const int n = row_len ? row_len[r] : n_cls;
      const double c = warp_row_cert<T, KIND>(scores + r * stride, n, vec_ok && n == n_cls);
      if (lane_id() == 0) out[r] = c;
    }
  } else if (WIDE) {
    // a warp takes 32 consecutive rows: lane k keeps row k's (sum, entropy)
    // pair and every lane finishes its own row at the end (the logs and
    // divisions leave the per-row chain; one coalesced store of 32 results)
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = (int)lane_id();
    for (int64_t r0 = warp * 32; r0 < n_rows; r0 += nw * 32) {
      RowPair mine{0.0, 0.0};
      int my_n = n_cls;
      const int nr = (int)min((int64_t)32, n_rows - r0);
      for (int k = 0; k < nr; ++k) {
        const int64_t r = r0 + k;
        const int n = row_len ? row_len[r] : n_cls;
        const RowPair pr = warp_row_pair<T, KIND>(scores + r * stride, n, vec_ok && n == n_cls);
        if (lane == k) {
          mine = pr;
          my_n = n;
        }
      }
      if (lane < nr) out[r0 + lane] = finish_cert<KIND>(mine, my_n, 0.0);
    }
  } else {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
      const int n = row_len ? row_len[r] : n_cls;
      out[r] = thread_row_cert<T, KIND>(scores + r * stride, n);
    }
  }
}

// --------------------------------------------------------- stage step ----
struct StepArgs {
  const void* scores;
  int64_t n_rows;
  int32_t n_cls;
  int64_t stride;
  int32_t vec_ok;
  const double* thr;
  const uint8_t* is_last;
  double* cert_out;
  uint8_t* stop_out;
  int64_t* deferred_idx;
  int64_t* n_deferred;
  double near_eps;
  int64_t* near_idx;
  int64_t* n_near;
  const uint8_t* payload;
  int64_t payload_bytes;
  uint8_t* next_payload;
  uint64_t* states;
  unsigned long long* counter;
  int64_t n_tiles;
  int32_t rows_per_tile;
  double log_n;  // ln(n_cls)
};

constexpr int kStepThreads = 256;
constexpr int kWideRowsPerWarp = 32;
constexpr int kWideTile = (kStepThreads / 32) * kWideRowsPerWarp;  // 256 rows: one per thread at the gate

__device__ __forceinline__ void copy_payload_row(const uint8_t* src, uint8_t* dst, int64_t bytes,
                                                 bool vec) {
  const int lane = (int)lane_id();
  if (vec) {
    const int64_t nv = bytes / 16;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (int64_t j = lane; j < nv; j += 32) d[j] = __ldg(s + j);
  } else {
    for (int64_t j = lane; j < bytes; j += 32) dst[j] = src[j];
  }
}

// Gate + compaction + payload gather for one tile; `cert` is this thread's
// row certainty (thread t owns row base + t when t < rows).
__device__ __forceinline__ void gate_tile(const StepArgs& a, int64_t tile, int64_t base, int rows,
                                          double cert, int64_t* s_rows, uint32_t* s_warp,
                                          uint64_t* s_misc) {
  const int t = threadIdx.x;
  const int64_t r = base + t;
  bool defer = false, near = false;
  if (t < rows) {
    const bool last = a.is_last ? a.is_last[r] != 0 : false;
    const double th = a.thr[r];
    const bool stop = last || cert >= th;
    defer = !stop;
    near = !last && fabs(cert - th) <= a.near_eps;
    if (a.cert_out) a.cert_out[r] = cert;
    if (a.stop_out) a.stop_out[r] = stop ? 1 : 0;
  }
  const PairScan ps = block_pair_scan(defer, near && a.near_idx != nullptr, a.states, tile, s_warp, s_misc);
  if (defer) a.deferred_idx[ps.a_off] = r;
  if (near && a.near_idx) a.near_idx[ps.b_off] = r;
  if (tile == a.n_tiles - 1 && t == 0) {
    *a.n_deferred = (int64_t)ps.a_total;
    if (a.n_near) *a.n_near = a.near_idx ? (int64_t)ps.b_total : 0;
  }
  if (a.payload && a.next_payload && a.payload_bytes > 0) {
    const uint32_t tile_count = __syncthreads_count(defer);
    const uint64_t tile_base = ps.a_total - tile_count;
    if (defer) s_rows[ps.a_off - tile_base] = r;
    __syncthreads();
    const bool vec = aligned16(a.payload) && aligned16(a.next_payload) && (a.payload_bytes % 16 == 0);
    for (uint32_t j = threadIdx.x >> 5; j < tile_count; j += blockDim.x >> 5) {
      const int64_t src_row = s_rows[j];
      copy_payload_row(a.payload + src_row * a.payload_bytes,
                       a.next_payload + (int64_t)(tile_base + j) * a.payload_bytes,
                       a.payload_bytes, vec);
    }
  }
}

template <typename T, int KIND, bool WIDE>
__global__ void __launch_bounds__(kStepThreads) stage_step_kernel(const __grid_constant__ StepArgs a) {
  __shared__ uint32_t s_warp[64];
  __shared__ uint64_t s_misc[4];
  __shared__ int64_t s_tile;
  __shared__ double s_cert[kStepThreads];
  __shared__ int64_t s_rows[kStepThreads];
  const int64_t tile = next_tile_id(a.counter, &s_tile);
  const int64_t base = tile * a.rows_per_tile;
  const int rows = (int)min((int64_t)a.rows_per_tile, a.n_rows - base);
  const T* scores = static_cast<const T*>(a.scores);
  double cert = 0.0;
  if (WIDE) {
    const int warp = threadIdx.x >> 5;
    // lane k keeps the pair of the warp's k-th row; one finishing pass
    static_assert(kWideRowsPerWarp == 32, "a row per lane");
    const int lane = (int)lane_id();
    RowPair mine{0.0, 0.0};
    for (int k = 0; k < kWideRowsPerWarp; ++k) {
      const int lr = warp * kWideRowsPerWarp + k;
      if (lr < rows) {
        const RowPair p = warp_row_pair<T, KIND>(scores + (base + lr) * a.stride, a.n_cls, a.vec_ok);
        if (lane == k) mine = p;
      }
    }
    const int lr = warp * kWideRowsPerWarp + lane;
    if (lr < rows) s_cert[lr] = finish_cert<KIND>(mine, a.n_cls, a.log_n);
    __syncthreads();
    if ((int)threadIdx.x < rows) cert = s_cert[threadIdx.x];
  } else {
    if ((int)threadIdx.x < rows)
      cert = thread_row_cert<T, KIND>(scores + (base + threadIdx.x) * a.stride, a.n_cls);
  }
  gate_tile(a, tile, base, rows, cert, s_rows, s_warp, s_misc);
}

// ------------------------------------------------------------- gate -------
struct GateArgs {
  const double* cert;
  const uint8_t* corr;
  int64_t n_rec;
  int32_t n_models;
  const int64_t* row;
  const int32_t* model;
  const double* thr;
  const uint8_t* is_last;
  int64_t n_items;
  uint8_t* stop_out;
  uint8_t* correct_out;
  int64_t* deferred_idx;
  int64_t* n_deferred;
  double near_eps;
  int64_t* near_idx;
  int64_t* n_near;
  uint64_t* states;
  unsigned long long* counter;
  int64_t n_tiles;
};

__global__ void __launch_bounds__(256) stage_gate_kernel(const __grid_constant__ GateArgs a) {
  __shared__ uint32_t s_warp[64];
  __shared__ uint64_t s_misc[4];
  __shared__ int64_t s_tile;
  const int64_t tile = next_tile_id(a.counter, &s_tile);
  const int64_t i = tile * blockDim.x + threadIdx.x;
  bool defer = false, near = false;
  if (i < a.n_items) {
    const int64_t r = a.row[i];
    const int m = a.model[i];
    const bool ok = r >= 0 && r < a.n_rec && m >= 0 && m < a.n_models;
    const double c = ok ? a.cert[r * a.n_models + m] : 0.0;
    const bool last = a.is_last ? a.is_last[i] != 0 : false;
    const double th = a.thr[i];
    const bool stop = last || c >= th;
    defer = !stop;
    near = !last && fabs(c - th) <= a.near_eps;
    if (a.stop_out) a.stop_out[i] = stop ? 1 : 0;
    if (a.correct_out) a.correct_out[i] = (stop && ok) ? a.corr[r * a.n_models + m] : 0;
  }
  const PairScan ps = block_pair_scan(defer, near && a.near_idx != nullptr, a.states, tile, s_warp, s_misc);
  if (defer) a.deferred_idx[ps.a_off] = i;
  if (near && a.near_idx) a.near_idx[ps.b_off] = i;
  if (tile == a.n_tiles - 1 && threadIdx.x == 0) {
    *a.n_deferred = (int64_t)ps.a_total;
    if (a.n_near) *a.n_near = a.near_idx ? (int64_t)ps.b_total : 0;
  }
}

size_t step_ws_bytes(int64_t n_rows) {
  const int64_t tiles = (n_rows + kWideTile - 1) / kWideTile;
  return round_up((size_t)(tiles + 1) * 8, 256) + 256;
}

template <typename T, int KIND>
cudaError_t launch_certainty(const void* scores, int64_t n_rows, int n_cls, int64_t stride,
                             const int32_t* row_len, double* out, cudaStream_t st) {
  const T* s = static_cast<const T*>(scores);
  const bool vec_ok = aligned16(scores) && ((stride * (int64_t)sizeof(T)) % 16 == 0);
  if (n_cls >= 32) {
    // margin: a row per warp; else 32 rows a warp (8 warps a block)
    int64_t blocks = KIND == GS_CERT_MARGIN ? (n_rows * 32 + 255) / 256 : (n_rows + 255) / 256;
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 32));
    certainty_kernel<T, KIND, true><<<(unsigned)blocks, 256, 0, st>>>(s, n_rows, n_cls, stride, row_len,
                                                                      vec_ok, out);
  } else {
    int64_t blocks = (n_rows + 255) / 256;
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 32));
    certainty_kernel<T, KIND, false><<<(unsigned)blocks, 256, 0, st>>>(s, n_rows, n_cls, stride, row_len,
                                                                       vec_ok, out);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_certainty(int kind, const void* scores, int64_t n_rows, int n_cls, int64_t stride,
                               const int32_t* row_len, double* out, cudaStream_t st) {
  switch (kind) {
    case GS_CERT_MARGIN: return launch_certainty<T, GS_CERT_MARGIN>(scores, n_rows, n_cls, stride, row_len, out, st);
    case GS_CERT_MAX_SOFTMAX: return launch_certainty<T, GS_CERT_MAX_SOFTMAX>(scores, n_rows, n_cls, stride, row_len, out, st);
    default: return launch_certainty<T, GS_CERT_ENTROPY>(scores, n_rows, n_cls, stride, row_len, out, st);
  }
}

template <typename T, int KIND>
cudaError_t launch_step(StepArgs a, cudaStream_t st) {
  const bool wide = a.n_cls >= 32;
  a.rows_per_tile = wide ? kWideTile : kStepThreads;
  a.log_n = a.n_cls > 1 ? std::log((double)a.n_cls) : 0.0;
  a.n_tiles = (a.n_rows + a.rows_per_tile - 1) / a.rows_per_tile;
  a.vec_ok = aligned16(a.scores) && ((a.stride * (int64_t)sizeof(T)) % 16 == 0);
  if (a.n_tiles > 0x7fffffff) return cudaErrorInvalidValue;
  if (wide)
    stage_step_kernel<T, KIND, true><<<(unsigned)a.n_tiles, kStepThreads, 0, st>>>(a);
  else
    stage_step_kernel<T, KIND, false><<<(unsigned)a.n_tiles, kStepThreads, 0, st>>>(a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_step(int kind, const StepArgs& a, cudaStream_t st) {
  switch (kind) {
    case GS_CERT_MARGIN: return launch_step<T, GS_CERT_MARGIN>(a, st);
    case GS_CERT_MAX_SOFTMAX: return launch_step<T, GS_CERT_MAX_SOFTMAX>(a, st);
    default: return launch_step<T, GS_CERT_ENTROPY>(a, st);
  }
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" int gs_certainty(const void* scores, int32_t dtype, int64_t n_rows, int32_t n_cls,
                            int64_t row_stride, const int32_t* row_len, int32_t kind,
                            double* cert_out, void* stream) {
  GS_REQUIRE(n_rows >= 0 && n_cls >= 1 && row_stride >= n_cls);
  GS_REQUIRE(kind >= GS_CERT_MARGIN && kind <= GS_CERT_ENTROPY);
  if (n_rows == 0) return GS_OK;
  GS_REQUIRE(scores && cert_out);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (dtype) {
    case GS_F32: e = dispatch_certainty<float>(kind, scores, n_rows, n_cls, row_stride, row_len, cert_out, st); break;
    case GS_F64: e = dispatch_certainty<double>(kind, scores, n_rows, n_cls, row_stride, row_len, cert_out, st); break;
    case GS_BF16: e = dispatch_certainty<bf16_t>(kind, scores, n_rows, n_cls, row_stride, row_len, cert_out, st); break;
    default: return GS_EINVAL;
  }
  GS_CUDA_TRY(e);
  return GS_OK;
}

extern "C" int gs_stage_step_workspace(int64_t n_rows, size_t* bytes) {
  GS_REQUIRE(bytes && n_rows >= 0);
  *bytes = step_ws_bytes(n_rows);
  return GS_OK;
}

extern "C" int gs_stage_step(const void* scores, int32_t dtype, int64_t n_rows, int32_t n_cls,
                             int64_t row_stride, int32_t kind, const double* thr,
                             const uint8_t* is_last, double* cert_out, uint8_t* stop_out,
                             int64_t* deferred_idx, int64_t* n_deferred, double near_eps,
                             int64_t* near_idx, int64_t* n_near, const void* payload,
                             int64_t payload_row_bytes, void* next_payload, void* workspace,
                             size_t workspace_bytes, void* stream) {
  GS_REQUIRE(n_rows >= 0 && n_cls >= 1 && row_stride >= n_cls && n_deferred);
  GS_REQUIRE(kind >= GS_CERT_MARGIN && kind <= GS_CERT_ENTROPY);
  GS_REQUIRE(payload_row_bytes >= 0);
  if (n_rows >= ((int64_t)1 << 31) - 1) return GS_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_rows == 0) {
    GS_CUDA_TRY(cudaMemsetAsync(n_deferred, 0, 8, st));
    if (n_near) GS_CUDA_TRY(cudaMemsetAsync(n_near, 0, 8, st));
    return GS_OK;
  }
  GS_REQUIRE(scores && thr && deferred_idx);
  // one tile (<= 256 narrow rows, <= kWideTile wide rows) needs no tile
  // counter or look-back states: no workspace memset
  const bool single = n_rows <= (n_cls >= 32 ? (int64_t)kWideTile : (int64_t)kStepThreads);
  if (!single) {
    const size_t need = step_ws_bytes(n_rows);
    if (!workspace || workspace_bytes < need) return GS_EWORKSPACE;
    GS_CUDA_TRY(cudaMemsetAsync(workspace, 0, need, st));
  }
  StepArgs a{};
  a.scores = scores;
  a.n_rows = n_rows;
  a.n_cls = n_cls;
  a.stride = row_stride;
  a.thr = thr;
  a.is_last = is_last;
  a.cert_out = cert_out;
  a.stop_out = stop_out;
  a.deferred_idx = deferred_idx;
  a.n_deferred = n_deferred;
  a.near_eps = near_eps;
  a.near_idx = near_idx;
  a.n_near = n_near;
  a.payload = static_cast<const uint8_t*>(payload);
  a.payload_bytes = payload_row_bytes;
  a.next_payload = static_cast<uint8_t*>(next_payload);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  a.counter = single ? nullptr : reinterpret_cast<unsigned long long*>(ws);
  a.states = single ? nullptr : reinterpret_cast<uint64_t*>(ws + 256);
  cudaError_t e;
  switch (dtype) {
    case GS_F32: e = dispatch_step<float>(kind, a, st); break;
    case GS_F64: e = dispatch_step<double>(kind, a, st); break;
    case GS_BF16: e = dispatch_step<bf16_t>(kind, a, st); break;
    default: return GS_EINVAL;
  }
  GS_CUDA_TRY(e);
  return GS_OK;
}

extern "C" int gs_stage_gate(const double* certainty, const uint8_t* correct, int64_t n_rec,
                             int32_t n_models, const int64_t* row, const int32_t* model,
                             const double* thr, const uint8_t* is_last, int64_t n_items,
                             uint8_t* stop_out, uint8_t* correct_out, int64_t* deferred_idx,
                             int64_t* n_deferred, double near_eps, int64_t* near_idx,
                             int64_t* n_near, void* workspace, size_t workspace_bytes,
                             void* stream) {
  GS_REQUIRE(n_items >= 0 && n_rec >= 0 && n_models >= 1 && n_deferred);
  if (n_items >= ((int64_t)1 << 31) - 1) return GS_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_items == 0) {
    GS_CUDA_TRY(cudaMemsetAsync(n_deferred, 0, 8, st));
    if (n_near) GS_CUDA_TRY(cudaMemsetAsync(n_near, 0, 8, st));
    return GS_OK;
  }
  GS_REQUIRE(certainty && correct && row && model && thr && deferred_idx);
  const int64_t n_tiles = (n_items + 255) / 256;
  if (n_tiles > 1) {  // one tile needs no tile counter or look-back states
    const size_t need = step_ws_bytes(n_items);
    if (!workspace || workspace_bytes < need) return GS_EWORKSPACE;
    GS_CUDA_TRY(cudaMemsetAsync(workspace, 0, need, st));
  }
  GateArgs a{};
  a.cert = certainty;
  a.corr = correct;
  a.n_rec = n_rec;
  a.n_models = n_models;
  a.row = row;
  a.model = model;
  a.thr = thr;
  a.is_last = is_last;
  a.n_items = n_items;
  a.stop_out = stop_out;
  a.correct_out = correct_out;
  a.deferred_idx = deferred_idx;
  a.n_deferred = n_deferred;
  a.near_eps = near_eps;
  a.near_idx = near_idx;
  a.n_near = n_near;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  a.counter = n_tiles > 1 ? reinterpret_cast<unsigned long long*>(ws) : nullptr;
  a.states = n_tiles > 1 ? reinterpret_cast<uint64_t*>(ws + 256) : nullptr;
  a.n_tiles = n_tiles;
  stage_gate_kernel<<<(unsigned)a.n_tiles, 256, 0, st>>>(a);
  GS_LAUNCH_CHECK();
  return GS_OK;
}

// Packed small-batch gate (the online path: batches of 1-8 items,
// src/synth.py:30): the batch's items arrive in ONE pinned host buffer
// {row i64[n], thr f64[n], model i32[n], is_last u8[n]}, the outcome leaves
// in ONE pinned host buffer {n_deferred i64, n_near i64, stop u8[n],
// correct u8[n], (8-aligned) near i64[n]}: one H2D, one kernel, one D2H on
// the caller's stream, then (sync != 0) a stream synchronize.  dev_buf holds
// the device copies (gs_stage_gate_packed_bytes) and, for n > 256, the
// look-back workspace.
static size_t packed_in_bytes(int64_t n) { return (size_t)n * 21; }
static size_t packed_out_bytes(int64_t n) { return round_up(16 + 2 * (size_t)n, 8) + 8 * (size_t)n; }

extern "C" int gs_stage_gate_packed_bytes(int64_t n_items, size_t* host_in_bytes,
                                          size_t* host_out_bytes, size_t* dev_bytes) {
  GS_REQUIRE(n_items >= 0);
  const size_t in = packed_in_bytes(n_items), out = packed_out_bytes(n_items);
  if (host_in_bytes) *host_in_bytes = in;
  if (host_out_bytes) *host_out_bytes = out;
  if (dev_bytes)
    *dev_bytes = round_up(in, 256) + round_up(out, 256) + round_up((size_t)n_items * 8 + 8, 256) +
                 step_ws_bytes(n_items);
  return GS_OK;
}

extern "C" int gs_stage_gate_packed(const double* certainty, const uint8_t* correct,
                                    int64_t n_rec, int32_t n_models, const void* host_in,
                                    int64_t n_items, double near_eps, void* host_out,
                                    void* dev_buf, size_t dev_bytes, int32_t sync,
                                    void* stream) {
  GS_REQUIRE(n_items >= 0 && host_out);
  size_t need = 0;
  gs_stage_gate_packed_bytes(n_items, nullptr, nullptr, &need);
  if (!dev_buf || dev_bytes < need) return GS_EWORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t in = packed_in_bytes(n_items), out = packed_out_bytes(n_items);
  uint8_t* d_in = static_cast<uint8_t*>(dev_buf);
  uint8_t* d_out = d_in + round_up(in, 256);
  uint8_t* d_def = d_out + round_up(out, 256);
  uint8_t* d_ws = d_def + round_up((size_t)n_items * 8 + 8, 256);
  if (n_items > 0) {
    GS_REQUIRE(host_in);
    GS_CUDA_TRY(cudaMemcpyAsync(d_in, host_in, in, cudaMemcpyHostToDevice, st));
  }
  int64_t* counts = reinterpret_cast<int64_t*>(d_out);
  const int64_t n = n_items;
  const int rc = gs_stage_gate(
      certainty, correct, n_rec, n_models, reinterpret_cast<const int64_t*>(d_in),
      reinterpret_cast<const int32_t*>(d_in + 16 * n), reinterpret_cast<const double*>(d_in + 8 * n),
      d_in + 20 * n, n, d_out + 16, d_out + 16 + n, reinterpret_cast<int64_t*>(d_def), counts,
      near_eps, reinterpret_cast<int64_t*>(d_out + round_up(16 + 2 * (size_t)n, 8)), counts + 1, d_ws,
      step_ws_bytes(n), stream);
  if (rc != GS_OK) return rc;
  GS_CUDA_TRY(cudaMemcpyAsync(host_out, d_out, out, cudaMemcpyDeviceToHost, st));
  if (sync) GS_CUDA_TRY(cudaStreamSynchronize(st));
  return GS_OK;
}
