/*
 * gearserve_b200.h — C ABI of the B200-native CascadeServe hot path.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * passed as void*.  No torch types cross this boundary.  Functions return
 * GS_OK (0) or a negative GS_E* code; gs_strerror() names it.  The library
 * keeps no global mutable state: scratch memory is caller-owned workspace
 * whose size is queried first, so every call is re-entrant per stream.
 *
 * The reference (gearserve, pure Python) has no native code; each entry
 * point below replaces one Python function of the reference, cited by
 * file:line under /root/reference/pkg/src/gearserve/.
 */
#ifndef GEARSERVE_B200_H
#define GEARSERVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_OK 0
#define GS_EINVAL (-1)       /* malformed argument -> Python ValueError      */
#define GS_ECUDA (-2)        /* CUDA runtime error -> Python RuntimeError    */
#define GS_EWORKSPACE (-3)   /* workspace smaller than the queried size      */
#define GS_EUNSUPPORTED (-4) /* shape outside the kernel's supported range   */

#define GS_MAX_MODELS 8      /* grid path: models per validation set        */
#define GS_MAX_STAGES 64     /* list path: stages per encoded cascade        */

/* certainty kinds for gs_certainty / gs_stage_step */
#define GS_CERT_MARGIN 0      /* Eq. 5: top1 - top2 (singleton: the score)   */
#define GS_CERT_MAX_SOFTMAX 1 /* extension: max_i softmax(x)_i              */
#define GS_CERT_ENTROPY 2     /* extension: 1 - H(softmax(x)) / ln(n_cls)    */

/* score dtypes */
#define GS_F32 0
#define GS_F64 1
#define GS_BF16 2

int gs_version(void);
/* Benchmark support: write `bytes` (> L2) to evict the L2 between timed
 * steps; max_carveout != 0 runs it with the largest shared-memory carveout
 * (the sweep kernels' configuration, so no L1/smem switch at the boundary). */
int gs_flush_l2(void* buffer, size_t bytes, int32_t max_carveout, void* stream);
const char* gs_strerror(int code);
/* last CUDA error string seen by this thread (for GS_ECUDA) */
const char* gs_last_cuda_error(void);

/* ------------------------------------------------------------------------
 * List path: drop-in for kernels.evaluate_encoded (src/kernels.py:93-108),
 * same arithmetic as _evaluate_numba (src/kernels.py:39-62).
 *   certainty    [n_rec, n_models] f64 row-major
 *   correct      [n_rec, n_models] u8
 *   stage_model  [n_casc, max_len] i32, -1 padded
 *   thresholds   [n_casc, max_len] f64 (last stage unused)
 *   n_stages     [n_casc] i32
 *   cost1        [n_models] f64
 * outputs: accuracy [n_casc] f64, mean_cost [n_casc] f64,
 *          forward_frac [n_casc, max_len] f64 (padding columns = 0)
 * ---------------------------------------------------------------------- */
int gs_eval_encoded_workspace(int64_t n_rec, int32_t n_models, int64_t n_casc,
                              int32_t max_len, size_t* bytes);
int gs_eval_encoded(const double* certainty, const uint8_t* correct,
                    int64_t n_rec, int32_t n_models,
                    const int32_t* stage_model, const double* thresholds,
                    const int32_t* n_stages, int64_t n_casc, int32_t max_len,
                    const double* cost1, double* accuracy, double* mean_cost,
                    double* forward_frac, void* workspace,
                    size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Grid path: the full cascade x per-stage-threshold product over per-model
 * threshold grids (cascades.ThresholdGrid, src/cascades.py:132-163), scored
 * with the same outputs as evaluate_encoded on the enumerated cascades.
 *
 * Model columns are taken in the given order (the caller passes them cheap
 * to expensive, the order sample_cascades uses, src/cascades.py:181-182).
 * Enumeration: every non-empty model subset ("structure"), by size, then
 * lexicographically (itertools.combinations order); inside a structure the
 * threshold index tuple (k_1..k_{K-1}) is lexicographic, k_1 slowest.
 *   grids     concatenated per-model grids on the DEVICE, f64, each strictly
 *             increasing (grid_len[j] values for model j)
 *   grid_len  HOST array [n_models]
 * gs_grid_info reports the config count and the workspace the tables need
 * (n_rec < 2^30).  gs_grid_build fills the prefix tables; it must run
 * before gs_grid_eval on the same workspace.  The workspace's histogram
 * region must be zero when gs_grid_build starts and is left zero when it
 * returns; pass GS_GRID_WORKSPACE_DIRTY on the first build of a fresh (or
 * reused-for-something-else) workspace to have it zeroed first.
 * ---------------------------------------------------------------------- */
#define GS_GRID_WORKSPACE_DIRTY 1
/* Four-model path only (else GS_EUNSUPPORTED): run one of the build's two
 * passes, for timing them apart.  RECORDS_PASS is the pass over the records
 * (bucket sort into keys, or the histogram of the streamed variant) and
 * must be followed by TABLES_PASS (keys / histogram -> prefix tables) on
 * the same workspace before gs_grid_eval; neither flag = both passes. */
#define GS_GRID_BUILD_RECORDS_PASS 2
#define GS_GRID_BUILD_TABLES_PASS 4

typedef struct gs_grid_info {
  int64_t n_configs;      /* total configs of the enumeration            */
  int64_t n_cells;        /* main prefix-table cells (dims 0..M-2)       */
  int64_t side_cells;     /* side table cells (dims 0..M-4), 0 if M < 4  */
  int32_t n_structures;   /* 2^n_models - 1                              */
  int32_t max_len;        /* = n_models (forward_frac row width)         */
  size_t workspace_bytes; /* for gs_grid_build / eval                    */
  int32_t build_launches; /* kernels one gs_grid_build enqueues           */
  int32_t eval_launches;  /* kernels one full-range gs_grid_eval enqueues */
  int32_t fast_path;      /* four-model packed path (n_rec < 2^21): 1,   */
                          /* 2 when gs_grid_build takes the bucket-sort  */
                          /* kernels (grid_len[1] < 1024, shared-memory  */
                          /* plan fits); 0: general path                 */
  int32_t reserved;
} gs_grid_info;

int gs_grid_plan(int64_t n_rec, int32_t n_models, const int32_t* grid_len,
                 gs_grid_info* info);
int gs_grid_build(const double* certainty, const uint8_t* correct,
                  int64_t n_rec, int32_t n_models, const double* grids,
                  const int32_t* grid_len, void* workspace,
                  size_t workspace_bytes, int32_t flags, void* stream);
/* Streamed build (gs_grid_info.fast_path != 0 only, else GS_EUNSUPPORTED):
 * gs_grid_accumulate adds the n_chunk records at certainty / correct (a
 * slice of the n_rec-record validation set) to the histogram, so host->device
 * copies of later slices overlap the binning of earlier ones;
 * gs_grid_finish turns the histogram of all n_rec records into the prefix
 * tables.  gs_grid_build == gs_grid_accumulate(all) + gs_grid_finish.  The
 * flags of the first accumulate of a build are those of gs_grid_build. */
int gs_grid_accumulate(const double* certainty, const uint8_t* correct,
                       int64_t n_chunk, int64_t n_rec, int32_t n_models,
                       const double* grids, const int32_t* grid_len,
                       void* workspace, size_t workspace_bytes, int32_t flags,
                       void* stream);
int gs_grid_finish(int64_t n_rec, int32_t n_models, const int32_t* grid_len,
                   void* workspace, size_t workspace_bytes, void* stream);
/* Many small three-model sweeps in one launch (config 1 stacked: the
 * reference's CPU default is launch-bound alone).  n_sets validation sets of
 * n_rec records each, certainty [n_sets][n_rec][3] f64 and correct
 * [n_sets][n_rec][3] u8 row-major on the DEVICE, per-set grids
 * [n_sets][grid_len[0] + grid_len[1] + grid_len[2]] f64 on the DEVICE (each
 * strictly increasing), grid_len [3] on the HOST, cost1 [3] on the DEVICE.
 * Outputs [n_sets][C] (accuracy, mean_cost) and [n_sets][C][3]
 * (forward_frac), C = 3 + 2 g0 + g1 + g0 g1, every config of each set's
 * enumeration in gs_grid_eval's order and with its values.  GS_EUNSUPPORTED
 * unless n_models == 3, (g0 + 1)(g1 + 1) <= 12800 and n_rec < 2^31. */
int gs_grid_sweep_batched(const double* certainty, const uint8_t* correct,
                          int64_t n_sets, int64_t n_rec, int32_t n_models,
                          const double* grids, const int32_t* grid_len,
                          const double* cost1, double* accuracy, double* mean_cost,
                          double* forward_frac, void* stream);
/* Score configs [config_begin, config_begin + config_count).  Any output
 * pointer may be NULL to skip it.  n_correct receives the integer correct
 * count (accuracy * n_rec) used by the exact Pareto reduction. */
int gs_grid_eval(int64_t n_rec, int32_t n_models, const int32_t* grid_len,
                 const double* cost1, int64_t config_begin,
                 int64_t config_count, double* accuracy, double* mean_cost,
                 double* forward_frac, uint32_t* n_correct,
                 const void* workspace, size_t workspace_bytes, void* stream);
/* Decode config indices into the encoded-cascade form of
 * cascades.encode_cascades (src/cascades.py:66-79): stage_model (-1 pad),
 * thresholds (grid values, 0 pad), n_stages.  max_len = n_models. */
int gs_grid_decode(int32_t n_models, const int32_t* grid_len,
                   const double* grids, const int64_t* config_idx,
                   int64_t count, int32_t* stage_model, double* thresholds,
                   int32_t* n_stages, void* stream);

/* ------------------------------------------------------------------------
 * Pareto front, semantics of cascades.pareto_filter (src/cascades.py:116-129):
 * keep items no other item dominates (acc >=, cost <=, one strict); exact
 * ties survive; output in input order.
 *
 * gs_pareto_counts: accuracy given as integer correct counts in [0, n_rec]
 * (division by the same n_rec is monotone, so this is exact).  O(n + n_rec).
 * Writes keep[n] (optional) and the kept indices (ascending, + base_index)
 * to kept_idx with their count to *n_kept (device int64).
 * gs_pareto_generic: float accuracies, O(n^2) tiled; for small lists.
 * ---------------------------------------------------------------------- */
int gs_pareto_counts_workspace(int64_t n, int64_t n_rec, size_t* bytes);
int gs_pareto_counts(const uint32_t* n_correct, const double* cost, int64_t n,
                     int64_t n_rec, int64_t base_index, uint8_t* keep,
                     int64_t* kept_idx, int64_t* n_kept, void* workspace,
                     size_t workspace_bytes, void* stream);
int gs_pareto_generic(const double* accuracy, const double* cost, int64_t n,
                      uint8_t* keep, void* stream);

/* ------------------------------------------------------------------------
 * Certainty of score rows: cascades.certainty (src/cascades.py:20-28) for
 * GS_CERT_MARGIN, bit-exact (top two found in the source dtype, subtracted
 * in f64; a row of length 1 returns its score).  row_len (optional, device
 * i32 [n_rows]) gives ragged row lengths <= n_cls (0 -> GS_EINVAL).
 * ---------------------------------------------------------------------- */
int gs_certainty(const void* scores, int32_t dtype, int64_t n_rows,
                 int32_t n_cls, int64_t row_stride, const int32_t* row_len,
                 int32_t kind, double* cert_out, void* stream);

/* ------------------------------------------------------------------------
 * Online stage step (EngineState.finish_batch gate, src/engine.py:355-383):
 * certainty of each row's logits -> gate (last || cert >= thr, inclusive)
 * -> stable compaction of deferred rows in batch order -> optional gather of
 * the deferred rows' payload into the next stage's contiguous buffer.
 *   thr       [n_rows] f64 per-row threshold (rows may carry different gears)
 *   is_last   [n_rows] u8 (NULL = none last)
 *   cert_out  [n_rows] f64 (optional), stop_out [n_rows] u8 (optional)
 *   deferred_idx [n_rows] i64 capacity; *n_deferred (device i64)
 *   near_idx  rows with |cert - thr| <= near_eps (non-last), ascending,
 *             *n_near (device i64); NULL to skip
 *   payload / next_payload: row-major, payload_row_bytes each (NULL to skip)
 * ---------------------------------------------------------------------- */
int gs_stage_step_workspace(int64_t n_rows, size_t* bytes);
int gs_stage_step(const void* scores, int32_t dtype, int64_t n_rows,
                  int32_t n_cls, int64_t row_stride, int32_t kind,
                  const double* thr, const uint8_t* is_last, double* cert_out,
                  uint8_t* stop_out, int64_t* deferred_idx,
                  int64_t* n_deferred, double near_eps, int64_t* near_idx,
                  int64_t* n_near, const void* payload,
                  int64_t payload_row_bytes, void* next_payload,
                  void* workspace, size_t workspace_bytes, void* stream);

/* Gate over precomputed certainty matrices (the engine's CompiledPlan.cert /
 * corr, src/engine.py:217): item i looks up cert[row[i], model[i]].  Writes
 * stop[i], correct[i] (= corr[row, model] for stopped items, else 0) and the
 * deferred item positions in batch order. */
int gs_stage_gate(const double* certainty, const uint8_t* correct,
                  int64_t n_rec, int32_t n_models, const int64_t* row,
                  const int32_t* model, const double* thr,
                  const uint8_t* is_last, int64_t n_items, uint8_t* stop_out,
                  uint8_t* correct_out, int64_t* deferred_idx,
                  int64_t* n_deferred, double near_eps, int64_t* near_idx,
                  int64_t* n_near, void* workspace, size_t workspace_bytes,
                  void* stream);

/* The same gate for one small online batch (EngineState.finish_batch on a
 * batch of <= max_profiled_batch items, src/engine.py:355-383) as ONE call:
 * one H2D of the packed items, the gate, one D2H of the packed outcome.
 *   host_in  (pinned) {row i64[n], thr f64[n], model i32[n], is_last u8[n]}
 *   host_out (pinned) {n_deferred i64, n_near i64, stop u8[n], correct u8[n],
 *                      pad to 8, near i64[n]}
 *   dev_buf  device scratch of gs_stage_gate_packed_bytes(n).dev_bytes
 *   sync     != 0: cudaStreamSynchronize before returning (host_out valid) */
int gs_stage_gate_packed_bytes(int64_t n_items, size_t* host_in_bytes,
                               size_t* host_out_bytes, size_t* dev_bytes);
int gs_stage_gate_packed(const double* certainty, const uint8_t* correct,
                         int64_t n_rec, int32_t n_models, const void* host_in,
                         int64_t n_items, double near_eps, void* host_out,
                         void* dev_buf, size_t dev_bytes, int32_t sync,
                         void* stream);




/* ------------------------------------------------------------------------
 * Config 4a: the exact Pareto front (cascades.pareto_filter semantics, exact
 * ties kept, src/cascades.py:116-129) of the full five-model cascade
 * m0 -> m1 -> m2 -> m3 -> m4 over every threshold tuple (k0, k1, k2, k3) of
 * grids of up to 1023 values (~1e12 configs at 1000 levels), each config
 * scored like _evaluate_numba (src/kernels.py:39-62) but never written out.
 * certainty [n, 5] f64, correct [n, 5] u8 on the device, n < 2^21; grids:
 * device, models 0..3 concatenated; grid_len HOST [5].  Config index =
 * ((k0 g1 + k1) g2 + k2) g3 + k3.
 *   prepare: bins, records sorted by (b2, b0), side tables; resets the
 *            per-accuracy minimum costs (mincost, int64 order-preserving
 *            cost bits at workspace + mincost_offset, n + 1 entries).
 *   pass1:   k0 in [k0_begin, k0_end): lowers mincost, and flags (a bit per
 *            row (k0, k1, k2) in the workspace, g0 g1 ceil(g2/32) words)
 *            the rows holding a config at or below mincost as it stood.
 *            Sharded runs reduce mincost with MIN across ranks before
 *            select.
 *   select:  the front's accuracies and cost keys; *n_front (device) = how
 *            many distinct accuracies it has.
 *   pass2:   k0 in [k0_begin, k0_end) (only the rows pass 1 flagged, for
 *            the k0 pass 1 walked: every front config's row is one; other
 *            k0 in full): every config on the front, in no
 *            order: out_index [cap] config index, out_cost [cap] mean cost,
 *            out_counts [cap][6] {correct, n, reach after stages 0..3};
 *            *out_n (device, zero it first) the count (may exceed cap);
 *            out_cap = 0: no list, only the per-accuracy summary (ties,
 *            min_index) -- routing-equivalent threshold tuples tie, and a
 *            1000-level front can hold 1e9 configs.
 * ---------------------------------------------------------------------- */
typedef struct gs_front5_info {
  int64_t n_configs;        /* g0 g1 g2 g3                                */
  size_t workspace_bytes;
  size_t mincost_offset;    /* byte offset of mincost in the workspace    */
  size_t front_offset;      /* after select: int64 [n + 1] the front point's
                               cost key per accuracy, or 0x7f7f7f7f7f7f7f7f */
  size_t ties_offset;       /* after pass2: u64 [n + 1] front configs per
                               accuracy (tied configs all counted)          */
  size_t min_index_offset;  /* after pass2: u64 [n + 1] their smallest index */
  int32_t k0_count;         /* g0: the k0 values to shard                 */
  int32_t bucket_shift;
} gs_front5_info;

int gs_front5_plan(int64_t n_rec, const int32_t* grid_len, gs_front5_info* info);
int gs_front5_prepare(const double* certainty, const uint8_t* correct, int64_t n_rec,
                      const double* grids, const int32_t* grid_len, void* workspace,
                      size_t workspace_bytes, void* stream);
int gs_front5_pass1(int64_t n_rec, const int32_t* grid_len, const double* cost1,
                    int32_t k0_begin, int32_t k0_end, void* workspace,
                    size_t workspace_bytes, void* stream);
int gs_front5_select(int64_t n_rec, const int32_t* grid_len, void* workspace,
                     size_t workspace_bytes, unsigned long long* n_front, void* stream);
int gs_front5_pass2(int64_t n_rec, const int32_t* grid_len, const double* cost1,
                    int32_t k0_begin, int32_t k0_end, void* workspace,
                    size_t workspace_bytes, unsigned long long* out_index,
                    double* out_cost, uint32_t* out_counts, unsigned long long* out_n,
                    int64_t out_cap, void* stream);

/* ------------------------------------------------------------------------
 * SP1's cascade sampler (cascades.sample_cascades, src/cascades.py:166-193)
 * on the device: numpy default_rng(seed)'s draws reproduced exactly, every
 * singleton first, duplicates dropped in order.  One job per seed, one warp
 * each.  order: device [n_models] model column of each cost rank (models
 * sorted by (runtime_table[1], index)); grids: device, concatenated per model
 * column, grid_off device [n_models + 1] (each grid < 65536 values).
 * Outputs per job (capacity n_models + n_samples rows): stage_model /
 * thresholds / n_stages in evaluate_encoded's encoding, grid_index (each
 * non-final stage's threshold index into its grid, -1 pad).  table: zeroed
 * scratch of 2 * table_cap u64, table_cap a power of two >= 2 * capacity.
 * ---------------------------------------------------------------------- */
typedef struct gs_sampler_job {
  uint64_t rng_state_hi, rng_state_lo, rng_inc_hi, rng_inc_lo;
  uint32_t rng_has_uint32, rng_uinteger;
  int64_t n_samples;
  int32_t* stage_model;          /* [cap, n_models]                        */
  double* thresholds;            /* [cap, n_models]                        */
  int32_t* n_stages;             /* [cap]                                  */
  int32_t* grid_index;           /* [cap, n_models]                        */
  uint64_t* table;               /* [2 * table_cap], zero on entry         */
  int64_t table_cap;
  int64_t* result;               /* [5]: count, rng state hi, lo, has_uint32, uinteger */
} gs_sampler_job;

int gs_sample_cascades(int32_t n_models, const int32_t* order, const double* grids,
                       const int32_t* grid_off, const gs_sampler_job* jobs,
                       int32_t n_jobs, void* stream);

/* ------------------------------------------------------------------------
 * Replay engine: engine.run (src/engine.py:452-520) in virtual-clock mode on
 * the device, for many independent runs per launch (config-5 trace replays,
 * the planner's simulator probes src/planner.py:293-356).  Each run is one
 * sequential event loop -- arrivals (EngineState.submit :299-319), batch
 * completions (finish_batch :355-383: the certainty gate and the replica
 * draws), measurement ticks (tick / maybe_switch_gear :389-410, :123-133)
 * and dispatch (scan_device / choose_dispatch :321-353, :248-253) -- with
 * numpy's PCG64 stream reproduced on the device, so records, windows,
 * queues and the final generator state equal the reference's.
 * ---------------------------------------------------------------------- */
typedef struct gs_engine_plan {
  const double* cert;            /* [n_records, n_cols] CompiledPlan.cert  */
  const uint8_t* corr;           /* [n_records, n_cols] CompiledPlan.corr  */
  int64_t n_records;
  int32_t n_cols;                /* models (profile order)                 */
  int32_t n_replicas;            /* <= GS_ENGINE_MAX_REPLICAS              */
  int32_t n_devices;             /* <= GS_ENGINE_MAX_DEVICES               */
  int32_t n_gears;
  int32_t max_stages;            /* L                                      */
  int32_t batch_cap;             /* max over models of max_profiled_batch  */
  const int32_t* replica_device; /* [R]                                    */
  const int32_t* replica_model;  /* [R] model column                       */
  const int32_t* replica_rank;   /* [R] rank of replica_id in string order */
  const int32_t* model_max_batch;  /* [n_cols]                             */
  const int64_t* model_runtime_us; /* [n_cols][batch_cap + 1]              */
  const int32_t* gear_n_stages;  /* [G]                                    */
  const int32_t* gear_model;     /* [G][L]                                 */
  const double* gear_thr;        /* [G][L] (last stage unused)             */
  const int32_t* gear_rep_off;   /* [G][L + 1] CSR offsets                 */
  const int32_t* gear_rep;       /* replica index per CSR entry            */
  const double* gear_cum;        /* np.cumsum of the load weights, per entry */
  const int32_t* gear_min_qlen;  /* [G][R] Gear.min_queue_length (default 1) */
  double qps_max;
} gs_engine_plan;

#define GS_ENGINE_MAX_REPLICAS 256
#define GS_ENGINE_MAX_DEVICES 64

typedef struct gs_engine_record { /* RequestRecord (src/engine.py:49-56)   */
  int64_t completion_us;
  int32_t request_id;            /* arrival index; arrival_us = arrivals[id] */
  uint8_t stages_executed;
  uint8_t correct;
  uint16_t gear_index;
} gs_engine_record;

typedef struct gs_engine_window { /* WindowRecord (src/engine.py:59-73)    */
  int64_t end_us;
  double measured_qps;
  int32_t first_stage_queue_len, gear_before, candidate_gear, gear_after;
  int64_t completed;
  int64_t p95_us;                /* -1: None                               */
  double accuracy;               /* NaN: None                              */
} gs_engine_window;

typedef struct gs_engine_job {
  const gs_engine_plan* plan;    /* device pointer                         */
  const int64_t* arrivals;       /* device [n_arrivals], non-decreasing    */
  int64_t n_arrivals;
  int64_t horizon_us;            /* WorkloadTrace.duration_us              */
  uint64_t rng_state_hi, rng_state_lo, rng_inc_hi, rng_inc_lo;
  uint32_t rng_has_uint32, rng_uinteger;   /* PCG64 bit_generator.state    */
  int32_t initial_gear;
  int32_t enable_ticks;
  int64_t measure_period_us;
  double alpha;
  uint64_t* rings;               /* scratch [n_replicas][ring_cap]: the queues */
  int64_t ring_cap;              /* >= n_arrivals (a queue never holds more) */
  int64_t* scratch;              /* scratch [n_arrivals] (window latencies) */
  gs_engine_record* records;     /* out [n_arrivals], completion order     */
  gs_engine_window* windows;     /* out [windows_cap]                      */
  int64_t windows_cap;
  int64_t* model_batches;        /* out [n_cols][batch_cap + 1]            */
  int64_t* replica_counts;       /* out [R][2]: routed arrivals, queue length at horizon */
  int64_t* result;               /* out [8]: arrivals, completed, in_flight,
                                    windows, rng state hi, lo, has_uint32, uinteger */
} gs_engine_job;

/* jobs: device array of n_jobs descriptors; one warp per job.  Replica ids
 * are ranked in replica_rank; n_replicas <= 256 (the dispatch key holds the
 * replica index in 8 bits) and arrival indices < 2^32. */
int gs_engine_run(const gs_engine_job* jobs, int32_t n_jobs, void* stream);

/* ------------------------------------------------------------------------
 * Threshold-grid quantiles on the device: np.quantile(column, qs) with
 * numpy's default "linear" method, bit-exact (cascades.build_threshold_grid,
 * src/cascades.py:150-163).  column: device f64, n values at `stride`
 * elements apart (a column of a row-major [n, M] matrix: stride = M);
 * qs: HOST array of n_q values in [0, 1]; out: device f64 [n_q].
 * ---------------------------------------------------------------------- */
/* ------------------------------------------------------------------------
 * A cascade stage's classifier head on the tensor cores, fused with the
 * stage step's certainty (north_star's tensor-core use; the reference runs a
 * model and then cascades.certainty on its scores, src/serving.py:79-97,
 * src/cascades.py:20-28): logits = features @ weight^T (+ bias) by
 * tcgen05.mma (bf16 in, f32 in TMEM), each row's certainty over the n_cls
 * logits in the epilogue; the logits never reach HBM unless logits_out.
 *   features  [n_rows, n_feat] bf16 row-major, 16-byte aligned
 *   weight    [n_cls, n_feat] bf16 row-major (nn.Linear layout), aligned
 *   bias      [n_cls] f32 or NULL;  n_feat % 64 == 0
 *   kind      GS_CERT_MARGIN / GS_CERT_MAX_SOFTMAX / GS_CERT_ENTROPY
 *   cert_out  [n_rows] f64;  logits_out [n_rows, n_cls] f32 or NULL
 * ---------------------------------------------------------------------- */
int gs_head_certainty(const void* features, const void* weight, const float* bias,
                      int64_t n_rows, int32_t n_cls, int32_t n_feat, int32_t kind,
                      double* cert_out, float* logits_out, void* stream);

int gs_quantiles_workspace(int64_t n, int32_t n_q, size_t* bytes);
int gs_quantiles(const double* column, int64_t n, int64_t stride,
                 const double* qs, int32_t n_q, double* out, void* workspace,
                 size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Validation ingest (host code, no GPU): the reference's validation JSONL
 * (formats.load_validation, src/formats.py:75-97) parsed into columnar
 * arrays with n_threads host threads.  gs_jsonl_open parses the file into a
 * handle and reports the shape (or the failing 1-based line and a message);
 * gs_jsonl_read fills caller arrays: sample_id [n], line_no [n] (optional),
 * scores[m] -> [n, width[m]] f64 (zero padded), row_len [n, M] i32,
 * correct [n, M] u8; gs_jsonl_close frees the handle.
 * ---------------------------------------------------------------------- */
#define GS_JSONL_MAX_MODELS 64

typedef struct gs_jsonl_info {
  int64_t n_records;
  int32_t n_models;
  int32_t width[GS_JSONL_MAX_MODELS];   /* max score-list length per model */
  char model_ids[GS_JSONL_MAX_MODELS][64]; /* first record's key order  */
  int64_t err_line;                     /* 1-based, 0 = no line        */
  char error[256];
} gs_jsonl_info;

int gs_jsonl_open(const char* path, int32_t n_threads, void** handle,
                  gs_jsonl_info* info);
int gs_jsonl_read(void* handle, int64_t* sample_id, int64_t* line_no,
                  double* const* scores, int32_t* row_len, uint8_t* correct);
void gs_jsonl_close(void* handle);

#ifdef __cplusplus
}
#endif
#endif /* GEARSERVE_B200_H */
