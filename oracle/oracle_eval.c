/*
 * oracle_eval.c — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C restatement of the reference's cascade walk, used as the parity
 * checker in tests/, by __graft_entry__.smoke(), and as bench.py's
 * cpu_baseline / --impl reference arm.  Compiled with -ffp-contract=off so
 * a*b+c is never fused, matching numba's default (no fastmath).
 *
 * oracle_evaluate_encoded restates _evaluate_numba
 *   /root/reference/pkg/src/gearserve/kernels.py:39-62
 * step for step: visits counted (the reference's f64 `+= 1.0`, :52, holds
 * the same exact integers; counted here as int64), stop test
 * `s == ns-1 || certainty[r, m] >= thresholds[c, s]` (:53), correct added as
 * an integer (:54), epilogue frac = count / n_rec, mean_cost += frac *
 * cost1[m] in stage order, accuracy = n_correct / n_rec (:57-61).
 * Configs are independent, so the outer loop may be split
 * over threads without changing any result.
 *
 * oracle_grid_configs enumerates the full cascade x threshold-grid product
 * in the order gridsweep.py documents, producing encoded cascades in the
 * layout of cascades.encode_cascades (src/cascades.py:66-79).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

static void eval_one(const double* restrict cert, const uint8_t* restrict corr, int64_t n_rec,
                     int32_t M, const int32_t* restrict sm, const double* restrict thr, int32_t ns,
                     int32_t L, const double* restrict cost1, double* restrict acc,
                     double* restrict cost, double* restrict frac) {
  /* visits are counted as integers and converted once: the reference's
     f64 `+= 1.0` holds the same exact integers (< 2^53) */
  int64_t visits[64] = {0};
  int64_t n_correct = 0;
  for (int64_t r = 0; r < n_rec; ++r) {
    const double* row = cert + r * M;
    const uint8_t* krow = corr + r * M;
    for (int32_t s = 0; s < ns; ++s) {
      const int32_t m = sm[s];
      visits[s] += 1;
      if (s == ns - 1 || row[m] >= thr[s]) {
        n_correct += krow[m];
        break;
      }
    }
  }
  for (int32_t s = 0; s < L; ++s) frac[s] = 0.0;
  double mean = 0.0;
  for (int32_t s = 0; s < ns; ++s) {
    const double f = (double)visits[s] / (double)n_rec;
    frac[s] = f;
    mean += f * cost1[sm[s]];
  }
  *cost = mean;
  *acc = (double)n_correct / (double)n_rec;
}

void oracle_evaluate_encoded(const double* cert, const uint8_t* corr, int64_t n_rec, int32_t M,
                             const int32_t* stage_model, const double* thresholds,
                             const int32_t* n_stages, int64_t n_casc, int32_t L,
                             const double* cost1, double* accuracy, double* mean_cost,
                             double* forward_frac, int32_t n_threads) {
#ifdef _OPENMP
  if (n_threads < 1) n_threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads)
#endif
  for (int64_t c = 0; c < n_casc; ++c) {
    eval_one(cert, corr, n_rec, M, stage_model + c * L, thresholds + c * L, n_stages[c], L,
             cost1, accuracy + c, mean_cost + c, forward_frac + c * L);
  }
}

/* Structures: non-empty subsets by size then lexicographic. */
int64_t oracle_grid_n_configs(int32_t M, const int32_t* glen) {
  int64_t total = 0;
  for (uint32_t mask = 1; mask < (1u << M); ++mask) {
    int64_t n = 1;
    int last = -1;
    for (int j = 0; j < M; ++j)
      if (mask >> j & 1u) last = j;
    for (int j = 0; j < last; ++j)
      if (mask >> j & 1u) n *= glen[j];
    total += n;
  }
  return total;
}

/* Write configs [begin, begin+count) as encoded cascades (width M). */
int oracle_grid_configs(int32_t M, const int32_t* glen, const double* grids, int64_t begin,
                        int64_t count, int32_t* stage_model, double* thresholds,
                        int32_t* n_stages) {
  int32_t goff[32];
  int off = 0;
  for (int j = 0; j < M; ++j) {
    goff[j] = off;
    off += glen[j];
  }
  int64_t base = 0, written = 0;
  for (int K = 1; K <= M && written < count; ++K) {
    int idx[32];
    for (int i = 0; i < K; ++i) idx[i] = i;
    while (1) {
      int64_t n = 1;
      for (int i = 0; i + 1 < K; ++i) n *= glen[idx[i]];
      /* configs [base, base+n) belong to this structure */
      for (int64_t local = 0; local < n; ++local) {
        const int64_t c = base + local;
        if (c >= begin + count) return 0;
        if (c < begin) {
          local = begin - base - 1; /* skip ahead */
          continue;
        }
        const int64_t o = c - begin;
        int64_t rem = local;
        int k[32];
        for (int t = K - 2; t >= 0; --t) {
          k[t] = (int)(rem % glen[idx[t]]);
          rem /= glen[idx[t]];
        }
        for (int t = 0; t < M; ++t) {
          stage_model[o * M + t] = t < K ? idx[t] : -1;
          thresholds[o * M + t] = (t < K - 1) ? grids[goff[idx[t]] + k[t]] : 0.0;
        }
        n_stages[o] = K;
        ++written;
      }
      base += n;
      int i = K - 1;
      while (i >= 0 && idx[i] == M - K + i) --i;
      if (i < 0) break;
      ++idx[i];
      for (int q = i + 1; q < K; ++q) idx[q] = idx[q - 1] + 1;
    }
  }
  return 0;
}
