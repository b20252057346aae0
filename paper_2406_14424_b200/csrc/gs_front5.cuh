// gs_front5.cuh — host interface of the config-4a Pareto-front path
// (gs_front5.cu).
#pragma once

#include <algorithm>

#include "gs_common.cuh"

namespace gs {

struct F5Layout {
  int32_t d0, d1, d2, d3, bucket_shift;
  size_t offTmp, offKeys, offPre02, offCur, offBstart, offS01, offC0, offMin, offFront, offGbest,
      offNFront, offTies, offMinIdx, offRowFlag, offK0Done, bytes;
  int32_t n_words;  // row-flag words per (k0, k1): ceil(g2 / 32)
};

bool f5_supported(int64_t n_rec, const int32_t* grid_len);
F5Layout f5_layout(const int32_t* grid_len, int64_t n_rec);
cudaError_t f5_prepare(const double* cert, const uint8_t* corr, int64_t n_rec, const double* grids,
                       const int32_t* grid_len, uint8_t* ws, cudaStream_t st);
cudaError_t f5_pass1(const int32_t* grid_len, int64_t n_rec, const double* cost1, uint8_t* ws,
                     int k0_begin, int k0_end, cudaStream_t st);
cudaError_t f5_select(const int32_t* grid_len, int64_t n_rec, uint8_t* ws,
                      unsigned long long* n_front, cudaStream_t st);
cudaError_t f5_pass2(const int32_t* grid_len, int64_t n_rec, const double* cost1, uint8_t* ws,
                     int k0_begin, int k0_end, unsigned long long* out_idx, double* out_cost,
                     uint32_t* out_rec, unsigned long long* out_count, int64_t out_cap,
                     cudaStream_t st);

}  // namespace gs
