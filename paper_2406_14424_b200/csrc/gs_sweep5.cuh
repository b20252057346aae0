// gs_sweep5.cuh — host interface of the five-model grid-sweep path
// (gs_sweep5.cu), used by gs_grid_build / gs_grid_eval in gs_sweep.cu.
#pragma once

#include <algorithm>

#include "gs_common.cuh"

namespace gs {

struct W5Layout {
  int32_t d0, d1, d2, d3;        // table dims (grid length + 1)
  int64_t cells2, cellsF;        // (b0, b1) slabs; full table cells
  size_t offTmp, offKeys, offCnt, offHP, offOff, offCur, offP, offT, offFaces, bytes;
};

bool w5_supported(int64_t n_rec, int32_t n_models, const int32_t* grid_len);
W5Layout w5_layout(const int32_t* grid_len, int64_t n_rec);
// build: bins, slab sort, side table P, and T (F without the b0 prefix)
cudaError_t w5_build(const double* cert, const uint8_t* corr, int64_t n_rec, const double* grids,
                     const int32_t* grid_len, uint8_t* workspace, bool dirty, cudaStream_t st);
// the b0 walk: scores the full cascade's configs in [cfg_begin, +cfg_count)
// and writes the face cells of F (for the other structures' regular eval)
cudaError_t w5_walk(int64_t n_rec, const int32_t* grid_len, int64_t full_begin, const double* cost1,
                    int64_t cfg_begin, int64_t cfg_count, double* acc, double* cost, double* frac,
                    uint32_t* n_correct, const uint8_t* workspace, cudaStream_t st);

}  // namespace gs
