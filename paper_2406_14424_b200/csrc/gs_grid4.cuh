// gs_grid4.cuh — host interface of the four-model grid-sweep fast path
// (gs_grid4.cu), used by gs_grid_build / gs_grid_eval in gs_sweep.cu.
#pragma once

#include "gs_common.cuh"

namespace gs {

constexpr int64_t kGrid4MaxRec = 1ll << 21;      // 21-bit packed count fields
constexpr size_t kGrid4SlabMax = 200 * 1024;      // one (b1, b2) slab in shared memory

struct Grid4Layout {
  int32_t d0, d1, d2, d2p, d1p;  // table dims (grid length + 1), padded pitches
  int32_t hp;                    // histogram row pitch (odd)
  int32_t nb, max_parts;         // sorted build: buckets (one per b1), record ranges
  int32_t W, nbk;                // eval units: column blocks of W columns, nbk per b0 slab
  bool sorted;                   // one-shot builds take the bucket-sort kernels
  size_t offH, offG0, offS, offGt, offR1, offP0, offCnt, offKeys, offOff, bytes;
};

bool grid4_supported(int64_t n_rec, int32_t n_models, const int32_t* grid_len);
Grid4Layout grid4_layout(const int32_t* grid_len, int64_t n_rec);
// accumulate: add n_chunk records to the histogram; finish: prefix tables
cudaError_t grid4_accumulate(const double* cert, const uint8_t* corr, int64_t n_chunk,
                             const double* grids, const int32_t* grid_len, uint8_t* workspace,
                             bool dirty, cudaStream_t st);
cudaError_t grid4_finish(const int32_t* grid_len, uint8_t* workspace, cudaStream_t st);
// passes: bit 0 the records pass, bit 1 the tables pass (3 = the whole build)
cudaError_t grid4_build(const double* cert, const uint8_t* corr, int64_t n_rec, const double* grids,
                        const int32_t* grid_len, uint8_t* workspace, bool dirty, int passes,
                        cudaStream_t st);
cudaError_t grid4_eval(int64_t n_rec, const int32_t* grid_len, const int64_t* struct_begin,
                       const uint32_t* struct_mask, int n_struct, const double* cost1,
                       int64_t cfg_begin, int64_t cfg_count, double* acc, double* cost,
                       double* frac, uint32_t* n_correct, const uint8_t* workspace,
                       cudaStream_t st);

}  // namespace gs
