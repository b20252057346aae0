// gs_quantile.cu — threshold-grid quantiles on the device.
//
// Reference: cascades.build_threshold_grid (/root/reference/pkg/src/
// gearserve/cascades.py:150-163) takes np.quantile(cert[:, j], k/levels)
// with numpy's default "linear" method.  numpy (lib/_function_base_impl.py,
// _quantile / _get_indexes / _lerp, pinned numpy 2.3.5) computes, for a
// sorted column a of n values:
//   v = (n - 1) * q                      virtual index (f64)
//   prev = floor(v), next = prev + 1     both -> n-1 when v >= n - 1
//   g = v - prev                         (f64; the -1 index case keeps g)
//   diff = a[next] - a[prev]
//   r = a[prev] + diff * g,  or  a[next] - diff * (1 - g) when g >= 0.5
// (separate multiplies and adds, no FMA) and returns a[n-1] (NaN) for every
// q when the column holds a NaN (NaNs sort last).  Here the column is
// gathered (any stride) into contiguous keys, sorted on the device with
// CUB's radix sort (a plain library sort, NaNs last like numpy), and one
// thread per q applies exactly that arithmetic.
#include <cub/device/device_radix_sort.cuh>

#include "gs_common.cuh"

namespace gs {
namespace {

__global__ void gather_column_kernel(const double* col, int64_t n, int64_t stride, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = col[i * stride];
    out[i] = x + 0.0;  // -0.0 -> +0.0: numpy compares them equal, CUB's key order would not
  }
}

__global__ void lerp_kernel(const double* a, int64_t n, const double* qs, int32_t n_q, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_q) return;
  if (isnan(a[n - 1])) {
    out[i] = a[n - 1];
    return;
  }
  const double q = qs[i];
  const double v = __dmul_rn((double)(n - 1), q);
  int64_t prev, next;
  const double fl = floor(v);
  if (v >= (double)(n - 1)) {
    prev = next = n - 1;
  } else if (v < 0.0) {
    prev = next = 0;
  } else {
    prev = (int64_t)fl;
    next = prev + 1;
  }
  // numpy: gamma = v - previous_indexes after the bound fix-ups (-1 / 0)
  const double prev_idx = v >= (double)(n - 1) ? -1.0 : (v < 0.0 ? 0.0 : fl);
  const double g = __dadd_rn(v, -prev_idx);
  const double lo = a[prev], hi = a[next];
  const double diff = __dadd_rn(hi, -lo);
  out[i] = g >= 0.5 ? __dadd_rn(hi, -__dmul_rn(diff, __dadd_rn(1.0, -g)))
                    : __dadd_rn(lo, __dmul_rn(diff, g));
}

size_t cub_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const double*)nullptr, (double*)nullptr, (int)n);
  return bytes;
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" int gs_quantiles_workspace(int64_t n, int32_t n_q, size_t* bytes) {
  GS_REQUIRE(bytes && n > 0 && n_q >= 0);
  if (n >= (int64_t)1 << 31) return GS_EUNSUPPORTED;
  *bytes = 2 * round_up((size_t)n * 8, 256) + round_up((size_t)n_q * 8, 256) + round_up(cub_bytes(n), 256);
  return GS_OK;
}

extern "C" int gs_quantiles(const double* column, int64_t n, int64_t stride, const double* qs,
                            int32_t n_q, double* out, void* workspace, size_t workspace_bytes,
                            void* stream) {
  GS_REQUIRE(column && n > 0 && stride >= 1 && n_q >= 0 && (n_q == 0 || (qs && out)));
  size_t need = 0;
  int rc = gs_quantiles_workspace(n, n_q, &need);
  if (rc != GS_OK) return rc;
  if (!workspace || workspace_bytes < need) return GS_EWORKSPACE;
  for (int i = 0; i < n_q; ++i)
    if (!(qs[i] >= 0.0 && qs[i] <= 1.0)) return GS_EINVAL;  // numpy: "Quantiles must be in [0, 1]"
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  double* keys = reinterpret_cast<double*>(ws);
  double* sorted = reinterpret_cast<double*>(ws + round_up((size_t)n * 8, 256));
  double* dq = reinterpret_cast<double*>(ws + 2 * round_up((size_t)n * 8, 256));
  void* tmp = ws + 2 * round_up((size_t)n * 8, 256) + round_up((size_t)n_q * 8, 256);
  size_t tmp_bytes = cub_bytes(n);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8));
  gather_column_kernel<<<(unsigned)blocks, 256, 0, st>>>(column, n, stride, keys);
  GS_LAUNCH_CHECK();
  GS_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, sorted, (int)n, 0, 64, st));
  if (n_q == 0) return GS_OK;
  GS_CUDA_TRY(cudaMemcpyAsync(dq, qs, (size_t)n_q * 8, cudaMemcpyHostToDevice, st));
  lerp_kernel<<<(n_q + 127) / 128, 128, 0, st>>>(sorted, n, dq, n_q, out);
  GS_LAUNCH_CHECK();
  return GS_OK;
}
