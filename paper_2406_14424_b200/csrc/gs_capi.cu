// gs_capi.cu — library-wide C ABI entry points (version, error strings).
#include <atomic>

#include "gs_common.cuh"

namespace gs {

static thread_local const char* t_last_cuda_error = "no error";

void set_cuda_error(cudaError_t e) { t_last_cuda_error = cudaGetErrorString(e); }

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  return dev;
}

int sm_count() {
  static std::atomic<int> cached[kMaxDevices];  // per device, 0 = not read yet
  const int dev = current_device();
  std::atomic<int>* slot = dev < kMaxDevices ? &cached[dev] : nullptr;
  int v = slot ? slot->load(std::memory_order_relaxed) : 0;
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
    v = 148;
  if (slot) slot->store(v, std::memory_order_relaxed);
  return v;
}

}  // namespace gs

extern "C" {

int gs_version(void) { return 1; }

const char* gs_strerror(int code) {
  switch (code) {
    case GS_OK:
      return "ok";
    case GS_EINVAL:
      return "invalid argument";
    case GS_ECUDA:
      return "CUDA error";
    case GS_EWORKSPACE:
      return "workspace too small";
    case GS_EUNSUPPORTED:
      return "unsupported shape";
    default:
      return "unknown error";
  }
}

const char* gs_last_cuda_error(void) { return gs::t_last_cuda_error; }

}  // extern "C"

// ------------------------------------------------------------ L2 flush --
// Benchmark support: evict the L2 between timed steps by writing `bytes`
// (> the 126 MB L2) with 16-byte stores.  The kernel asks for the largest
// shared-memory carveout, like the sweep kernels, so the SMs do not switch
// their L1 / shared-memory split at the step boundary (a generic fill kernel
// runs with the default split, and the next kernel needing 200+ KB of shared
// memory waits for the reconfiguration).
namespace gs {
namespace {
__global__ void __launch_bounds__(512) flush_kernel(uint4* buf, size_t n16, uint32_t v) {
  const uint4 w = make_uint4(v, v, v, v);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    buf[i] = w;
}
}  // namespace
}  // namespace gs

extern "C" int gs_flush_l2(void* buffer, size_t bytes, int32_t max_carveout, void* stream) {
  GS_REQUIRE(buffer && bytes >= 16);
  static gs::SmemAttr carve;  // (unused size slot: the carveout is set once per device)
  if (max_carveout) {
    const int dev = gs::current_device();
    if (dev < gs::kMaxDevices && carve.bytes[dev].load() == 0) {
      GS_CUDA_TRY(cudaFuncSetAttribute(gs::flush_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       100));
      carve.bytes[dev].store(1);
    }
  }
  gs::flush_kernel<<<(unsigned)(gs::sm_count() * 4), 512, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint4*>(buffer), bytes / 16, 0u);
  GS_LAUNCH_CHECK();
  return GS_OK;
}
