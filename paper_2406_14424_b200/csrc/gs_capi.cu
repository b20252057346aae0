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
