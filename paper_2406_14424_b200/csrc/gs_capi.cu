// gs_capi.cu — library-wide C ABI entry points (version, error strings).
#include <atomic>

#include "gs_common.cuh"

namespace gs {

static thread_local const char* t_last_cuda_error = "no error";

void set_cuda_error(cudaError_t e) { t_last_cuda_error = cudaGetErrorString(e); }

int sm_count() {
  static std::atomic<int> cached{0};
  int v = cached.load(std::memory_order_relaxed);
  if (v > 0) return v;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
    v = 148;
  cached.store(v, std::memory_order_relaxed);
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
