// micro_store.cu — output-store patterns and TMA bulk-copy granularity on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_store tools/micro_store.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int C = 1 << 20;  // configs

// store patterns: frac[C][4] f64, cost[C], acc[C], nc[C]
template <int MODE>
__global__ void __launch_bounds__(512) k_store(double* frac, double* cost, double* acc, uint32_t* nc) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < C; i += stride) {
    const double v = (double)i;
    if (MODE == 0) {  // two 16-byte stores per config (current kernels)
      double2* row = reinterpret_cast<double2*>(frac + 4ll * i);
      row[0] = make_double2(v, v + 1);
      row[1] = make_double2(v + 2, v + 3);
    } else if (MODE == 1) {  // one 32-byte store per config
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(frac + 4ll * i), "d"(v),
                   "d"(v + 1), "d"(v + 2), "d"(v + 3)
                   : "memory");
    }
    if (MODE <= 1) {
      cost[i] = v;
      acc[i] = v;
      nc[i] = i;
    }
    if (MODE == 2) {  // frac only, 16-byte stores
      double2* row = reinterpret_cast<double2*>(frac + 4ll * i);
      row[0] = make_double2(v, v + 1);
      row[1] = make_double2(v + 2, v + 3);
    }
    if (MODE == 3)  // frac only, 32-byte stores
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(frac + 4ll * i), "d"(v),
                   "d"(v + 1), "d"(v + 2), "d"(v + 3)
                   : "memory");
    if (MODE == 4) reinterpret_cast<double4*>(frac)[i] = make_double4(v, v, v, v);  // plain memset-like
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// TMA bulk copies of `chunk` bytes each, `per_cta` bytes per CTA
__global__ void k_bulk(const uint8_t* src, int per_cta, int chunk, int issuers) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* s = src + (size_t)blockIdx.x * per_cta;
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"(per_cta)
                 : "memory");
  __syncthreads();
  if ((int)threadIdx.x < issuers)
    for (int off = threadIdx.x * chunk; off < per_cta; off += issuers * chunk)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sm + off)),
          "l"(s + off), "r"(min(chunk, per_cta - off)), "r"(smem_u32(&bar))
          : "memory");
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}\n" ::"r"(
          smem_u32(&bar))
      : "memory");
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / 20;
}

int main() {
  double *frac, *cost, *acc;
  uint32_t* nc;
  cudaMalloc(&frac, 32ll * C);
  cudaMalloc(&cost, 8ll * C);
  cudaMalloc(&acc, 8ll * C);
  cudaMalloc(&nc, 4ll * C);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"frac 2x16B + cost + acc + nc", "frac 1x32B + cost + acc + nc",
                         "frac only 2x16B", "frac only 1x32B", "frac only double4"};
  for (int blocksx = 2; blocksx <= 8; blocksx *= 2) {
    printf("store patterns, %d configs (52 B / 32 B each), grid %d x 512\n", C, sms * blocksx);
    printf("  %-32s %7.2f us\n", names[0], timeit([&] { k_store<0><<<sms * blocksx, 512>>>(frac, cost, acc, nc); }));
    printf("  %-32s %7.2f us\n", names[1], timeit([&] { k_store<1><<<sms * blocksx, 512>>>(frac, cost, acc, nc); }));
    printf("  %-32s %7.2f us\n", names[2], timeit([&] { k_store<2><<<sms * blocksx, 512>>>(frac, cost, acc, nc); }));
    printf("  %-32s %7.2f us\n", names[3], timeit([&] { k_store<3><<<sms * blocksx, 512>>>(frac, cost, acc, nc); }));
    printf("  %-32s %7.2f us\n", names[4], timeit([&] { k_store<4><<<sms * blocksx, 512>>>(frac, cost, acc, nc); }));
  }
  // TMA: 101 CTAs x 163 KB (the plane kernel's load), various chunk sizes
  uint8_t* src;
  const int per_cta = 163 * 1024 / 16 * 16;
  cudaMalloc(&src, (size_t)per_cta * 148);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, per_cta);
  const int chunks[] = {1616, 4096, 16384, 32768, per_cta};
  const int issuers[] = {1, 32};
  for (int is : issuers)
    for (int ch : chunks) {
      int c16 = ch / 16 * 16;
      float t = timeit([&] { k_bulk<<<101, 128, per_cta>>>(src, per_cta, c16, is); });
      printf("bulk 101 CTAs x %d B, chunk %6d B, %2d issuers: %7.2f us (%.0f GB/s)\n", per_cta, c16, is,
             t, 101.0 * per_cta / t / 1e3);
    }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
