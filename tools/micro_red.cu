// micro_red.cu — L2 reduction throughput on B200 for the histogram design.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_red tools/micro_red.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int N = 1000000;

__global__ void gen(uint32_t* idx, uint32_t* idx2, uint32_t ncell, uint32_t ncell2) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)r * 2654435761u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    idx[r] = h % ncell;
    idx2[r] = (h / 7u) % ncell2;
  }
}

__global__ void init_rec(double* cert, uint32_t* corr) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)r * 2654435761u;
    for (int j = 0; j < 4; ++j) {
      h ^= h >> 13;
      h *= 2246822519u;
      cert[4ll * r + j] = (h >> 8) * (1.0 / 16777216.0);
    }
    corr[r] = h & 0x01010101u;
  }
}

template <int MODE>
__global__ void __launch_bounds__(1024) k(const uint32_t* idx, const uint32_t* idx2,
                                         unsigned long long* T64, unsigned long long* S64,
                                         uint32_t* T32, float* F4, unsigned long long* sink) {
  __shared__ uint32_t sm[12288];
  if (MODE == 6) {
    for (int i = threadIdx.x; i < 12288; i += blockDim.x) sm[i] = 0;
    __syncthreads();
  }
  unsigned long long acc = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    const uint32_t c = __ldg(idx + r);
    if (MODE == 0) acc += c;  // loads only
    if (MODE == 1) atomicAdd(T64 + c, 1ull | (1ull << 21));
    if (MODE == 2) {
      atomicAdd(T64 + c, 1ull | (1ull << 21));
      atomicAdd(S64 + __ldg(idx2 + r), 1ull);
    }
    if (MODE == 3) atomicAdd(T32 + c, 1u);
    if (MODE == 4)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(F4 + 4ull * c), "f"(1.f),
                   "f"(1.f), "f"(0.f), "f"(1.f)
                   : "memory");
    if (MODE == 5) atomicAdd(S64 + __ldg(idx2 + r), 1ull);
    if (MODE == 6) {
      atomicAdd(T64 + c, 1ull | (1ull << 21));
      atomicAdd(sm + (__ldg(idx2 + r) % 12288u), 1u);
    }
    if (MODE == 7) atomicAdd(T32 + (c >> 1) * 2 + (c & 1), 1u), atomicAdd(T32 + 2 * 1048576 + (c % 4096), 1u);
    if (MODE == 8) acc += atomicAdd(T64 + c, 1ull | (1ull << 16));  // ATOMG with the old value used
  }
  if ((MODE == 0 || MODE == 8) && acc == 12345) sink[0] = acc;
  if (MODE == 6) {
    __syncthreads();
    for (int i = threadIdx.x; i < 12288; i += blockDim.x)
      if (sm[i]) atomicAdd(T32 + i, sm[i]);
  }
}

// record-stream variants: 1M records of 32 B certainty + 4 B correct
template <int MODE>
__global__ void __launch_bounds__(1024) k_rec(const double* cert, const uint32_t* corr, float* F4,
                                              unsigned long long* sink) {
  __shared__ uint32_t s_c0[256];
  if (MODE == 2) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_c0[i] = 0;
    __syncthreads();
  }
  double acc = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    const double2 p = __ldg(reinterpret_cast<const double2*>(cert + 4ll * r));
    const double x2 = __ldg(cert + 4ll * r + 2);
    const uint32_t k = __ldg(corr + r);
    if (MODE == 0) {
      acc += p.x + p.y + x2 + k;
      continue;
    }
    const uint32_t h = (uint32_t)(p.x * 101.0) * 10201u + (uint32_t)(p.y * 101.0) * 101u +
                       (uint32_t)(x2 * 101.0);
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(F4 + 4ull * (h % 1030301u)),
                 "f"(1.f), "f"((float)(k & 1)), "f"((float)((k >> 8) & 1)), "f"((float)((k >> 16) & 1))
                 : "memory");
    if (MODE == 2 && (k >> 24)) atomicAdd(s_c0 + (h & 255u), 1u);
  }
  if (MODE == 0 && acc == 12345.0) sink[0] = 1;
  if (MODE == 2) {
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) atomicAdd((uint32_t*)sink + i, s_c0[i]);
  }
}

template <int MODE>
float run(int blocks, const uint32_t* idx, const uint32_t* idx2, unsigned long long* T64,
          unsigned long long* S64, uint32_t* T32, float* F4, unsigned long long* sink) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<MODE><<<blocks, 1024>>>(idx, idx2, T64, S64, T32, F4, sink);
  cudaEventRecord(a);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) k<MODE><<<blocks, 1024>>>(idx, idx2, T64, S64, T32, F4, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  uint32_t *idx, *idx2, *T32;
  unsigned long long *T64, *S64, *sink;
  float* F4;
  const uint32_t ncell = 101 * 101 * 101, ncell2 = 101 * 101;
  cudaMalloc(&idx, N * 4);
  cudaMalloc(&idx2, N * 4);
  cudaMalloc(&T64, 8ull * ncell);
  cudaMalloc(&S64, 8ull * ncell2);
  cudaMalloc(&T32, 4ull * 3 * 1048576);
  cudaMalloc(&F4, 16ull * ncell);
  cudaMalloc(&sink, 8);
  gen<<<592, 256>>>(idx, idx2, ncell, ncell2);
  cudaDeviceSynchronize();
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mult = 1; mult <= 2; ++mult) {
    const int blocks = sms * mult;
    printf("blocks=%d (x1024 threads), N=%d records\n", blocks, N);
    printf("  loads only (4 MB idx)            %7.2f us\n", run<0>(blocks, idx, idx2, T64, S64, T32, F4, sink));
    printf("  1 RED.64 / rec, 1M-cell table    %7.2f us\n", run<1>(blocks, idx, idx2, T64, S64, T32, F4, sink));
    printf("  2 RED.64 / rec (+10K-cell table) %7.2f us\n", run<2>(blocks, idx, idx2, T64, S64, T32, F4, sink));
    printf("  1 RED.32 / rec, 1M-cell table    %7.2f us\n", run<3>(blocks, idx, idx2, T64, S64, T32, F4, sink));
    printf("  1 RED.v4.f32 / rec               %7.2f us\n", run<4>(blocks, idx, idx2, T64, S64, T32, F4, sink));
    printf("  1 RED.64 / rec, 10K-cell table   %7.2f us\n", run<5>(blocks, idx, idx2, T64, S64, T32, F4, sink));
    printf("  RED.64 + smem ATOMS / rec        %7.2f us\n", run<6>(blocks, idx, idx2, T64, S64, T32, F4, sink));
    printf("  2 RED.32 / rec (1M + 4K cells)   %7.2f us\n", run<7>(blocks, idx, idx2, T64, S64, T32, F4, sink));
    printf("  1 ATOMG.64 / rec (old value used) %7.2f us\n", run<8>(blocks, idx, idx2, T64, S64, T32, F4, sink));
  }
  {
    double* cert;
    uint32_t* corr;
    cudaMalloc(&cert, 32ll * N);
    cudaMalloc(&corr, 4ll * N);
    init_rec<<<592, 256>>>(cert, corr);
    unsigned long long* sk;
    cudaMalloc(&sk, 4096);
    float* big;
    cudaMalloc(&big, 256ll << 20);  // flush buffer
    auto t = [&](auto f) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float tot = 0;
      for (int i = 0; i < 23; ++i) {
        cudaMemsetAsync(big, 0, 256ll << 20);
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (i >= 3) tot += ms;
      }
      return tot * 1000.f / 20;
    };
    printf("record stream, 1M x 36 B, 148 x 1024 threads, L2 flushed:\n");
    printf("  loads only                       %7.2f us\n", t([&] { k_rec<0><<<sms, 1024>>>(cert, corr, F4, sk); }));
    printf("  loads + 1 RED.v4 / rec           %7.2f us\n", t([&] { k_rec<1><<<sms, 1024>>>(cert, corr, F4, sk); }));
    printf("  loads + RED.v4 + smem c0 ATOMS   %7.2f us\n", t([&] { k_rec<2><<<sms, 1024>>>(cert, corr, F4, sk); }));
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
