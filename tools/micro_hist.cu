// micro_hist.cu — which part of the grid histogram costs what (B200).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_hist micro_hist.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int N = 1000000, M = 4, G = 100;

__device__ __forceinline__ int upper_count(const double* g, int n, double x) {
  int base = 0, len = n;
  while (len > 1) {
    const int half = len >> 1;
    base = (g[base + half - 1] <= x) ? base + half : base;
    len -= half;
  }
  return base + (g[base] <= x ? 1 : 0);
}

constexpr int NB = 2048;
__device__ __forceinline__ int lut_bucket(double x, double lo, double hi, double scale) {
  if (!(x >= lo)) return 0;
  if (x >= hi) return NB - 1;
  const int q = (int)((x - lo) * scale);
  return q > NB - 1 ? NB - 1 : q;
}
__device__ uint32_t g_lut[3 * NB];
__global__ void build_lut(const double* grids) {
  __shared__ uint32_t cnt[NB];
  for (int j = 0; j < 3; ++j) {
    for (int i = threadIdx.x; i < NB; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const double* g = grids + j * G;
    const double lo = g[0], hi = g[G - 1], sc = NB / (hi - lo);
    for (int i = threadIdx.x; i < G; i += blockDim.x) atomicAdd(&cnt[lut_bucket(g[i], lo, hi, sc)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t run = 0;
      for (int q = 0; q < NB; ++q) { g_lut[j * NB + q] = run | ((run + cnt[q]) << 16); run += cnt[q]; }
    }
    __syncthreads();
  }
}

template <int V>
__global__ void __launch_bounds__(512) k_hist(const double* cert, const uint32_t* corr, const double* grids,
                                              float* F, unsigned long long* H, unsigned long long* sink) {
  __shared__ double sg[3 * G];
  __shared__ uint32_t sl[3 * NB];
  for (int i = threadIdx.x; i < 3 * G; i += blockDim.x) sg[i] = grids[i];
  if (V >= 7) for (int i = threadIdx.x; i < 3 * NB; i += blockDim.x) sl[i] = g_lut[i];
  __syncthreads();
  double lo[3], hi[3], sc[3];
  for (int j = 0; j < 3; ++j) { lo[j] = sg[j * G]; hi[j] = sg[j * G + G - 1]; sc[j] = NB / (hi[j] - lo[j]); }
  unsigned long long acc = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    uint32_t cell;
    uint32_t w = 0;
    if (V == 5) {
      cell = (uint32_t)((r * 2654435761u) % (101u * 101u * 101u));
    } else {
      const double2 a = reinterpret_cast<const double2*>(cert + r * M)[0];
      const double2 b = reinterpret_cast<const double2*>(cert + r * M)[1];
      w = corr[r];
      if (V == 0) {
        acc += __double_as_longlong(a.x + a.y + b.x + b.y) + w;
        continue;
      }
      int b0, b1, b2;
      if (V >= 7) {
        const double xs[3] = {a.x, a.y, b.x};
        int bb[3];
        for (int j = 0; j < 3; ++j) {
          const uint32_t e = sl[j * NB + lut_bucket(xs[j], lo[j], hi[j], sc[j])];
          const int l = e & 0xffff, u = e >> 16;
          bb[j] = l + (u > l ? upper_count(sg + j * G + l, u - l, xs[j]) : 0);
        }
        b0 = bb[0]; b1 = bb[1]; b2 = bb[2];
      } else {
        b0 = upper_count(sg, G, a.x); b1 = upper_count(sg + G, G, a.y); b2 = upper_count(sg + 2 * G, G, b.x);
      }
      cell = (b0 * 101 + b1) * 101 + b2;
    }
    if (V == 1 || V == 7) { acc += cell; continue; }
    if (V == 2 || V == 5) {
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(F + cell * 4), "f"(1.f),
                   "f"((float)(w & 1)), "f"((float)((w >> 8) & 1)), "f"((float)((w >> 16) & 1)) : "memory");
    }
    if (V == 3 || V == 8) atomicAdd(H + cell, 1ull | ((unsigned long long)(w & 1) << 16));
    if (V == 4) atomicAdd(F + cell, 1.f);
    if (V == 6) asm volatile("red.global.add.u64 [%0], %1;" ::"l"(H + cell), "l"(1ull) : "memory");
  }
  if (acc == 0x12345) *sink = acc;
}

__global__ void init(double* cert, uint32_t* corr, double* grids) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N * M; i += gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ 0x9e3779b9u;
    h ^= h >> 15; h *= 0x85ebca6bu; h ^= h >> 13;
    cert[i] = (h & 0xffffff) / 16777216.0;
    if (i < N) corr[i] = h & 0x01010101u;
  }
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < 3 * G; i += gridDim.x * blockDim.x)
    grids[i] = (i % G) / (double)G;
}

template <int V>
float run(const double* c, const uint32_t* k, const double* g, float* F, unsigned long long* H,
          unsigned long long* s, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k_hist<V><<<blocks, 512>>>(c, k, g, F, H, s);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) k_hist<V><<<blocks, 512>>>(c, k, g, F, H, s);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 20 * 1000;
}

int main() {
  double *cert, *grids;
  uint32_t* corr;
  float* F;
  unsigned long long *H, *sink;
  cudaMalloc(&cert, N * M * 8);
  cudaMalloc(&corr, N * 4);
  cudaMalloc(&grids, 3 * G * 8);
  cudaMalloc(&F, 101 * 101 * 101 * 16);
  cudaMalloc(&H, 101 * 101 * 101 * 8);
  cudaMalloc(&sink, 8);
  init<<<592, 256>>>(cert, corr, grids);
  build_lut<<<1, 256>>>(grids);
  cudaDeviceSynchronize();
  const char* names[] = {"load only", "load+bins", "load+bins+red.v4.f32", "load+bins+atom.u64",
                         "load+bins+atom.f32", "hashed cells, red.v4.f32 (no loads)", "load+bins+red.u64", "load+LUT bins", "load+LUT bins+atom.u64"};
  for (int blocks : {148, 296, 592}) {
    printf("blocks=%d\n", blocks);
    printf("  %-40s %8.2f us\n", names[0], run<0>(cert, corr, grids, F, H, sink, blocks));
    printf("  %-40s %8.2f us\n", names[1], run<1>(cert, corr, grids, F, H, sink, blocks));
    printf("  %-40s %8.2f us\n", names[2], run<2>(cert, corr, grids, F, H, sink, blocks));
    printf("  %-40s %8.2f us\n", names[3], run<3>(cert, corr, grids, F, H, sink, blocks));
    printf("  %-40s %8.2f us\n", names[4], run<4>(cert, corr, grids, F, H, sink, blocks));
    printf("  %-40s %8.2f us\n", names[5], run<5>(cert, corr, grids, F, H, sink, blocks));
    printf("  %-40s %8.2f us\n", names[6], run<6>(cert, corr, grids, F, H, sink, blocks));
    printf("  %-40s %8.2f us\n", names[7], run<7>(cert, corr, grids, F, H, sink, blocks));
    printf("  %-40s %8.2f us\n", names[8], run<8>(cert, corr, grids, F, H, sink, blocks));
  }
  return 0;
}
