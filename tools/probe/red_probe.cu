// Throughput of scattered L2 vector reductions (red.global.add.v2.f32) into a
// 1.3M-entry float2 array: the cost of the column-side scatter a symmetric
// (upper-triangle) SpMV layout would need.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_red(float2* __restrict__ out, int n, int64_t total, uint32_t seed) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < total; i += stride) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    const int j = (int)(h % (uint32_t)n);
    atomicAdd(out + j, make_float2(1.0f, 0.5f));
  }
}

int main() {
  const int n = 1300000;
  const int64_t total = 94000000;  // ~ upper-triangle entries at C3
  float2* out;
  cudaMalloc(&out, sizeof(float2) * n);
  cudaMemset(out, 0, sizeof(float2) * n);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int blocks : {148 * 8, 148 * 16, 148 * 32}) {
    k_red<<<blocks, 256>>>(out, n, total, 1);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_red<<<blocks, 256>>>(out, n, total, r + 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("blocks %d: %.1f us per 94M scattered red.v2.f32 (%.2f G/s)\n", blocks, ms / 5 * 1e3,
           total / (ms / 5 * 1e-3) / 1e9);
  }
  return 0;
}
