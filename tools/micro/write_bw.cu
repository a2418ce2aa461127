// Pure-write vs copy HBM bandwidth with 16-byte vector stores (grid-stride, 148 x k CTAs):
// the roofline of the write-bound kernels (C4 bank correlation: 86 GB of corr per step).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/write_bw tools/micro/write_bw.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_write(float4* __restrict__ p, size_t n, int streaming) {
  const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    if (streaming) __stcs(p + i, v); else p[i] = v;
  }
}
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  const size_t bytes = 8ull << 30, n = bytes / 16;
  float4 *a, *b;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid_mul : {4, 8, 16}) {
    const int grid = 148 * grid_mul;
    for (int s = 0; s < 2; ++s) {
      for (int w = 0; w < 2; ++w) k_write<<<grid, 512>>>(a, n, s);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k_write<<<grid, 512>>>(a, n, s);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("write%s grid %d: %.0f GB/s\n", s ? " (st.global.cs)" : "", grid, 5.0 * bytes / ms / 1e6);
    }
    for (int w = 0; w < 2; ++w) k_copy<<<grid, 512>>>(a, b, n / 2);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_copy<<<grid, 512>>>(a, b, n / 2);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy grid %d: %.0f GB/s (read + write)\n", grid, 5.0 * bytes / ms / 1e6);
  }
  return 0;
}
