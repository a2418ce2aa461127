// Microbenchmark: FP32 FMA throughput on B200 for FFMA (3-register), FFMA with an immediate,
// and packed FFMA2 (fma.rn.f32x2).  8 independent chains per thread, many warps.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ffma(float* out, float a, float b, int iters) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b, int iters) {
  unsigned long long x[8];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&av), B = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x * 0.001f + i, i); x[i] = *reinterpret_cast<unsigned long long*>(&v); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
  }
  float s = 0; for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&x[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// 32-bit integer multiply-add (IMAD, wrap-around) throughput, 8 independent chains
__global__ void k_imad(unsigned* out, unsigned a, unsigned b, int iters) {
  unsigned x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7u + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = x[i] * a + b;
  }
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// FP64 DFMA throughput, and IMAD + DFMA interleaved (separate pipes?)
__global__ void k_dfma(double* out, double a, double b, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mix(double* out, double a, double b, unsigned ia, unsigned ib, int iters) {
  double x[4]; unsigned y[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = threadIdx.x * 0.001 + i;
#pragma unroll
  for (int i = 0; i < 8; ++i) y[i] = threadIdx.x * 7u + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = fma(x[i], a, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) y[i] = y[i] * ia + ib;
  }
  double s = 0; for (int i = 0; i < 4; ++i) s += x[i];
  unsigned t = 0; for (int i = 0; i < 8; ++i) t += y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + t;
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
  int iters = 20000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_ffma<<<148 * 8, 256>>>(d, 1.0001f, 0.5f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * 148.0 * 8 * 256;
    printf("FFMA  : %.2f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
    cudaEventRecord(e0); k_ffma2<<<148 * 8, 256>>>(d, 1.0001f, 0.5f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 4.0 * 8 * iters * 148.0 * 8 * 256;
    printf("FFMA2 : %.2f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
    cudaEventRecord(e0); k_imad<<<148 * 8, 256>>>(reinterpret_cast<unsigned*>(d), 1664525u, 1013904223u, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 1.0 * 8 * iters * 148.0 * 8 * 256;
    printf("IMAD  : %.2f ms  %.1f T IMAD/s  (%.1f per clk per SM at 1965 MHz)\n", ms, ops / ms / 1e9,
           ops / (ms * 1e-3) / 148 / 1.965e9);
    double* dd; cudaMalloc(&dd, 148 * 8 * 256 * 8);
    cudaEventRecord(e0); k_dfma<<<148 * 8, 256>>>(dd, 1.0001, 0.5, iters / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double dops = 1.0 * 8 * (iters / 4) * 148.0 * 8 * 256;
    printf("DFMA  : %.2f ms  %.1f T DFMA/s  (%.1f per clk per SM)\n", ms, dops / ms / 1e9, dops / (ms * 1e-3) / 148 / 1.965e9);
    cudaEventRecord(e0); k_mix<<<148 * 8, 256>>>(dd, 1.0001, 0.5, 1664525u, 1013904223u, iters / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double mops = 1.0 * 12 * (iters / 4) * 148.0 * 8 * 256;
    printf("MIX 4 DFMA + 8 IMAD: %.2f ms  %.1f T op/s  (%.1f mul-adds per clk per SM)\n", ms, mops / ms / 1e9,
           mops / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
