// Microbenchmark + layout check: tcgen05.mma (kind::f16, bf16 in, fp32 accumulate, A and B from
// shared memory) at M = 128 and small N, with the A operand a Hankel view of one sequence u:
// A[m][k] = u[8m + k] as a K-major no-swizzle operand whose core matrices overlap (leading byte
// offset 16 B, stride byte offset 128 B).  Prints max |D - D_ref| and cycles per MMA for N in
// {16, 32, 64, 128, 256}.   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_rate tc_rate.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

constexpr int K = 48;          // taps per MMA chain (3 k-steps of 16)
constexpr int NMAX = 256;
constexpr int ULEN = 8 * 128 + K + 8;

__global__ void k_tc(const float* __restrict__ u_g, const float* __restrict__ b_g, float* __restrict__ d_out, int N,
                     int reps, long long* cycles, int hankel) {
  __shared__ __align__(1024) __nv_bfloat16 A[128 * K];       // used when !hankel (materialised)
  __shared__ __align__(1024) __nv_bfloat16 U[ULEN];
  __shared__ __align__(1024) __nv_bfloat16 B[NMAX * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < ULEN; i += blockDim.x) U[i] = __float2bfloat16(u_g[i]);
  // A materialised in the canonical K-major no-swizzle layout: (m, k) at (m/8)*SBO + (k/8)*128 + (m%8)*16 + (k%8)*2, SBO = K/8*128
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const int off = (m / 8) * (K / 8) * 64 + (k / 8) * 64 + (m % 8) * 8 + (k % 8);
    A[off] = __float2bfloat16(u_g[8 * m + k]);
  }
  // B[k][n] K-major: (n, k) at (n/8)*(K/8)*128 + (k/8)*128 + (n%8)*16 + (k%8)*2 bytes
  for (int i = tid; i < NMAX * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const int off = (n / 8) * (K / 8) * 64 + (k / 8) * 64 + (n % 8) * 8 + (k % 8);
    B[off] = __float2bfloat16(b_g[k * NMAX + n]);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" :: "r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = tslot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (0u << 16) | ((uint32_t)(N >> 3) << 17) |
                         ((uint32_t)(128 >> 4) << 24);
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int ks = 0; ks < K / 16; ++ks) {
        const uint64_t ad = hankel ? desc(su32(U) + ks * 32, 16, 128) : desc(su32(A) + ks * 256, 128, (K / 8) * 128);
        const uint64_t bd = desc(su32(B) + ks * 256, 128, (K / 8) * 128);
        mma(tm, ad, bd, idesc, (r > 0 || ks > 0) ? 1u : 0u);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" :: "r"(su32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}\n"
                 :: "r"(su32(&bar)) : "memory");
    t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // read D: warp w holds lanes 32w..32w+31; 16 columns at a time
  const int w = tid >> 5, lane = tid & 31;
  if (w < 4 && blockIdx.x == 0) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(tm + ((uint32_t)(32 * w) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 16; ++j) d_out[(32 * w + lane) * NMAX + c0 + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" :: "r"(tm));
}

int main() {
  std::vector<float> u(ULEN), b(K * NMAX);
  srand(1);
  for (auto& x : u) x = (float)(rand() % 17 - 8);
  for (auto& x : b) x = (float)(rand() % 9 - 4);
  float *du, *db, *dd;
  long long* dc;
  cudaMalloc(&du, u.size() * 4); cudaMalloc(&db, b.size() * 4); cudaMalloc(&dd, 128 * NMAX * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(du, u.data(), u.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  std::vector<float> d(128 * NMAX);
  for (int hankel = 1; hankel >= 0; --hankel)
    for (int N : {16, 32, 64, 128, 256}) {
      // correctness (reps = 1)
      k_tc<<<1, 128>>>(du, db, dd, N, 1, dc, hankel);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          double s = 0;
          for (int k = 0; k < K; ++k) s += (double)u[8 * m + k] * b[k * NMAX + n];
          err = std::max(err, std::abs(s - d[m * NMAX + n]));
        }
      // throughput: 148 CTAs, reps x 4 MMAs each
      const int reps = 2048;
      long long cyc = 0;
      k_tc<<<148, 128>>>(du, db, dd, N, reps, dc, hankel);
      cudaDeviceSynchronize();
      cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
      const double per = (double)cyc / (reps * (K / 16));
      printf("%s N=%3d  max|err|=%g  cycles/MMA=%.2f  (floor %d)  MAC/clk/SM=%.0f\n", hankel ? "hankel A" : "plain  A", N,
             err, per, 128 * N / 256, 128.0 * N * 16 / per);
    }
  return 0;
}
