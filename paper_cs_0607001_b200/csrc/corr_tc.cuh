// corr_tc.cuh -- template-bank correlation on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in TMEM), sm_100a.
//
// For a bank of templates the per-scale correlation (a5-a6 of SURVEY.md section 8)
// is a dense contraction: for term i (band W_{i+1} at stride g = 2^{i+1}, or
// U_J at g = 2^J)
//     D[t][tau] = sum_k conj(b_t[k]) W[tau + g k]
// for every template t and every lag tau.  With the lags as the N dimension and
// (template, re/im) as the M dimension, the data operand B[k][tau] = W[tau + g k]
// is a dilated Hankel matrix.  In the canonical no-swizzle MN-major operand
// layout (8 lags x 8 taps core matrices, tap rows 16 B apart) such a matrix is
// exactly a buffer Z of 16-byte rows Z[j] = W[base + ge j .. base + ge j + 7]
// (ge = g for g <= 8; for g > 8 the taps are zero-stuffed to stride 8): the
// core matrix of lags 8n.., taps 8k.. starts at row 8n/ge + 8k, so the operand
// descriptor's N-direction stride is 128/ge bytes and its K-direction stride
// 128 bytes.  Z costs 16/ge bytes per band value per (plane, split) and is built
// in shared memory once per term; no Hankel matrix is ever materialised.
//
// Complex arithmetic: M rows are (t, re) and (t, im); K runs over the re plane
// taps then the im plane taps; conj(b) w = (br wr + bi wi) + i (br wi - bi wr).
// Precision: fp32 operands are split x = hi + lo into two bf16 (8 + 8 mantissa
// bits); three bf16 MMAs (hi.hi + hi.lo + lo.hi) accumulate in fp32 in TMEM
// (4e-6 of peak, inside the 1e-4 tolerance; one TF32 pass is not).
//
// Eq. (4): the terms of a lag tile are taken coarsest first and
// accumulate into the same TMEM accumulator; after term i it holds corr_i, which
// the epilogue stores (and reduces to per-tile peak partials) before term i-1's
// MMAs may accumulate on it.  Kernel structure: see k_correlate_tc below.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace sidwt {

constexpr int kTcTilePair = 512;      // lags of a tile pair (two 256-lag accumulators)
constexpr int kTcM = 128;             // MMA M: 64 templates x (re, im)
constexpr int kTcTemplates = 64;
constexpr int kTcMaxStages = 16;      // template-operand ring depth limit
constexpr int kTcStageBytes = 16384;  // ring stage: two K steps x (hi, lo) x 4 KB

struct TcTerm {
  int band, g, ge, f, kmin, ntap;     // f = g / ge (zero-stuffing factor)
  int toff;                           // offset of the term's taps in the template table
  int kp;                             // padded taps per plane (multiple of 16)
  int ksteps;                         // 2 * kp / 16
  int kofs;                           // first K step of this term in the image
  int nz;                             // Z rows
};

struct TcParams {
  CUtensorMap tmap;                   // corr as a 4-D tensor [rows][n_t][J+1][N] of 8-byte elements
  int N, J, ext, stride, ML, n_t, n_mt, ntiles, total_ksteps, nz_max;   // ntiles: 256-lag tiles per row
  int want_corr, want_peaks;
  long long rows;
  int stages;                         // ring depth
  int a_shared;                       // 1: every template K step feeds both units of a tile pair
  int stg_len;                        // band staging floats per plane
  long long npairs;                   // rows * n_mt * ntiles / 2
  int prof;                           // debug: CTA 0 prints per-role wait cycles (SIDWT_TC_PROF=1)
  TcTerm term[17];                    // indexed by processing step (0 = coarsest, A_J)
};

// ---------------------------------------------------------------------------
// PTX wrappers (tcgen05 / TMEM)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
               :: "r"(smem_u32(slot)), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(taddr), "r"(ncols) : "memory");
}

// D[tmem] (+)= A[smem] . B[smem], kind::f16 (bf16 inputs, fp32 accumulate)
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
               :: "r"(smem_u32(bar)) : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor, no swizzle (SM100 version field = 1).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Instruction descriptor: D fp32, A/B bf16, A K-major, B MN-major, M = 128, N = 256.
constexpr uint32_t kTcIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
                              ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat16 ha = __float2bfloat16_rn(a), hb = __float2bfloat16_rn(b);
  return (uint32_t)__bfloat16_as_ushort(ha) | ((uint32_t)__bfloat16_as_ushort(hb) << 16);
}
// (a, b) -> packed bf16x2 hi = rn(a, b), lo = rn(a - hi_a, b - hi_b); low half = a
__device__ __forceinline__ void split_bf16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(a - hf.x, b - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void split_bf16(float v, float& hi, float& lo) {
  hi = __bfloat162float(__float2bfloat16_rn(v));
  lo = v - hi;
}

// ---------------------------------------------------------------------------
// Template operand images: img[mt][kstep][split][4096 B], K-major no-swizzle core
// matrices: element (m, kk) at (m/8)*256 + (kk/8)*128 + (m%8)*16 + (kk%8)*2.
// One thread per (mt, kstep, split, m).
// Row order (TMEM lane of the accumulator): m = 32 q + 16 k + 8 c + b holds component c
// (0 re, 1 im) of template tc_row_template(q, k, b) = 16 q + 8 k + (b >> 1) + 4 (b & 1), so a
// 16x256b TMEM load gives each epilogue thread (re, im) of one template for two adjacent
// lags, and the template rows of a quarter-warp differ in bit 2 (conflict-free swizzled
// staging stores).
// ---------------------------------------------------------------------------
#ifndef SIDWT_NO_KERNELS
__global__ void k_tc_images(const float2* __restrict__ taps, int taps_per_t, TcParams p, unsigned char* __restrict__ img) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)p.n_mt * p.total_ksteps * 2 * kTcM;
  if (gid >= total) return;
  const int m = (int)(gid % kTcM);
  const int split = (int)((gid / kTcM) % 2);
  const int q = (int)((gid / (2 * kTcM)) % p.total_ksteps);
  const int mt = (int)(gid / ((long long)2 * kTcM * p.total_ksteps));
  int step = 0;
  while (step < p.J && q >= p.term[step + 1].kofs) ++step;
  const TcTerm tm = p.term[step];
  const int kk = q - tm.kofs;
  const int kb_per_plane = tm.kp / 16;
  const int plane = kk / kb_per_plane;
  const int k0 = 16 * (kk % kb_per_plane);
  const int b = m & 7, c = (m >> 3) & 1, kq = m >> 4;             // kq = 2 q + k
  const int t = mt * kTcTemplates + 8 * kq + (b >> 1) + 4 * (b & 1);
  unsigned char* blk = img + ((size_t)(mt * p.total_ksteps + q) * 2 + split) * 4096;
  for (int e = 0; e < 16; ++e) {
    const int kpp = k0 + e;
    float v = 0.f;
    if (t < p.n_t && (kpp % tm.f) == 0 && kpp / tm.f < tm.ntap) {
      const float2 b = taps[(size_t)t * taps_per_t + tm.toff + kpp / tm.f];
      v = (c == 0) ? (plane == 0 ? b.x : b.y) : (plane == 0 ? -b.y : b.x);
    }
    float hi, lo;
    split_bf16(v, hi, lo);
    const __nv_bfloat16 out = __float2bfloat16_rn(split == 0 ? hi : lo);
    const int off = (m >> 3) * 256 + (e >> 3) * 128 + (m & 7) * 16 + (e & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(blk + off) = out;
  }
}

#endif  // SIDWT_NO_KERNELS

// ---------------------------------------------------------------------------
// The bank correlation kernel: persistent, warp-specialised, one CTA per SM.
//
// Work unit = (256-lag tile, term).  Tiles come in pairs (adjacent lags of one
// row and template tile); the units of a pair alternate between the two TMEM
// accumulators (acc 0: first tile, acc 1: second), term by term, coarsest first:
//   (tile0, A_J) (tile1, A_J) (tile0, D_J) (tile1, D_J) ... (tile0, D_1) (tile1, D_1)
// so the epilogue of one unit overlaps the MMAs of the next, and (a_shared) each
// template K step in the ring feeds both units of a pair.
//   warp 0     : bulk-copy producer of the template operand ring
//   warp 1     : MMA issuer (one thread)
//   warps 2-5  : Z builders: band segment -> smem staging (bulk copy), split into
//                bf16 hi/lo 16-byte rows (double-buffered Z)
//   warps 6-13 : epilogue, two warps per TMEM lane group (4 x 32-lag chunks each):
//                tcgen05.ld (next chunk prefetched), complex interleave through a
//                per-warp shared-memory transpose, one 256-byte template row per
//                store instruction, fused peak partials (|.|^2 max per chunk)
// ---------------------------------------------------------------------------
constexpr int kTcNZB = 2;                 // Z buffers
constexpr int kTcBuildWarps = 5;
constexpr int kTcEpiWarps = 8;
constexpr int kTcEpiBytes = 8192;         // per epilogue warp: 2 buffers x two 16 x 16 x 8 B TMA boxes (128B swizzle)
constexpr int kTcFirstBuild = 3;         // warp 2: band stager
constexpr int kTcFirstEpi = kTcFirstBuild + kTcBuildWarps;
constexpr int kTcWarps = kTcFirstEpi + kTcEpiWarps;
constexpr int kTcThreads = 32 * kTcWarps;
constexpr int kTcRegsProd = 96, kTcRegsEpi = 160;   // registers per thread after setmaxnreg (8 warps each: 8 x 96 + 8 x 160 = 2048)
static_assert(kTcFirstEpi == 8 && kTcWarps == 16, "setmaxnreg: the epilogue is warpgroups 2-3");

struct TcSmem {
  int ring, zbuf, stg, epi, total;
};
__host__ __device__ inline TcSmem tc_smem_layout(const TcParams& p) {
  TcSmem m;
  m.ring = 1024;
  m.zbuf = m.ring + p.stages * kTcStageBytes;
  m.stg = m.zbuf + kTcNZB * 4 * p.nz_max * 16;
  m.epi = (m.stg + 2 * 2 * p.stg_len * 4 + 1023) & ~1023;      // 1024-aligned (128B swizzle atoms)
  m.total = m.epi + kTcEpiWarps * kTcEpiBytes;
  return m;
}

struct TcUnit { int row, mt, tile, step, half; };

__device__ __forceinline__ TcUnit tc_unit(const TcParams& p, int pair, int k) {
  // k = step * 2 + half within the pair; 32-bit arithmetic (npairs < 2^30, host-checked)
  TcUnit u;
  u.step = k >> 1;
  u.half = k & 1;
  const int tp = p.ntiles >> 1;                                 // tile pairs per (row, template tile)
  const int bt = pair / tp;
  u.tile = 2 * (pair - bt * tp) + u.half;
  u.row = bt / p.n_mt;
  u.mt = bt - u.row * p.n_mt;
  return u;
}

// mbarrier wait that suspends the warp (time hint) instead of spinning, so waiting
// roles do not take issue slots from the epilogue warps sharing their SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITS_%=;\n}\n" :: "r"(smem_u32(bar)), "r"(parity), "r"(1000000u) : "memory");
}

// Waits of the role pipeline; with -DSIDWT_TC_PROFILE they are timed (clock64) and
// CTA 0 prints per-role totals when SIDWT_TC_PROF is set.
#ifdef SIDWT_TC_PROFILE
#define TC_TWAIT(bar, par, acc)                                   \
  do {                                                            \
    const long long _t0 = clock64();                              \
    mbar_wait(bar, par);                                          \
    acc += clock64() - _t0;                                       \
  } while (0)
#define TC_CLOCK() clock64()
#else
#define TC_TWAIT(bar, par, acc) mbar_wait(bar, par)
#define TC_CLOCK() 0LL
#endif

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(smem_u32(bar)) : "memory");
}
// per-warpgroup register budget: the kernels launch with 512 threads x 128 registers; a role's
// warpgroups release registers (dec) or take the released ones (inc)
template <int N>
__device__ __forceinline__ void set_max_regs() {
  if constexpr (N > 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" :: "n"(N));
  else if constexpr (N < 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" :: "n"(N));
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" :: "r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 16 lanes x 32 columns: thread t = a + 4 b gets, for rep r = 0..3, lanes b and b + 8 at
// columns 8 r + 2 a, 8 r + 2 a + 1 -> registers 4 r + {0: (b, 2a), 1: (b, 2a+1), 2: (b+8, 2a), 3: (b+8, 2a+1)}
__device__ __forceinline__ void tmem_ld16x256_x4(uint32_t taddr, uint32_t (&r)[32], int o) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[o + 0]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]), "=r"(r[o + 5]),
        "=r"(r[o + 6]), "=r"(r[o + 7]), "=r"(r[o + 8]), "=r"(r[o + 9]), "=r"(r[o + 10]), "=r"(r[o + 11]),
        "=r"(r[o + 12]), "=r"(r[o + 13]), "=r"(r[o + 14]), "=r"(r[o + 15])
      : "r"(taddr));
}

// wait for this thread's outstanding tcgen05.ld; the registers of `r` are tied to the
// wait so no use of them can be scheduled before it
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
                 "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
                 "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :: "memory");
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t saddr, int x0, int x1, int x2, int x3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n"
               :: "l"(map), "r"(saddr), "r"(x0), "r"(x1), "r"(x2), "r"(x3) : "memory");
}

#ifndef SIDWT_NO_KERNELS
__global__ void __launch_bounds__(kTcThreads, 1)
k_correlate_tc(const float* __restrict__ bands, const unsigned char* __restrict__ img, float2* __restrict__ corr,
               PeakF* __restrict__ partials, const __grid_constant__ TcParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const TcSmem L = tc_smem_layout(p);
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);     // [S]
  uint64_t* empty = full + S;                                   // [S]
  uint64_t* zfull = empty + S;                                  // [2]
  uint64_t* zempty = zfull + 2;                                 // [2]
  uint64_t* accfull = zempty + 2;                               // [2]
  uint64_t* accempty = accfull + 2;                             // [2]
  uint64_t* stgbar = accempty + 2;                              // [2]
  uint64_t* stgempty = stgbar + 2;                              // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(stgempty + 2);
  unsigned char* ring = smem_raw + L.ring;
  unsigned char* zbuf = smem_raw + L.zbuf;
  float* stg = reinterpret_cast<float*>(smem_raw + L.stg);
  const int zplane = p.nz_max * 16;                             // bytes per (plane, split)
  const int units_per_pair = 2 * (p.J + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&zfull[b], 32 * kTcBuildWarps);
      mbar_init(&zempty[b], 1);
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], kTcEpiWarps);
      mbar_init(&stgbar[b], 1);
      mbar_init(&stgempty[b], kTcBuildWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  // Template-operand ring schedule per (tile pair, term) with K = ksteps: the first unit
  // consumes K steps; the second reuses the last R = min(K, S) of them from the ring
  // (resident) and reloads steps 0 .. K - R - 1; the ring index advances by 2K - R.
  // First unit releases steps 0 .. K - R - 1, the second everything it consumes.
  auto ring_at = [&](int s0, uint32_t ph0, int i, int& s_, uint32_t& ph_) {
    s_ = s0 + i;
    ph_ = ph0;
    while (s_ >= S) { s_ -= S; ph_ ^= 1u; }
  };
  // register budget by role (whole warpgroups 0-1 producers, 2-3 epilogue; setmaxnreg at the head
  // of each arm so that the arm's allocation follows it)
  if (warp < kTcFirstEpi) {
  set_max_regs<kTcRegsProd>();
  if (warp == 0) {
    // ===================== template operand producer =====================
    if (lane == 0) {
      long long w_empty = 0, t_start = TC_CLOCK();
      int s = 0;
      uint32_t ph = 0;                                          // slot / phase parity of the ring head
      for (int pair = blockIdx.x; pair < (int)p.npairs; pair += gridDim.x) {
        const int mt = (pair / (p.ntiles >> 1)) % p.n_mt;
        const unsigned char* img_mt = img + (size_t)mt * p.total_ksteps * 8192;
        for (int step = 0; step <= p.J; ++step) {
          const TcTerm& tm = p.term[step];
          const int K = tm.ksteps >> 1;                          // stages (two K steps each)
          const int R = p.a_shared ? min(K, S) : 0;
          const unsigned char* src = img_mt + (size_t)tm.kofs * 8192;
          for (int i = 0; i < 2 * K - R; ++i) {
            const int kk = i < K ? i : i - K;
            TC_TWAIT(&empty[s], ph ^ 1u, w_empty);
            mbar_expect_tx(&full[s], kTcStageBytes);
            bulk_load_g2s(ring + s * kTcStageBytes, src + (size_t)kk * kTcStageBytes, kTcStageBytes, &full[s]);
            if (++s == S) { s = 0; ph ^= 1u; }
          }
        }
      }
      if (p.prof && blockIdx.x == 0)
        printf("[tc prof] producer: total %lld  wait_empty %lld\n", TC_CLOCK() - t_start, w_empty);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      long long w_z = 0, w_acc = 0, w_full = 0, t_start = TC_CLOCK();
      const uint64_t desc_ring = smem_desc(smem_u32(ring), 128, 256);
      int s = 0;                                                // ring head slot / parity
      uint32_t ph = 0;
      long long u = 0;                                          // unit counter
      for (int pair = blockIdx.x; pair < (int)p.npairs; pair += gridDim.x) {
        for (int step = 0; step <= p.J; ++step) {
          const TcTerm& tm = p.term[step];
          const int K = tm.ksteps >> 1;                          // stages (two K steps each)
          const int R = p.a_shared ? min(K, S) : 0;
          const int kbpp = tm.kp / 16;
          const uint32_t sbo_b = 128u / (uint32_t)tm.ge;
          for (int a = 0; a < 2; ++a, ++u) {
            const int zb = (int)(u & 1);
            TC_TWAIT(&zfull[zb], (uint32_t)((u >> 1) & 1), w_z);
            TC_TWAIT(&accempty[a], (uint32_t)(((u >> 1) & 1) ^ 1), w_acc);
            tc_fence_after();
            const uint64_t desc_z = smem_desc(smem_u32(zbuf) + zb * 4 * zplane, 128, sbo_b);
            const uint32_t d = tbase + a * 256;
            bool first = step == 0;
            for (int n = 0; n < K; ++n) {
              // ring offset and stage of the n-th stage of this unit
              int off, kq;
              bool wait_full, release;
              if (a == 0) { off = n; kq = n; wait_full = true; release = n < K - R; }
              else if (n < R) { off = K - R + n; kq = K - R + n; wait_full = false; release = true; }
              else { off = K + (n - R); kq = n - R; wait_full = true; release = true; }
              int ss;
              uint32_t pp;
              ring_at(s, ph, off, ss, pp);
              if (wait_full) {
                TC_TWAIT(&full[ss], pp, w_full);
                tc_fence_after();
              }
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int kk = 2 * kq + h;
                const int pl = kk >= kbpp, kb = kk - pl * kbpp;
                const uint64_t dah = desc_ring + (uint64_t)((ss * kTcStageBytes + h * 8192) >> 4);
                const uint64_t dal = dah + (4096 >> 4);
                const uint64_t dbh = desc_z + (uint64_t)(((pl * 2 + 0) * zplane + kb * 256) >> 4);
                const uint64_t dbl = desc_z + (uint64_t)(((pl * 2 + 1) * zplane + kb * 256) >> 4);
                if (!(p.prof & 4)) {
                  umma_bf16(d, dah, dbh, kTcIdesc, first ? 0u : 1u);
                  umma_bf16(d, dah, dbl, kTcIdesc, 1u);
                  umma_bf16(d, dal, dbh, kTcIdesc, 1u);
                }
                first = false;
              }
              if (release) umma_commit(&empty[ss]);
            }
            umma_commit(&accfull[a]);
            umma_commit(&zempty[zb]);
          }
          int ns;
          uint32_t np;
          ring_at(s, ph, 2 * K - R, ns, np);
          s = ns; ph = np;
        }
      }
      if (p.prof && blockIdx.x == 0)
        printf("[tc prof] mma: total %lld  wait_z %lld  wait_acc %lld  wait_full %lld  units %lld\n",
               TC_CLOCK() - t_start, w_z, w_acc, w_full, u);
    }
    __syncwarp();
  } else if (warp == 2) {
    // ===================== band stager (one thread) =====================
    // Unit u's band segment (both planes) -> staging buffer u & 1 by two bulk copies
    // (symmetric extension: contiguous, margins present), once the builders released it.
    if (lane == 0 && p.ext != 0) {
      long long u = 0;
      for (int pair = blockIdx.x; pair < (int)p.npairs; pair += gridDim.x) {
        const TcUnit u0 = tc_unit(p, pair, 0);
        const float* brow_ = bands + (size_t)u0.row * (p.J + 1) * 2 * p.stride;
        for (int k = 0; k < units_per_pair; ++k, ++u) {
          const int sb = (int)(u & 1);
          const TcTerm& tm = p.term[k >> 1];
          const int pos0 = (u0.tile + (k & 1)) * 256 + tm.g * tm.kmin;
          const int a = pos0 + p.ML;
          const int a4 = a & ~3;
          const int need = (a - a4) + tm.ge * (tm.nz - 1) + 8;
          int len = (need + 3) & ~3;
          if (a4 + len > p.stride) len = p.stride - a4;
          const float* src = brow_ + (size_t)tm.band * 2 * p.stride + a4;
          float* dst = stg + (size_t)sb * 2 * p.stg_len;
          mbar_wait_sleep(&stgempty[sb], (uint32_t)(((u >> 1) & 1) ^ 1));
          mbar_expect_tx(&stgbar[sb], (uint32_t)(2 * len * 4));
          bulk_load_g2s(dst, src, (uint32_t)(len * 4), &stgbar[sb]);
          bulk_load_g2s(dst + p.stg_len, src + p.stride, (uint32_t)(len * 4), &stgbar[sb]);
        }
      }
    }
    __syncwarp();
  } else if (warp < kTcFirstEpi) {
    // ===================== Z builders =====================
    // Z[zb][plane][split][j] (16 bytes) = bf16 hi / lo of band[pos0 + ge j .. + 7]; four
    // threads per row (two elements each), rows of both planes spread over the builders.
    constexpr int NB = 32 * kTcBuildWarps;
    const int bt = threadIdx.x - 32 * kTcFirstBuild;
    const int e2 = bt & 3;                                      // element pair of the row
    const int rb = bt >> 2;                                     // first row of this thread
    constexpr int RS = NB / 4;                                  // row step
    const bool sym = p.ext != 0;
    long long w_stg = 0, w_ze = 0, t_start = TC_CLOCK(), b_conv = 0;
    long long u = 0;
    for (int pair = blockIdx.x; pair < (int)p.npairs; pair += gridDim.x) {
      for (int k = 0; k < units_per_pair; ++k, ++u) {
        const int zb = (int)(u & 1), sb = (int)(u & 1);
        const TcUnit un = tc_unit(p, pair, k);
        const TcTerm tm = p.term[un.step];                      // by value: fields in registers
        const int ge = tm.ge, nz = tm.nz;
        const int pos0 = un.tile * 256 + tm.g * tm.kmin;
        float* sp = stg + (size_t)sb * 2 * p.stg_len;
        int off, lim;
        if (sym) {
          const int a = pos0 + p.ML;
          const int a4 = a & ~3;
          off = a - a4;
          const int need = off + ge * (nz - 1) + 8;
          int len = (need + 3) & ~3;
          if (a4 + len > p.stride) len = p.stride - a4;
          lim = len - 1;
          TC_TWAIT(&stgbar[sb], (uint32_t)((u >> 1) & 1), w_stg);
        } else {
          // periodic: wrapped gather into the staging buffer (builders themselves)
          off = 0;
          const int need = ge * (nz - 1) + 8;
          lim = need - 1;
          const float* b0 = bands + ((size_t)un.row * (p.J + 1) + tm.band) * 2 * p.stride;
          for (int i = bt; i < need; i += NB) {
            const int idx = (pos0 + i) & (p.N - 1);
            sp[i] = __ldg(b0 + idx);
            sp[p.stg_len + i] = __ldg(b0 + p.stride + idx);
          }
          named_bar(1, NB);
        }
        TC_TWAIT(&zempty[zb], (uint32_t)(((u >> 1) & 1) ^ 1), w_ze);
        const long long _b1 = TC_CLOCK();
        unsigned char* zb_ptr = zbuf + zb * 4 * zplane;
        const int nfast = min(nz, max(0, (lim - 7 - off) / ge + 1));   // rows needing no clamp
#pragma unroll
        for (int pl = 0; pl < 2; ++pl) {
          const float* src = sp + pl * p.stg_len + off + 2 * e2;
          uint32_t* zh = reinterpret_cast<uint32_t*>(zb_ptr + (pl * 2 + 0) * zplane) + e2;
          uint32_t* zl = reinterpret_cast<uint32_t*>(zb_ptr + (pl * 2 + 1) * zplane) + e2;
          int j = rb;
          for (; j + 3 * RS < nfast; j += 4 * RS) {
            float x0[4], x1[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) { x0[q] = src[ge * (j + q * RS)]; x1[q] = src[ge * (j + q * RS) + 1]; }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t hw, lw;
              split_bf16x2(x0[q], x1[q], hw, lw);
              zh[(j + q * RS) * 4] = hw;
              zl[(j + q * RS) * 4] = lw;
            }
          }
          for (; j < nz; j += RS) {
            const int i0 = off + ge * j + 2 * e2;
            const float x0 = sp[pl * p.stg_len + min(i0, lim)];
            const float x1 = sp[pl * p.stg_len + min(i0 + 1, lim)];
            uint32_t hw, lw;
            split_bf16x2(x0, x1, hw, lw);
            zh[j * 4] = hw;
            zl[j * 4] = lw;
          }
        }
        fence_proxy_async_smem();
        mbar_arrive(&zfull[zb]);
        __syncwarp();
        if (sym && lane == 0) mbar_arrive(&stgempty[sb]);       // staging buffer free
        if (!sym) named_bar(1, NB);
        b_conv += TC_CLOCK() - _b1;
      }
    }
    if (p.prof && blockIdx.x == 0 && bt == 0)
      printf("[tc prof] builder: total %lld  wait_stg %lld  wait_zempty %lld  convert %lld\n",
             TC_CLOCK() - t_start, w_stg, w_ze, b_conv);
  }
  } else {
    set_max_regs<kTcRegsEpi>();
    // ===================== epilogue (8 warps; TMEM lane group = warp & 3) =====================
    // Per 32-lag chunk, two 16x256b TMEM loads (lane blocks k = 0, 1 of the warp's 32 lanes)
    // give thread (a, b) the complex values of templates tr[k] = 8 k + (b >> 1) + 4 (b & 1)
    // (of the warp's 16) at lags 8 rep + 2 a + {0, 1}, rep = 0..3: 16-byte (re, im, re, im)
    // pairs, stored into a per-warp staging area (two buffers alternating per 32 lags; two
    // TMA boxes lags 0-15 / 16-31 of 16 template rows x 128 B, 128B-swizzled: chunk q of row
    // r at q ^ (r & 7); conflict-free), then a 4-D TMA tensor store per box (coalesced
    // 128-byte rows; templates past n_t clipped by the tensor bounds).  Peaks from registers.
    const int ew = warp - kTcFirstEpi;
    const int lg = warp & 3;
    const int hh = ew >> 2;                                     // column half: chunks 4 hh .. 4 hh + 3
    unsigned char* epi = smem_raw + L.epi + ew * kTcEpiBytes;
    const int ta = lane & 3, tb = lane >> 2;
    const int tr0 = (tb >> 1) + 4 * (tb & 1), tr1 = 8 + tr0;     // template rows (of the warp's 16)
    long long w_acc = 0, t_start = TC_CLOCK(), w_tm = 0, w_rd = 0, t_st = 0, t_pk = 0;
    long long u = 0;
    int cb = 0;                                                 // staging buffer of the next chunk
    for (int pair = blockIdx.x; pair < (int)p.npairs; pair += gridDim.x) {
      for (int k = 0; k < units_per_pair; ++k, ++u) {
        const TcUnit un = tc_unit(p, pair, k);
        const int a = k & 1;
        const int ti = p.J - un.step;
        const int t0 = un.mt * kTcTemplates + lg * 16;
        const int tau_h = un.tile * 256 + hh * 128;
        TC_TWAIT(&accfull[a], (uint32_t)((u >> 1) & 1), w_acc);
        tc_fence_after();
        float bm2[2] = {-1.f, -1.f}, bre[2] = {0.f, 0.f}, bim[2] = {0.f, 0.f};
        int btau[2] = {0x7fffffff, 0x7fffffff};
        const uint32_t tcol = tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)(a * 256 + hh * 128);
        // TMEM loads double-buffered: chunk c + 1 is in flight while chunk c is staged and scanned
        uint32_t va[32], vb[32];
        tmem_ld16x256_x4(tcol, va, 0);
        tmem_ld16x256_x4(tcol + (16u << 16), va, 16);
#pragma unroll
        for (int c = 0; c < 4; ++c, cb ^= 1) {
          uint32_t (&v)[32] = (c & 1) ? vb : va;
          uint32_t (&vn)[32] = (c & 1) ? va : vb;
          const long long c0 = TC_CLOCK();
          tmem_wait_ld(v);
          const long long c1 = TC_CLOCK();
          w_tm += c1 - c0;
          if (c < 3) {
            tmem_ld16x256_x4(tcol + (c + 1) * 32, vn, 0);
            tmem_ld16x256_x4(tcol + (16u << 16) + (c + 1) * 32, vn, 16);
          }
          if (c == 3) {                                         // accumulator fully read: release it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[a]);
          }
          unsigned char* buf = epi + cb * 4096;
          const int tau_c = tau_h + c * 32;
          const long long c2 = TC_CLOCK();
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");   // buffer cb free
          __syncwarp();
          const long long c3 = TC_CLOCK();
          w_rd += c3 - c2;
#pragma unroll
          for (int kb = 0; kb < 2; ++kb) {
            const int r = kb ? tr1 : tr0;
#pragma unroll
            for (int rep = 0; rep < 4; ++rep) {
              const uint32_t* q = v + 16 * kb + 4 * rep;
              const int ch = ta + 4 * (rep & 1);
              *reinterpret_cast<float4*>(buf + (rep >> 1) * 2048 + r * 128 + ((ch ^ (r & 7)) << 4)) =
                  make_float4(__uint_as_float(q[0]), __uint_as_float(q[2]), __uint_as_float(q[1]), __uint_as_float(q[3]));
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          const int u_tau = __shfl_sync(0xffffffffu, tau_c, 0);
          const int u_ti = __shfl_sync(0xffffffffu, ti, 0);
          const int u_t0 = __shfl_sync(0xffffffffu, t0, 0);
          const int u_row = __shfl_sync(0xffffffffu, un.row, 0);
          const uint32_t u_sa = __shfl_sync(0xffffffffu, smem_u32(buf), 0);
          if (lane == 0) {
            if (p.want_corr) {
              tma_store_4d(&p.tmap, u_sa, u_tau, u_ti, u_t0, u_row);
              tma_store_4d(&p.tmap, u_sa + 2048, u_tau + 16, u_ti, u_t0, u_row);
            }
            bulk_commit();                                      // (possibly empty) group per chunk
          }
          const long long c4 = TC_CLOCK();
          t_st += c4 - c3;
          if (p.want_peaks) {
#pragma unroll
            for (int kb = 0; kb < 2; ++kb) {
              float m2[8];
              float mx = -1.f;
#pragma unroll
              for (int i = 0; i < 8; ++i) {                     // i = 2 rep + j: lag 8 rep + 2 ta + j
                const uint32_t* q = v + 16 * kb + 4 * (i >> 1);
                m2[i] = mag2f(__uint_as_float(q[i & 1]), __uint_as_float(q[2 + (i & 1)]));
                mx = fmaxf(mx, m2[i]);
              }
              if (mx > bm2[kb]) {
                int bi = 7;
#pragma unroll
                for (int i = 6; i >= 0; --i) bi = (m2[i] == mx) ? i : bi;
                float vr = 0.f, vi = 0.f;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const uint32_t* q = v + 16 * kb + 4 * (i >> 1);
                  vr = (i == bi) ? __uint_as_float(q[i & 1]) : vr;
                  vi = (i == bi) ? __uint_as_float(q[2 + (i & 1)]) : vi;
                }
                bm2[kb] = mx; btau[kb] = tau_c + 8 * (bi >> 1) + 2 * ta + (bi & 1); bre[kb] = vr; bim[kb] = vi;
              }
            }
          }
          t_pk += TC_CLOCK() - c4;
        }
        if (p.want_peaks) {
#pragma unroll
          for (int kb = 0; kb < 2; ++kb) {
#pragma unroll
            for (int off = 1; off <= 2; off <<= 1) {            // the 4 threads (ta) of a template
              const float om2 = __shfl_xor_sync(0xffffffffu, bm2[kb], off);
              const int otau = __shfl_xor_sync(0xffffffffu, btau[kb], off);
              const float ore = __shfl_xor_sync(0xffffffffu, bre[kb], off);
              const float oim = __shfl_xor_sync(0xffffffffu, bim[kb], off);
              if (beats(om2, otau, bm2[kb], btau[kb])) { bm2[kb] = om2; btau[kb] = otau; bre[kb] = ore; bim[kb] = oim; }
            }
            const int t = t0 + (kb ? tr1 : tr0);
            if (ta == 0 && t < p.n_t) {
              PeakF b;
              b.m2 = bm2[kb]; b.tau = btau[kb]; b.re = bre[kb]; b.im = bim[kb];
              partials[(((size_t)un.row * p.n_t + t) * (p.J + 1) + ti) * (2 * p.ntiles) + 2 * un.tile + hh] = b;
            }
          }
        }
      }
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
    if (p.prof && blockIdx.x == 0 && lane == 0)
      printf("[tc prof] epilogue warp %d: total %lld  wait_accfull %lld tmem %lld stgread %lld stage %lld peak %lld\n", warp,
             TC_CLOCK() - t_start, w_acc, w_tm, w_rd, t_st, t_pk);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

#endif  // SIDWT_NO_KERNELS

}  // namespace sidwt
