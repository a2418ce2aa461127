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
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace sidwt {

constexpr int kTcTilePair = 512;      // lags of a tile pair (two 256-lag accumulators)
constexpr int kTcM = 128;             // MMA M: 64 templates x (re, im)
constexpr int kTcTemplates = 64;
constexpr int kTcMaxStages = 32;      // template-operand ring depth limit (8 KB per stage)
constexpr int kTcThreads = 256;

struct TcTerm {
  int band, g, ge, f, kmin, ntap;     // f = g / ge (zero-stuffing factor)
  int toff;                           // offset of the term's taps in the template table
  int kp;                             // padded taps per plane (multiple of 16)
  int ksteps;                         // 2 * kp / 16
  int kofs;                           // first K step of this term in the image
  int nz;                             // Z rows
};

struct TcParams {
  int N, J, ext, stride, ML, n_t, n_mt, ntiles, total_ksteps, nz_max;   // ntiles: 256-lag tiles per row
  int want_corr, want_peaks;
  long long rows;
  int stages;                         // ring depth
  int a_shared;                       // 1: every template K step feeds both units of a tile pair
  int stg_len;                        // band staging floats per plane
  long long npairs;                   // rows * n_mt * ntiles / 2
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
__device__ __forceinline__ void split_bf16(float v, float& hi, float& lo) {
  hi = __bfloat162float(__float2bfloat16_rn(v));
  lo = v - hi;
}

// ---------------------------------------------------------------------------
// Template operand images: img[mt][kstep][split][4096 B], K-major no-swizzle core
// matrices: element (m, kk) at (m/8)*256 + (kk/8)*128 + (m%8)*16 + (kk%8)*2.
// One thread per (mt, kstep, split, m).
// ---------------------------------------------------------------------------
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
  const int t = mt * kTcTemplates + (m >> 1);
  const int c = m & 1;
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

// ---------------------------------------------------------------------------
// The bank correlation kernel: persistent, warp-specialised, one CTA per SM.
//
// Work unit = (256-lag tile, term).  Tiles come in pairs (adjacent lags of one
// row and template tile); the units of a pair alternate between the two TMEM
// accumulators (acc 0: first tile, acc 1: second), term by term, coarsest first:
//   (tile0, A_J) (tile1, A_J) (tile0, D_J) (tile1, D_J) ... (tile0, D_1) (tile1, D_1)
// so the epilogue of one unit overlaps the MMAs of the next, and (a_shared) each
// template K step in the ring feeds both units of a pair.
//   warp 0    : bulk-copy producer of the template operand ring
//   warp 1    : MMA issuer (one thread)
//   warps 2-3 : Z builders: band segment -> smem staging (bulk copy), split into
//               bf16 hi/lo 16-byte rows (double-buffered Z)
//   warps 4-7 : epilogue: TMEM -> registers (tcgen05.ld), corr_s stores through a
//               per-warp shared-memory transpose (whole 128-byte lines per store
//               instruction), fused per-tile peak partials
// ---------------------------------------------------------------------------
constexpr int kTcNZB = 2;                 // Z buffers
constexpr int kTcEpiPitch = 272;          // bytes per template row of the epilogue transpose (256 + 16)

struct TcSmem {
  int ring, zbuf, stg, epi, total;
};
__host__ __device__ inline TcSmem tc_smem_layout(const TcParams& p) {
  TcSmem m;
  m.ring = 1024;
  m.zbuf = m.ring + p.stages * 8192;
  m.stg = m.zbuf + kTcNZB * 4 * p.nz_max * 16;
  m.epi = m.stg + 2 * 2 * p.stg_len * 4;
  m.total = m.epi + 4 * 16 * kTcEpiPitch;
  return m;
}

struct TcUnit { long long row; int mt, tile, step, half; };

__device__ __forceinline__ TcUnit tc_unit(const TcParams& p, long long pair, int k) {
  // k = step * 2 + half within the pair
  TcUnit u;
  u.step = k >> 1;
  u.half = k & 1;
  const long long tg = 2 * pair + u.half;
  u.tile = (int)(tg % p.ntiles);
  const long long bt = tg / p.ntiles;
  u.mt = (int)(bt % p.n_mt);
  u.row = bt / p.n_mt;
  return u;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" :: "r"(id), "r"(n) : "memory");
}

__global__ void __launch_bounds__(kTcThreads, 1)
k_correlate_tc(const float* __restrict__ bands, const unsigned char* __restrict__ img, float2* __restrict__ corr,
               PeakF* __restrict__ partials, TcParams p) {
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
  uint32_t* tslot = reinterpret_cast<uint32_t*>(stgbar + 2);
  unsigned char* ring = smem_raw + L.ring;
  unsigned char* zbuf = smem_raw + L.zbuf;
  float* stg = reinterpret_cast<float*>(smem_raw + L.stg);
  const int zplane = p.nz_max * 16;                             // bytes per (plane, split)
  const int units_per_pair = 2 * (p.J + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&zfull[b], 64);
      mbar_init(&zempty[b], 1);
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], 4);
      mbar_init(&stgbar[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    // ===================== template operand producer =====================
    if (lane == 0) {
      long long n = 0;                                          // ring load counter
      for (long long pair = blockIdx.x; pair < p.npairs; pair += gridDim.x) {
        const int mt = (int)(((2 * pair) / p.ntiles) % p.n_mt);
        const unsigned char* img_mt = img + (size_t)mt * p.total_ksteps * 8192;
        for (int k = 0; k < units_per_pair; ++k) {
          if (p.a_shared && (k & 1)) continue;                  // second unit reuses the stages
          const TcTerm& tm = p.term[k >> 1];
          for (int kk = 0; kk < tm.ksteps; ++kk, ++n) {
            const int s = (int)(n % S);
            mbar_wait(&empty[s], (uint32_t)(((n / S) & 1) ^ 1));
            mbar_expect_tx(&full[s], 8192);
            bulk_load_g2s(ring + s * 8192, img_mt + (size_t)(tm.kofs + kk) * 8192, 8192, &full[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t ring_a = smem_u32(ring), z_a = smem_u32(zbuf);
      long long n = 0;                                          // ring consume counter
      long long u = 0;                                          // unit counter
      for (long long pair = blockIdx.x; pair < p.npairs; pair += gridDim.x) {
        for (int k = 0; k < units_per_pair; ++k, ++u) {
          const int step = k >> 1, a = k & 1, zb = (int)(u & 1);
          const TcTerm& tm = p.term[step];
          mbar_wait(&zfull[zb], (uint32_t)((u >> 1) & 1));
          mbar_wait(&accempty[a], (uint32_t)(((u >> 1) & 1) ^ 1));
          tc_fence_after();
          const int kbpp = tm.kp / 16;
          const uint32_t sbo_b = 128u / (uint32_t)tm.ge;
          const uint32_t zbase = z_a + zb * 4 * zplane;
          const uint32_t d = tbase + a * 256;
          const bool wait_full = !p.a_shared || a == 0;
          const bool release = !p.a_shared || a == 1;
          const long long n0 = (p.a_shared && a == 1) ? n - tm.ksteps : n;
          for (int kk = 0; kk < tm.ksteps; ++kk) {
            const long long nn = n0 + kk;
            const int s = (int)(nn % S);
            if (wait_full) {
              mbar_wait(&full[s], (uint32_t)((nn / S) & 1));
              tc_fence_after();
            }
            const uint32_t a_hi = ring_a + s * 8192, a_lo = a_hi + 4096;
            const int pl = kk / kbpp, kb = kk % kbpp;
            const uint32_t zh = zbase + (pl * 2 + 0) * zplane + kb * 256;
            const uint32_t zl = zbase + (pl * 2 + 1) * zplane + kb * 256;
            const uint64_t dah = smem_desc(a_hi, 128, 256), dal = smem_desc(a_lo, 128, 256);
            const uint64_t dbh = smem_desc(zh, 128, sbo_b), dbl = smem_desc(zl, 128, sbo_b);
            umma_bf16(d, dah, dbh, kTcIdesc, (step == 0 && kk == 0) ? 0u : 1u);
            umma_bf16(d, dah, dbl, kTcIdesc, 1u);
            umma_bf16(d, dal, dbh, kTcIdesc, 1u);
            if (release) umma_commit(&empty[s]);
          }
          if (!p.a_shared || a == 0) n += tm.ksteps;
          umma_commit(&accfull[a]);
          umma_commit(&zempty[zb]);
        }
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ===================== Z builders (64 threads) =====================
    const int bt = threadIdx.x - 64;
    auto stage_band = [&](long long pair, int k, int sb) {
      // symmetric extension: contiguous band segment -> stg[sb] by two bulk copies
      const TcUnit un = tc_unit(p, pair, k);
      const TcTerm& tm = p.term[un.step];
      const int pos0 = un.tile * 256 + tm.g * tm.kmin;
      const int a = pos0 + p.ML;
      const int a4 = a & ~3;
      const int need = (a - a4) + tm.ge * (tm.nz - 1) + 8;
      int len = (need + 3) & ~3;
      if (a4 + len > p.stride) len = p.stride - a4;
      const float* src = bands + ((size_t)un.row * (p.J + 1) + tm.band) * 2 * p.stride + a4;
      float* dst = stg + (size_t)sb * 2 * p.stg_len;
      mbar_expect_tx(&stgbar[sb], (uint32_t)(2 * len * 4));
      bulk_load_g2s(dst, src, (uint32_t)(len * 4), &stgbar[sb]);
      bulk_load_g2s(dst + p.stg_len, src + p.stride, (uint32_t)(len * 4), &stgbar[sb]);
    };
    const bool sym = p.ext != 0;
    long long u = 0;
    long long first_pair = blockIdx.x;
    if (sym && bt == 0 && first_pair < p.npairs) stage_band(first_pair, 0, 0);
    for (long long pair = blockIdx.x; pair < p.npairs; pair += gridDim.x) {
      for (int k = 0; k < units_per_pair; ++k, ++u) {
        const int zb = (int)(u & 1), sb = (int)(u & 1);
        // prefetch the next unit's band segment
        if (sym && bt == 0) {
          long long np = pair;
          int nk = k + 1;
          if (nk == units_per_pair) { nk = 0; np = pair + gridDim.x; }
          if (np < p.npairs) stage_band(np, nk, sb ^ 1);
        }
        const TcUnit un = tc_unit(p, pair, k);
        const TcTerm& tm = p.term[un.step];
        const int pos0 = un.tile * 256 + tm.g * tm.kmin;
        float* sp = stg + (size_t)sb * 2 * p.stg_len;
        int off, lim;
        if (sym) {
          const int a = pos0 + p.ML;
          const int a4 = a & ~3;
          off = a - a4;
          const int need = off + tm.ge * (tm.nz - 1) + 8;
          int len = (need + 3) & ~3;
          if (a4 + len > p.stride) len = p.stride - a4;
          lim = len - 1;
          mbar_wait(&stgbar[sb], (uint32_t)((u >> 1) & 1));
        } else {
          // periodic: wrapped gather into the staging buffer
          off = 0;
          const int need = tm.ge * (tm.nz - 1) + 8;
          lim = need - 1;
          const float* b0 = bands + ((size_t)un.row * (p.J + 1) + tm.band) * 2 * p.stride;
          for (int i = bt; i < need; i += 64) {
            const int idx = (pos0 + i) & (p.N - 1);
            sp[i] = __ldg(b0 + idx);
            sp[p.stg_len + i] = __ldg(b0 + p.stride + idx);
          }
          named_bar(1, 64);
        }
        mbar_wait(&zempty[zb], (uint32_t)(((u >> 1) & 1) ^ 1));
        unsigned char* zb_ptr = zbuf + zb * 4 * zplane;
        for (int it = bt; it < 2 * tm.nz; it += 64) {
          const int pl = it >= tm.nz;
          const int j = it - pl * tm.nz;
          const float* src = sp + pl * p.stg_len;
          const int i0 = off + tm.ge * j;
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = src[min(i0 + e, lim)];
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float h0, l0, h1, l1;
            split_bf16(v[2 * e], h0, l0);
            split_bf16(v[2 * e + 1], h1, l1);
            hw[e] = pack_bf16x2(h0, h1);
            lw[e] = pack_bf16x2(l0, l1);
          }
          *reinterpret_cast<uint4*>(zb_ptr + (pl * 2 + 0) * zplane + j * 16) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          *reinterpret_cast<uint4*>(zb_ptr + (pl * 2 + 1) * zplane + j * 16) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
        fence_proxy_async_smem();
        mbar_arrive(&zfull[zb]);
        named_bar(1, 64);                                       // staging buffer free for the next prefetch
      }
    }
  } else {
    // ===================== epilogue (warps 4-7, TMEM lane group = warp & 3) =====================
    const int lg = warp & 3;
    unsigned char* epi = smem_raw + L.epi + lg * 16 * kTcEpiPitch;
    const int tl = lg * 16 + (lane >> 1);                       // template within the tile
    const bool odd = lane & 1;
    long long u = 0;
    for (long long pair = blockIdx.x; pair < p.npairs; pair += gridDim.x) {
      for (int k = 0; k < units_per_pair; ++k, ++u) {
        const TcUnit un = tc_unit(p, pair, k);
        const int a = k & 1;
        const int ti = p.J - un.step;
        const int t = un.mt * kTcTemplates + tl;
        const bool valid = t < p.n_t;
        const int tau_tile = un.tile * 256;
        mbar_wait(&accfull[a], (uint32_t)((u >> 1) & 1));
        tc_fence_after();
        PeakF best;
        best.m2 = -1.f; best.tau = 0x7fffffff; best.re = 0.f; best.im = 0.f;
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          float v[32];
          tmem_ld32(tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)(a * 256 + c * 32), v);
          if (c == 7) {                                         // accumulator fully read: release it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&accempty[a]);
          }
          float x[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) x[i] = __shfl_xor_sync(0xffffffffu, odd ? v[i] : v[16 + i], 1);
          // even lane: lags c*32 + 0..15 = (v[i], x[i]); odd lane: c*32 + 16.. = (x[i], v[16+i])
          float re[16], im[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) { re[i] = odd ? x[i] : v[i]; im[i] = odd ? v[16 + i] : x[i]; }
          const int tau = tau_tile + c * 32 + (odd ? 16 : 0);
          if (p.want_peaks && valid) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float m2 = mag2f(re[i], im[i]);
              if (m2 > best.m2) { best.m2 = m2; best.tau = tau + i; best.re = re[i]; best.im = im[i]; }
            }
          }
          if (p.want_corr) {
            // transpose: row (template) lane>>1, 16-byte chunks h*8 + i, chunk i >= 8 stored at (i ^ 4)
            unsigned char* rowp = epi + (lane >> 1) * kTcEpiPitch;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int cl = (odd ? 8 : 0) + i;
              const int cp = cl ^ (odd ? 4 : 0);
              *reinterpret_cast<float4*>(rowp + cp * 16) = make_float4(re[2 * i], im[2 * i], re[2 * i + 1], im[2 * i + 1]);
            }
            __syncwarp();
            // 8 instructions x 512 B: rows 2r, 2r+1 (lanes 0-15 / 16-31), chunk lane & 15
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              const int trow = 2 * r + (lane >> 4);
              const int cl = lane & 15;
              const int cp = cl ^ ((cl >> 3) << 2);
              const float4 val = *reinterpret_cast<const float4*>(epi + trow * kTcEpiPitch + cp * 16);
              const int tt = un.mt * kTcTemplates + lg * 16 + trow;
              if (tt < p.n_t) {
                float2* dst = corr + (((size_t)un.row * p.n_t + tt) * (p.J + 1) + ti) * p.N + tau_tile + c * 32;
                reinterpret_cast<float4*>(dst)[cl] = val;
              }
            }
            __syncwarp();
          }
        }
        if (p.want_peaks) {
          PeakF o;
          o.m2 = __shfl_xor_sync(0xffffffffu, best.m2, 1);
          o.tau = __shfl_xor_sync(0xffffffffu, best.tau, 1);
          o.re = __shfl_xor_sync(0xffffffffu, best.re, 1);
          o.im = __shfl_xor_sync(0xffffffffu, best.im, 1);
          if (beats(o.m2, o.tau, best.m2, best.tau)) best = o;
          if (!odd && valid) partials[(((size_t)un.row * p.n_t + t) * (p.J + 1) + ti) * p.ntiles + un.tile] = best;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

}  // namespace sidwt
