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
// Eq. (4): the terms are taken coarsest first and accumulate into
// the same TMEM accumulator; after term i the accumulator holds corr_i, which the
// epilogue stores (and reduces to per-tile peak partials) before term i-1 starts.
//
// One CTA = (row, template tile of 64, 512 lags): two accumulators of 128 lanes x
// 256 fp32 columns (all 512 TMEM columns).  Thread 0 streams the template operand
// (pre-built bf16 hi/lo images, 8 KB per 16-tap K step) through an S-stage ring of
// bulk async copies (mbarrier complete_tx) and issues the MMAs; tcgen05.commit
// frees ring stages and signals the epilogue.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace sidwt {

constexpr int kTcLags = 512;          // lags per CTA (two N=256 accumulators)
constexpr int kTcM = 128;             // MMA M: 64 templates x (re, im)
constexpr int kTcTemplates = 64;
constexpr int kTcStages = 10;         // template-operand ring depth (8 KB per stage)
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
  int N, J, ext, stride, ML, n_t, n_mt, ntiles, total_ksteps, nz_max;
  int want_corr, want_peaks;
  long long rows;
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
// The bank correlation kernel.
// smem: [mbar full[S], empty[S], acc][tmem slot][ring S x 8 KB][Z: 4 x nz_max x 16 B][peak scratch]
// ---------------------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(kTcThreads, 1)
k_correlate_tc(const float* __restrict__ bands, const unsigned char* __restrict__ img, float2* __restrict__ corr,
               PeakF* __restrict__ partials, TcParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + S;
  uint64_t* accbar = empty + S;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accbar + 1);
  unsigned char* ring = smem_raw + 1024;
  unsigned char* zbuf = ring + S * 8192;
  const int zplane = p.nz_max * 16;                                   // bytes per (plane, split)
  PeakF* red = reinterpret_cast<PeakF*>(zbuf + 4 * zplane);           // [64 templates][2 col halves]

  const int tile = blockIdx.x % p.ntiles;
  const long long bt = blockIdx.x / p.ntiles;
  const int mt = (int)(bt % p.n_mt);
  const long long row = bt / p.n_mt;
  const int tau0 = tile * kTcLags;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(accbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  const unsigned char* img_mt = img + (size_t)mt * p.total_ksteps * 8192;
  const int Q = p.total_ksteps;
  auto load_stage = [&](int q) {
    const int s = q % S;
    mbar_expect_tx(&full[s], 8192);
    bulk_load_g2s(ring + s * 8192, img_mt + (size_t)q * 8192, 8192, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < S && q < Q; ++q) load_stage(q);

  const float* brow = bands + (size_t)row * (p.J + 1) * 2 * p.stride;
  const uint32_t ring_a = smem_u32(ring);
  const uint32_t z_a = smem_u32(zbuf);
  int q = 0;                                                          // global K step counter

  for (int step = 0; step <= p.J; ++step) {
    const TcTerm tm = p.term[step];
    const int ti = p.J - step;                                        // scale index of corr after this term
    // ---- build Z for this term: Z[plane][split][j][e] = split(W[pos0 + ge j + e])
    {
      const float* b0 = brow + (size_t)tm.band * 2 * p.stride;
      const int pos0 = tau0 + tm.g * tm.kmin;
      const int items = 2 * tm.nz * 4;                                // (plane, row, e-pair)
      for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int ep = it & 3;
        const int j = (it >> 2) % tm.nz;
        const int pl = (it >> 2) / tm.nz;
        const float* src = b0 + (size_t)pl * p.stride;
        float v[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int pos = pos0 + tm.ge * j + 2 * ep + u;
          int idx;
          if (p.ext == 0) idx = pos & (p.N - 1);
          else idx = min(max(pos + p.ML, 0), p.stride - 1);
          v[u] = __ldg(src + idx);
        }
        float h0, l0, h1, l1;
        split_bf16(v[0], h0, l0);
        split_bf16(v[1], h1, l1);
        uint32_t* zh = reinterpret_cast<uint32_t*>(zbuf + (pl * 2 + 0) * zplane + j * 16) + ep;
        uint32_t* zl = reinterpret_cast<uint32_t*>(zbuf + (pl * 2 + 1) * zplane + j * 16) + ep;
        *zh = pack_bf16x2(h0, h1);
        *zl = pack_bf16x2(l0, l1);
      }
    }
    fence_proxy_async_smem();
    __syncthreads();

    // ---- MMA issue (one thread)
    if (threadIdx.x == 0) {
      tc_fence_after();
      const int kbpp = tm.kp / 16;
      const uint32_t sbo_b = 128u / (uint32_t)tm.ge;
      const uint32_t acc1_off = (uint32_t)(256 / tm.ge) * 16u;        // Z rows of lag offset 256
      for (int kk = 0; kk < tm.ksteps; ++kk, ++q) {
        const int s = q % S;
        mbar_wait(&full[s], (uint32_t)((q / S) & 1));
        tc_fence_after();
        const uint32_t a_hi = ring_a + s * 8192, a_lo = a_hi + 4096;
        const int pl = kk / kbpp, kb = kk % kbpp;
        const uint32_t zh = z_a + (pl * 2 + 0) * zplane + kb * 256;
        const uint32_t zl = z_a + (pl * 2 + 1) * zplane + kb * 256;
        const uint64_t dah = smem_desc(a_hi, 128, 256), dal = smem_desc(a_lo, 128, 256);
#pragma unroll
        for (int acc = 0; acc < 2; ++acc) {
          const uint32_t d = tbase + acc * 256;
          const uint64_t dbh = smem_desc(zh + acc * acc1_off, 128, sbo_b);
          const uint64_t dbl = smem_desc(zl + acc * acc1_off, 128, sbo_b);
          const uint32_t first = (step == 0 && kk == 0) ? 0u : 1u;
          umma_bf16(d, dah, dbh, kTcIdesc, first);
          umma_bf16(d, dah, dbl, kTcIdesc, 1u);
          umma_bf16(d, dal, dbh, kTcIdesc, 1u);
        }
        umma_commit(&empty[s]);
        // refill the stage consumed two steps ago (its MMAs are done or nearly so)
        const int qr = q - 2;
        if (qr >= 0 && qr + S < Q) {
          mbar_wait(&empty[qr % S], (uint32_t)((qr / S) & 1));
          load_stage(qr + S);
        }
      }
      umma_commit(accbar);
    }
    // ---- epilogue: corr_ti from TMEM (every thread)
    mbar_wait(accbar, (uint32_t)(step & 1));
    tc_fence_after();
    {
      const int lg = warp & 3, hh = warp >> 2;
      const int m = lg * 32 + lane;
      const int tl = m >> 1;                                          // template within the tile
      const int t = mt * kTcTemplates + tl;
      const bool odd = lane & 1;
      const bool valid = t < p.n_t;
      PeakF best;
      best.m2 = -1.f; best.tau = 0x7fffffff; best.re = 0.f; best.im = 0.f;
      float2* dst = valid ? corr + (((size_t)row * p.n_t + t) * (p.J + 1) + ti) * p.N : nullptr;
#pragma unroll 1
      for (int acc = 0; acc < 2; ++acc) {
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          const int col = acc * 256 + hh * 128 + c * 32;
          float v[32];
          tmem_ld32(tbase + ((uint32_t)(lg * 32) << 16) + (uint32_t)col, v);
          float x[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) x[i] = __shfl_xor_sync(0xffffffffu, odd ? v[i] : v[16 + i], 1);
          // even lane: lags col..col+15 = (v[i], x[i]); odd lane: col+16.. = (x[i], v[16+i])
          const int tau = tau0 + col + (odd ? 16 : 0);
          float re[16], im[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) { re[i] = odd ? x[i] : v[i]; im[i] = odd ? v[16 + i] : x[i]; }
          if (valid) {
            if (p.want_corr) {
              float4* o = reinterpret_cast<float4*>(dst + tau);
#pragma unroll
              for (int i = 0; i < 8; ++i) o[i] = make_float4(re[2 * i], im[2 * i], re[2 * i + 1], im[2 * i + 1]);
            }
            if (p.want_peaks) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float m2 = mag2f(re[i], im[i]);
                if (m2 > best.m2) { best.m2 = m2; best.tau = tau + i; best.re = re[i]; best.im = im[i]; }
              }
            }
          }
        }
      }
      if (p.want_peaks) {
        PeakF o;
        o.m2 = __shfl_xor_sync(0xffffffffu, best.m2, 1);
        o.tau = __shfl_xor_sync(0xffffffffu, best.tau, 1);
        o.re = __shfl_xor_sync(0xffffffffu, best.re, 1);
        o.im = __shfl_xor_sync(0xffffffffu, best.im, 1);
        if (beats(o.m2, o.tau, best.m2, best.tau)) best = o;
        if (!odd) red[tl * 2 + hh] = best;
      }
    }
    tc_fence_before();
    __syncthreads();
    if (p.want_peaks && threadIdx.x < kTcTemplates) {
      const int t = mt * kTcTemplates + threadIdx.x;
      if (t < p.n_t) {
        PeakF b = red[threadIdx.x * 2], o = red[threadIdx.x * 2 + 1];
        if (beats(o.m2, o.tau, b.m2, b.tau)) b = o;
        partials[(((size_t)row * p.n_t + t) * (p.J + 1) + ti) * p.ntiles + tile] = b;
      }
    }
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

}  // namespace sidwt
