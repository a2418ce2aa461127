// corr_tcs.cuh -- single-template correlation on the 5th-generation tensor cores
// ("single-template tensor-core correlation, Toeplitz-block GEMM"),
// sm_100a.  Float families, one template, symmetric extension.
//
// Term i (band W at stride g = 2^lg, taps b[k] at support positions kmin + k, k < n):
//     D[tau] = sum_k conj(b[k]) W[tau + g (kmin + k)]          (a5)
// Within residue class r (tau = r + g q) this is an ordinary correlation of the
// decimated sequence u_r[j] = W[r + g (kmin + j)] with the template.  Blocks of 64
// consecutive q form one GEMM column: with q = 64 blk + p,
//     D[r + g (64 blk + p)] = sum_j A[p][j] u_r[64 blk + j],   A[p][j] = conj(b[j - p])
// so A (M = 128 rows = 64 shifts p x (re, im)) is the template's Toeplitz matrix,
// shared by every row, term-wise constant, and precomputed once (image in global
// memory, streamed through a shared-memory ring by bulk copies); B (N = one column per
// (blk, r), N / 64 columns per row) is the band gathered at stride g, built in shared
// memory per K step by builder warps from the term's band segment; K runs over
// j in [0, n + 63) (padded to 16) for the re plane then the im plane.  fp32 operands
// are split into bf16 hi + lo; three MMAs (hi.hi + hi.lo + lo.hi) per plane and K step
// accumulate in fp32 in TMEM (same precision scheme as corr_tc.cuh).
//
// Eq. (4): one CTA owns a whole row (persistent over rows) and takes
// the terms coarsest first; the row's running corr lives in shared memory: the epilogue
// of term i adds D_i to it (acc = corr_{i+1} + D_i = corr_i), tracks the row's peak for
// that scale (a7) -- so no peak partials and no finalize kernel -- and one bulk copy
// stores corr_i (none in the peaks-only mode).
//
// Roles (448 threads):  warp 0 template-operand producer (bulk copies of image stages);
// warp 1 MMA issuer (one thread); warps 2-9 builders (+ the band segment loader);
// warps 10-13 epilogue (TMEM -> staging -> corr, four lane quarters of TMEM).
#pragma once
#include "corr_tc.cuh"

namespace sidwt {

constexpr int kTcsWarps = 14;
constexpr int kTcsThreads = 32 * kTcsWarps;
constexpr int kTcsFirstBuild = 2, kTcsBuildWarps = 8;
constexpr int kTcsFirstEpi = 10;
constexpr int kTcsAStage = 16384;               // one K step: 2 planes x (hi, lo) x 128 rows x 16 x bf16

struct TcsTerm {
  int band, lg, kmin, ntap, toff;
  int ksteps, kofs;                             // K steps (16 taps each) and first K step in the image
  int pos_lo;                                   // first fine-grid position of the term's band segment
  int a4;                                       // band index (pos + ML) of the segment start, 16-byte aligned
  int seg_len;                                  // floats loaded per plane (multiple of 4)
  int pad;                                      // shared-memory padding (floats) after every 64 g positions
};

struct TcsParams {
  int N, J, stride, ML, ncols, ncols_alloc, stages, seg_alloc;
  int want_corr;
  int merged;                                   // 1: hi | lo B products merged into one N = 2 ncols MMA
  int prof;                                     // debug (-DSIDWT_TC_PROFILE, SIDWT_TC_PROF=1): CTA 0 prints role waits
  long long rows;
  TcsTerm term[17];                             // indexed by processing step (0 = coarsest, A_J)
};

struct TcsSmem { size_t bars, ring, bst, stg, band, acc, total; };
__host__ __device__ inline TcsSmem tcs_smem_layout(const TcsParams& p) {
  TcsSmem L;
  L.bars = 0;
  L.ring = 1024;
  L.bst = L.ring + (size_t)p.stages * kTcsAStage;
  L.stg = L.bst + (size_t)2 * p.ncols * 128;      // two B stages of ncols x 16 x 2 planes x 2 splits x bf16
  L.band = L.stg + 128 * 32 * 4;
  L.acc = L.band + (size_t)2 * p.seg_alloc * 4;
  L.total = L.acc + (size_t)p.N * 8;              // the row's running corr (eq. (4) suffix sum)
  return L;
}

// Template Toeplitz images: img[kofs + ks][plane][split][4096 B], rows m = 64 c + p,
// K-major no-swizzle core matrices ((m, kk) at (m/8)*256 + (kk/8)*128 + (m%8)*16 + (kk%8)*2).
// conj(b) w = (br wr + bi wi) + i (br wi - bi wr): row (p, re) = (br | bi), (p, im) = (-bi | br).
__global__ void k_tcs_images(const float2* __restrict__ taps, TcsParams p, int total_ksteps,
                             unsigned char* __restrict__ img) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)total_ksteps * 4 * 128) return;
  const int m = (int)(gid % 128);
  const int split = (int)((gid / 128) % 2);
  const int plane = (int)((gid / 256) % 2);
  const int q = (int)(gid / 512);
  int step = 0;
  while (step < p.J && q >= p.term[step + 1].kofs) ++step;
  const TcsTerm tm = p.term[step];
  const int ks = q - tm.kofs;
  const int c = m >> 6, pp = m & 63;
  unsigned char* blk = img + ((size_t)q * 4 + plane * 2 + split) * 4096;
  for (int kk = 0; kk < 16; ++kk) {
    const int k = 16 * ks + kk - pp;            // template tap index
    float v = 0.f;
    if (k >= 0 && k < tm.ntap) {
      const float2 b = taps[tm.toff + k];
      v = (c == 0) ? (plane == 0 ? b.x : b.y) : (plane == 0 ? -b.y : b.x);
    }
    float hi, lo;
    split_bf16(v, hi, lo);
    const __nv_bfloat16 o = __float2bfloat16_rn(split == 0 ? hi : lo);
    *reinterpret_cast<__nv_bfloat16*>(blk + (m >> 3) * 256 + (kk >> 3) * 128 + (m & 7) * 16 + (kk & 7) * 2) = o;
  }
}

__device__ __forceinline__ bool elect_one_sync() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n" : "=r"(pred));
  return pred != 0;
}

// Pipeline stages: a term's K steps are taken plane by plane (all re-plane K steps, then all
// im-plane ones), two K steps per stage, so the band segment of one plane can be reloaded for
// the next term while the other plane is being processed.  Stage s of a term with ksteps K
// steps: plane s / nsp, K steps 2 (s % nsp) + {0, 1} (the last stage of a plane may hold one).
__host__ __device__ inline int tcs_nsp(int ksteps) { return (ksteps + 1) >> 1; }

// Builders: the B operand of one plane's stages (K-major bf16 hi / lo blocks).  Thread chunk
// (n, h, kk) = taps j = 16 (2 kp + kk) + 8 h + e (e < 8) of column n = blk g + r: position
// r + g (64 blk + kmin + j), segment index off0 + r + g (64 blk + j), shared-memory index
// idx + pad (idx >> (lg + 6)).  LG >= 0 makes the stride a compile-time constant.  Software
// pipelined: the band values of the next stage are loaded right after a stage is handed over.
template <int LG>
__device__ __forceinline__ void tcs_build_phase(const TcsParams& p, const TcsTerm& tm, int tb, const float* src,
                                                unsigned char* bst, uint64_t* bfull, uint64_t* bempty, uint32_t& qb,
                                                long long& w_be, long long& t_build) {
  constexpr int U = 2;                                        // chunks per thread per stage
  const int lg = LG >= 0 ? LG : tm.lg;
  const int g = 1 << lg, sh = lg + 6;
  const int off0 = tm.pos_lo + p.ML - tm.a4;                  // segment index of position pos_lo
  const int lim = p.stride - tm.a4;                           // segment indices >= lim are past the band
  const int bstage = p.ncols * 128, bblock = p.ncols * 32;
  const int nsp = tcs_nsp(tm.ksteps);
  int base[U], oo[U], kks[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int ci = tb + u * 32 * kTcsBuildWarps;
    const int n = ci % p.ncols;
    const int h = (ci / p.ncols) & 1;
    const int kk = ci / (2 * p.ncols);
    const int r = n & (g - 1), blk = n >> lg;
    base[u] = off0 + r + g * (64 * blk + 16 * kk + 8 * h);
    oo[u] = ci < p.ncols * 4 ? kk * 2 * bblock + (n >> 3) * 256 + h * 128 + (n & 7) * 16 : -1;
    kks[u] = kk;
  }
  auto load = [&](int kp, float (&v)[U][8]) {
    const int kc = min(2, tm.ksteps - 2 * kp);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i0 = base[u] + 32 * g * kp;
      if (oo[u] < 0 || kks[u] >= kc) {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[u][e] = 0.f;
      } else if (i0 + 7 * g < lim) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int idx = i0 + g * e;
          v[u][e] = src[idx + tm.pad * (idx >> sh)];
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int idx = i0 + g * e;
          v[u][e] = idx < lim ? src[idx + tm.pad * (idx >> sh)] : 0.f;
        }
      }
    }
  };
  float v[U][8];
  load(0, v);
  for (int kp = 0; kp < nsp; ++kp, ++qb) {
    const int kc = min(2, tm.ksteps - 2 * kp);
    const uint32_t bs = qb & 1, bph = (qb >> 1) & 1;
    TC_TWAIT(&bempty[bs], bph ^ 1, w_be);
    const long long t_b0 = TC_CLOCK();
    unsigned char* b0 = bst + (size_t)bs * bstage;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (oo[u] < 0 || kks[u] >= kc) continue;
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) split_bf16x2(v[u][2 * e], v[u][2 * e + 1], hi[e], lo[e]);
      *reinterpret_cast<uint4*>(b0 + oo[u]) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(b0 + oo[u] + bblock) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    fence_proxy_async_smem();
    mbar_arrive(&bfull[bs]);
    if (kp + 1 < nsp) load(kp + 1, v);
    t_build += TC_CLOCK() - t_b0;
  }
}

__global__ void __launch_bounds__(kTcsThreads, 1)
k_correlate_tcs(const float* __restrict__ bands, const unsigned char* __restrict__ img, float2* __restrict__ corr,
                int32_t* __restrict__ lag, float2* __restrict__ val,
                const __grid_constant__ TcsParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const TcsSmem L = tcs_smem_layout(p);
  const int S = p.stages;
  uint64_t* afull = reinterpret_cast<uint64_t*>(smem_raw);      // [S]
  uint64_t* aempty = afull + S;                                   // [S]
  uint64_t* bfull = aempty + S;                                   // [2]
  uint64_t* bempty = bfull + 2;                                   // [2]
  uint64_t* dfull = bempty + 2;                                   // [2]
  uint64_t* dempty = dfull + 2;                                   // [2]
  uint64_t* bandfull = dempty + 2;                                // [2] (one per plane)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bandfull + 2);
  PeakF* red = reinterpret_cast<PeakF*>(smem_raw + 512);          // [4] epilogue warp partials
  unsigned char* ring = smem_raw + L.ring;
  unsigned char* bst = smem_raw + L.bst;
  float* stg = reinterpret_cast<float*>(smem_raw + L.stg);
  float* band = reinterpret_cast<float*>(smem_raw + L.band);      // [2 planes][seg_alloc]
  float2* acc = reinterpret_cast<float2*>(smem_raw + L.acc);      // [N]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nterms = p.J + 1;
  const int bstage = p.ncols * 128;                               // bytes of one B stage
  const int bblock = p.ncols * 32;                                // bytes of one (plane, split) block

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&afull[i], 1); mbar_init(&aempty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bfull[i], 32 * kTcsBuildWarps); mbar_init(&bempty[i], 1);
      mbar_init(&dfull[i], 1); mbar_init(&dempty[i], 32 * 4);
    }
    mbar_init(&bandfull[0], 1);
    mbar_init(&bandfull[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tslot, 2 * p.ncols_alloc);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  // band segment of (row, step) -> smem (two planes), one thread
  // (pieces of 64 g positions, each followed by `pad` floats, so that the builders' strided
  //  reads of different 64-lag blocks fall into different banks)
  auto load_band = [&](long long row, int step, int pl) {
    const TcsTerm& tm = p.term[step];
    const float* src = bands + ((size_t)row * (p.J + 1) + tm.band) * 2 * p.stride + tm.a4 + (size_t)pl * p.stride;
    const int P = 64 << tm.lg;
    mbar_expect_tx(&bandfull[pl], tm.seg_len * 4u);
    for (int i = 0, o = 0; o < tm.seg_len; ++i, o += P)
      bulk_load_g2s(band + pl * p.seg_alloc + i * (P + tm.pad), src + o, (uint32_t)min(P, tm.seg_len - o) * 4u,
                    &bandfull[pl]);
  };

  if (warp == 0) {
    // ---------------- template operand producer
    if (lane == 0) {
      uint32_t q = 0;
      long long w_a = 0;
      for (long long row = blockIdx.x; row < p.rows; row += gridDim.x)
        for (int step = 0; step < nterms; ++step) {
          const TcsTerm& tm = p.term[step];
          const int nsp = tcs_nsp(tm.ksteps);
          for (int st = 0; st < 2 * nsp; ++st, ++q) {
            const int pl = st / nsp, k0 = 2 * (st % nsp), kc = min(2, tm.ksteps - k0);
            const uint32_t slot = q % S, ph = (q / S) & 1;
            TC_TWAIT(&aempty[slot], ph ^ 1, w_a);
            mbar_expect_tx(&afull[slot], kc * (kTcsAStage / 2));
            for (int kk = 0; kk < kc; ++kk)
              bulk_load_g2s(ring + (size_t)slot * kTcsAStage + kk * (kTcsAStage / 2),
                            img + (size_t)(tm.kofs + k0 + kk) * kTcsAStage + pl * (kTcsAStage / 2), kTcsAStage / 2,
                            &afull[slot]);
          }
        }
      if (p.prof && blockIdx.x == 0) printf("tcs cta0 producer: wait aempty %lld\n", w_a);
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp runs the loop (warp-uniform values stay in
    // uniform registers), one elected lane issues the MMAs and the commits
    {
      const uint32_t idesc0 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.ncols >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);
      const uint32_t idesc2 = (idesc0 & ~(0x3Fu << 17)) | ((uint32_t)((2 * p.ncols) >> 3) << 17);
      const bool merged = p.merged != 0;
      uint32_t q = 0, qb = 0, qd = 0;
      long long w_d = 0, w_af = 0, w_bf = 0;
      const long long t_start = TC_CLOCK();
      const uint32_t ring0 = smem_u32(ring), bst0 = smem_u32(bst);
      // descriptors differ only in their start address: precompute the fixed fields once
      const uint64_t dA = smem_desc(ring0, 128, 256), dB = smem_desc(bst0, 128, 256);
      const uint32_t bblock16 = (uint32_t)bblock >> 4, bstage16 = (uint32_t)bstage >> 4;
      for (long long row = blockIdx.x; row < p.rows; row += gridDim.x)
        for (int step = 0; step < nterms; ++step, ++qd) {
          const int nsp = tcs_nsp(p.term[step].ksteps);
          const int ksteps = p.term[step].ksteps;
          const uint32_t db = qd & 1, dph = (qd >> 1) & 1;
          TC_TWAIT(&dempty[db], dph ^ 1, w_d);
          tc_fence_after();
          const uint32_t dt = tmem + db * p.ncols_alloc;
          for (int st = 0; st < 2 * nsp; ++st, ++q, ++qb) {
            const int kc = min(2, ksteps - 2 * (st % nsp));
            const uint32_t slot = q % S, ph = (q / S) & 1;
            const uint32_t bs = qb & 1, bph = (qb >> 1) & 1;
            TC_TWAIT(&afull[slot], ph, w_af);
            TC_TWAIT(&bfull[bs], bph, w_bf);
            tc_fence_after();
            if (elect_one_sync()) {
              const uint64_t a0 = dA + (uint64_t)(slot * (kTcsAStage >> 4)), b0 = dB + (uint64_t)(bs * bstage16);
              for (int kk = 0; kk < kc; ++kk) {
                const uint64_t ahi = a0 + (uint64_t)(kk * (8192 >> 4));
                const uint64_t alo = ahi + (uint64_t)(4096 >> 4);
                const uint64_t bhi = b0 + (uint64_t)(kk * 2 * bblock16);
                const uint32_t acc0 = (st > 0 || kk > 0) ? 1u : 0u;
                if (merged) {
                  // D[:, 0:nc] += A_hi B_hi and D[:, nc:2nc] += A_hi B_lo in one MMA over the adjacent
                  // hi | lo blocks (N = 2 nc, A_hi read once), then D[:, 0:nc] += A_lo B_hi
                  umma_bf16(dt, ahi, bhi, idesc2, acc0);
                  umma_bf16(dt, alo, bhi, idesc0, 1u);
                } else {
                  const uint64_t blo = bhi + (uint64_t)bblock16;
                  umma_bf16(dt, ahi, bhi, idesc0, acc0);
                  umma_bf16(dt, ahi, blo, idesc0, 1u);
                  umma_bf16(dt, alo, bhi, idesc0, 1u);
                }
              }
              umma_commit(&aempty[slot]);
              umma_commit(&bempty[bs]);
            }
            __syncwarp();
          }
          if (elect_one_sync()) umma_commit(&dfull[db]);
          __syncwarp();
        }
      if (p.prof && blockIdx.x == 0 && lane == 0)
        printf("tcs cta0 mma: total %lld wait dempty %lld afull %lld bfull %lld\n", TC_CLOCK() - t_start, w_d, w_af, w_bf);
    }
  } else if (warp < kTcsFirstEpi) {
    // ---------------- builders (128 threads) + band loader (thread 64)
    const int tb = threadIdx.x - 32 * kTcsFirstBuild;
    uint32_t qb = 0, qband = 0;
    bool first = true;
    long long w_band = 0, w_be = 0, t_build = 0;
    for (long long row = blockIdx.x; row < p.rows; row += gridDim.x)
      for (int step = 0; step < nterms; ++step, ++qband) {
        const TcsTerm& tm = p.term[step];
        if (first && tb == 0) { load_band(row, step, 0); load_band(row, step, 1); }
        first = false;
        for (int pl = 0; pl < 2; ++pl) {
          TC_TWAIT(&bandfull[pl], qband & 1, w_band);
          const float* src = band + pl * p.seg_alloc;
          switch (tm.lg) {
            case 1: tcs_build_phase<1>(p, tm, tb, src, bst, bfull, bempty, qb, w_be, t_build); break;
            case 2: tcs_build_phase<2>(p, tm, tb, src, bst, bfull, bempty, qb, w_be, t_build); break;
            case 3: tcs_build_phase<3>(p, tm, tb, src, bst, bfull, bempty, qb, w_be, t_build); break;
            case 4: tcs_build_phase<4>(p, tm, tb, src, bst, bfull, bempty, qb, w_be, t_build); break;
            case 5: tcs_build_phase<5>(p, tm, tb, src, bst, bfull, bempty, qb, w_be, t_build); break;
            case 6: tcs_build_phase<6>(p, tm, tb, src, bst, bfull, bempty, qb, w_be, t_build); break;
            default: tcs_build_phase<-1>(p, tm, tb, src, bst, bfull, bempty, qb, w_be, t_build); break;
          }
          // every builder is done with this plane's segment: load the next term's (overlaps the
          // other plane's stages)
          named_bar(1, 32 * kTcsBuildWarps);
          if (tb == 0) {
            long long nrow = row;
            int nstep = step + 1;
            if (nstep == nterms) { nstep = 0; nrow += gridDim.x; }
            if (nrow < p.rows) load_band(nrow, nstep, pl);
          }
        }
      }
    if (p.prof && blockIdx.x == 0 && tb == 0)
      printf("tcs cta0 builder: wait band %lld bempty %lld build %lld\n", w_band, w_be, t_build);
  } else {
    // ---------------- epilogue (128 threads, TMEM lane quarter = warp % 4)
    const int te = threadIdx.x - 32 * kTcsFirstEpi;
    const int quarter = warp & 3;
    const int m = 32 * quarter + lane;                            // TMEM lane = A row (64 c + p)
    uint32_t qd = 0;
    long long w_df = 0, t_epi = 0;
    for (long long row = blockIdx.x; row < p.rows; row += gridDim.x) {
      for (int step = 0; step < nterms; ++step, ++qd) {
        const TcsTerm& tm = p.term[step];
        const int ti = p.J - step;
        const int g = 1 << tm.lg;
        const uint32_t db = qd & 1, dph = (qd >> 1) & 1;
        float2* cur = p.want_corr ? corr + ((size_t)row * (p.J + 1) + ti) * p.N : nullptr;
        PeakF best; best.m2 = 0.f; best.tau = -1; best.re = 0.f; best.im = 0.f;
        TC_TWAIT(&dfull[db], dph, w_df);
        const long long t_e0 = TC_CLOCK();
        tc_fence_after();
        const int lgR = tm.lg < 5 ? tm.lg : 5;
        const int R = 1 << lgR;                                   // residues per chunk
        const int nch = (p.ncols + 31) / 32;
        const int cw = p.ncols < 32 ? p.ncols : 32;               // columns per chunk
        for (int ch = 0; ch < nch; ++ch) {
          const int n0 = ch * 32;
          uint32_t v[32];
          const uint32_t ta = tmem + db * p.ncols_alloc + ((uint32_t)(32 * quarter) << 16) + n0;
          tmem_ld32_nowait(ta, v);
          tmem_wait_ld(v);
          if (p.merged) {                                         // add the A_hi B_lo half
            uint32_t w[32];
            tmem_ld32_nowait(ta + p.ncols, w);
            tmem_wait_ld(w);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(w[i]));
          }
          if (ch == nch - 1) { tc_fence_before(); mbar_arrive(&dempty[db]); }
          // staging: row m, 32 floats, 16-byte chunks XOR-swizzled by m % 8
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4)
            *reinterpret_cast<uint4*>(stg + m * 32 + ((c4 ^ (m & 7)) << 2)) = make_uint4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
          if (ch == 0 && te == 0) bulk_wait_read_all();            // corr_{i+1} store has read acc
          named_bar(2, 128);
          // outputs of the chunk in lag order: idx -> (bl, p, rr); n_local = bl R + rr
          const int r0 = n0 & (g - 1), blk0 = n0 >> tm.lg;
          // acc[tau] (+)= D: lanes take consecutive lags
          const int nper = (64 * cw) / 128;
#pragma unroll 4
          for (int i = 0; i < nper; ++i) {
            const int idx = te + 128 * i;
            const int rr = idx & (R - 1);
            const int pp = (idx >> lgR) & 63;
            const int bl = idx >> (lgR + 6);
            const int nl = (bl << lgR) + rr;
            const int tau = r0 + rr + g * (64 * (blk0 + bl) + pp);
            const int cre = ((nl >> 2) ^ (pp & 7)) << 2;
            float re = stg[pp * 32 + cre + (nl & 3)];
            float im = stg[(64 + pp) * 32 + cre + (nl & 3)];
            if (step > 0) {
              const float2 a = acc[tau];
              re += a.x; im += a.y;
            }
            acc[tau] = make_float2(re, im);
            const float m2 = mag2f(re, im);
            if (best.tau < 0 || m2 > best.m2 || (m2 == best.m2 && tau < best.tau)) {
              best.m2 = m2; best.tau = tau; best.re = re; best.im = im;
            }
          }
          named_bar(2, 128);
        }
        // the row's peak at this scale: warp argmax (largest |.|^2, then smallest lag), then 4 warps
        const unsigned mb = best.tau >= 0 ? __float_as_uint(best.m2) : 0u;
        const unsigned mmax = __reduce_max_sync(0xffffffffu, mb);
        const unsigned cand = (best.tau >= 0 && mb == mmax) ? (unsigned)best.tau : 0xffffffffu;
        const unsigned tmin = __reduce_min_sync(0xffffffffu, cand);
        if (best.tau >= 0 && (unsigned)best.tau == tmin) red[warp - kTcsFirstEpi] = best;
        fence_proxy_async_smem();                                  // acc writes -> visible to the bulk copy
        named_bar(2, 128);
        if (te == 0 && cur) {
          bulk_store_s2g(cur, acc, (uint32_t)p.N * 8u);
          bulk_commit();
        }
        if (te == 0 && lag) {
          PeakF b = red[0];
          for (int w = 1; w < 4; ++w) {
            const PeakF o = red[w];
            if (o.m2 > b.m2 || (o.m2 == b.m2 && o.tau < b.tau)) b = o;
          }
          const size_t e = (size_t)row * (p.J + 1) + ti;
          lag[e] = b.tau;
          if (val) val[e] = make_float2(b.re, b.im);
        }
        named_bar(2, 128);
        t_epi += TC_CLOCK() - t_e0;
      }
    }
    if (te == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    if (p.prof && blockIdx.x == 0 && te == 0) printf("tcs cta0 epilogue: wait dfull %lld work %lld\n", w_df, t_epi);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 2 * p.ncols_alloc);
}

}  // namespace sidwt
