// corr_tcs.cuh -- single-template correlation on the 5th-generation tensor cores
// ("single-template tensor-core correlation, Toeplitz-block GEMM"),
// sm_100a.  Float families, one template, symmetric extension.
//
// Term i (band W at stride g = 2^lg, taps b[k] at support positions kmin + k, k < n):
//     D[tau] = sum_k conj(b[k]) W[tau + g (kmin + k)]          (a5)
// Within residue class r (tau = r + g q) this is an ordinary correlation of the
// decimated sequence u_r[j] = W[r + g (kmin + j)] with the template (the paper's even/odd
// branch sequences).  Blocks of 64 consecutive q form one data
// row of the GEMM: with q = 64 blk + p,
//     D[r + g (64 blk + p)] = sum_j u_r[64 blk + j] T[p][j],   T[p][j] = conj(b[j - p])
// so the M side (128 rows, one per n = blk g + r, N / 64 of them per row) is the band read
// at stride g, and the N side (64 shifts p x (re, im) = 128 columns, interleaved 2 p + c) is
// the template's Toeplitz matrix -- shared by every row, term-wise constant, precomputed
// once (image in global memory, streamed through a shared-memory ring by bulk copies).
// K runs over j in [0, n + 63) (padded to 16) for the re plane, then the im plane.  fp32
// operands are split into bf16 hi + lo; per plane and K step two MMAs accumulate in fp32
// in TMEM: data_hi x [T_hi | T_lo] (N = 256: the template's hi and lo images are adjacent,
// so data_hi is read once for both) and data_lo x T_hi (N = 128), i.e. hi.hi + hi.lo + lo.hi
// (the precision scheme of corr_tc.cuh).
//
// The data operand without per-K-step building.  A[n][k] = u_r[64 blk + k] is a Hankel
// matrix in (blk, k): K step ks (k = 16 ks + kk) of row n reads the same values as
// K step ks - 4 of row n + g.  So one buffer per (term, plane, split) holds every
// value once, as 16-byte rows R[kc][n'] = u_r[64 blk' + 8 kc + e], e < 8 (n' = blk' g + r,
// kc < 8 the 8-tap chunk inside a 64-tap window, n' up to ncols + g X_kc), and the
// operand of K step ks = 4 X + i is the canonical K-major no-swizzle view starting at
// row (2 i, X g) with SBO = 128 B (8 consecutive rows) and LBO = the distance of chunk
// planes 2 i and 2 i + 1.  Converter warps fill the buffer once per (term, plane) with
// coalesced loads of the fine-grid band from global memory (a permutation of the
// band segment, no duplication), split into hi / lo bf16; the MMA then runs all K steps
// of the plane from it.  Three buffers (term-plane s in buffer s % 3) let the converters run
// up to two term-planes ahead of the MMAs.
//
// Eq. (4) and the peaks in one epilogue pass.  TMEM lane n holds the
// data row (blk, r): 64 consecutive lags of residue class r, re and im side by side.  One
// CTA owns a whole row (persistent over rows) and takes the terms coarsest first; the
// row's running corr lives in shared memory (complex, one float2 of padding per 64 lags,
// so the lanes of a warp hit different banks for every g).  The epilogue of term i adds
// D_i to it (acc = corr_{i+1} + D_i = corr_i) straight from the TMEM registers, tracks the
// row's peak at that scale (a7) on the same values -- no peak partials, no finalize
// kernel -- and writes corr_i (none in the peaks-only mode).
//
// Roles (512 threads):  warp 0 template-operand producer (bulk copies of image stages);
// warp 1 MMA issuer (the warp runs the loop, one elected lane issues); warps 2-4 convert
// the re plane, warps 5-7 the im plane; warps 8-15 epilogue (two warps per TMEM lane
// quarter: shifts p < 32 and p >= 32).
#pragma once
#include "corr_tc.cuh"

namespace sidwt {

constexpr int kTcsWarps = 16;
constexpr int kTcsThreads = 32 * kTcsWarps;
constexpr int kTcsRegsProd = 160, kTcsRegsEpi = 96;   // registers per thread after setmaxnreg (8 x prod + 8 x epi = 2048)
constexpr int kTcsFirstConv = 2, kTcsConvWarps = 6;     // 3 warps (96 threads) per plane
constexpr int kTcsConvThreads = 96;
constexpr int kTcsFirstEpi = 8, kTcsEpiWarps = 8, kTcsEpiThreads = 32 * kTcsEpiWarps;
constexpr int kTcsSlots = 3;                     // data-operand buffers (term-plane s uses slot s % 3)
constexpr int kTcsAStage = 16384;               // one K step: 2 planes x (hi, lo) x 128 rows x 16 x bf16

struct TcsTerm {
  int band, lg, kmin, ntap, toff;
  int ksteps, kofs;                             // K steps (16 taps each) and first K step in the image
  int kcoff[9];                                 // first buffer row of chunk plane kc (kcoff[8] = rows per split)
  int pf_a4, pf_len;                            // band floats [pf_a4, pf_a4 + pf_len) the converters read (L2 prefetch)
};

struct TcsParams {
  int N, J, stride, ML, ncols, ncols_alloc, stages, brows_max;
  int want_corr;
  int prof;                                     // debug (-DSIDWT_TC_PROFILE, SIDWT_TC_PROF=1): CTA 0 prints role waits
  long long rows;
  TcsTerm term[17];                             // indexed by processing step (0 = coarsest, A_J)
};

// buffer rows of a term: chunk plane kc holds n' in [0, ncols + g X_kc), X_kc the largest
// column shift (ks / 4) of the K steps ks = 4 X + kc / 2 that read it (none: empty plane)
__host__ __device__ inline void tcs_term_rows(TcsTerm& tm, int ncols) {
  const int g = 1 << tm.lg;
  int o = 0;
  for (int kc = 0; kc < 8; ++kc) {
    int X = -1;
    for (int ks = 0; ks < tm.ksteps; ++ks)
      if ((ks & 3) == (kc >> 1)) X = ks >> 2;
    tm.kcoff[kc] = o;
    o += X < 0 ? 0 : ncols + g * X;
  }
  tm.kcoff[8] = o;
}

// padded position of lag tau in the running corr (float2 units): one float2 of padding per 64
// lags, so that the 16 lanes of a 64-bit shared-memory phase (16 consecutive data rows n =
// blk g + r, same shift p) fall on different banks for every g; a thread's run of 8 shifts
// is a base plus compile-time offsets
__host__ __device__ __forceinline__ int tcs_pad(int tau) { return tau + (tau >> 6); }

struct TcsSmem { size_t bars, ring, bbuf, bslot, acc, total; };
__host__ __device__ inline TcsSmem tcs_smem_layout(const TcsParams& p) {
  TcsSmem L;
  L.bars = 0;
  L.ring = 1024;
  L.bbuf = L.ring + (size_t)p.stages * kTcsAStage;
  L.bslot = (size_t)2 * p.brows_max * 16;         // one plane: (hi, lo) x rows x 16 B
  L.acc = L.bbuf + kTcsSlots * L.bslot;
  L.total = L.acc + (size_t)(tcs_pad(p.N) + 2) * 8;   // the row's running corr (eq. (4) suffix sum), float2
  return L;
}

// Template Toeplitz images: img[kofs + ks][plane][split][4096 B], rows m = 2 p + c,
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
  const int c = m & 1, pp = m >> 1;
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

__device__ __forceinline__ void prefetch_l2(const void* g, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" :: "l"(g), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool elect_one_sync() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n" : "=r"(pred));
  return pred != 0;
}


// Pipeline stages of the template operand: a term's K steps are taken plane by plane (all
// re-plane K steps, then all im-plane ones), two K steps per stage.  Stage s of a term with
// ksteps K steps: plane s / nsp, K steps 2 (s % nsp) + {0, 1} (the last stage of a plane may
// hold one).
__host__ __device__ inline int tcs_nsp(int ksteps) { return (ksteps + 1) >> 1; }

// Converter: one plane of one term -> buffer rows (hi block, then lo block).  Rows come in
// groups of V = min(4, g) consecutive residues r (same kc, same blk'): their band positions
// r + g (kmin + 64 blk' + 8 kc + e) are V consecutive floats for every e, so a group is
// 8 vector loads from global memory (coalesced across the warp) and 2 V 16-byte shared
// stores.  Thread tc takes groups q = tc + 96 b.  A round is G groups (3 of 4 rows or 4 of
// 2: at most 96 floats in registers); the first round -- for C3 the whole term-plane when
// g >= 4 -- is loaded before waiting for the buffer, so the load latency overlaps the MMAs
// still reading it.  Positions at or past the band stride meet zero Toeplitz entries: their
// loads are clamped to the last in-band vector (finite values; V divides idx and stride).
template <int V>
__device__ __forceinline__ void tcs_convert(const TcsParams& p, const TcsTerm& tm, int tc, const float* __restrict__ src,
                                            unsigned char* buf, uint64_t* bfull, uint64_t* bempty, uint32_t par,
                                            long long& w_be) {
  constexpr int G = 2;
  const int lg = tm.lg;
  const int g = 1 << lg;
  const int brows = tm.kcoff[8];
  const int nq = brows / V;                                   // every chunk plane has a multiple of 4 rows
  const int base = p.ML + g * tm.kmin;                        // band index of (r = 0, m = 0), a multiple of V
  const int lim = p.stride - V;
  // register slot k of a group holds residue row (k + rot) % V, rot = (lane / (8 / V)) % V: the 8
  // lanes of a 16-byte store phase then write 8 different 16-byte slots (conflict-free)
  const int rot = (tc >> (V == 4 ? 1 : 2)) & (V - 1);
  auto load = [&](int b, float (&v)[8][V]) {
    const int q = tc + kTcsConvThreads * b;
    if (q < nq) {
      const int t = q * V;
      int kc = 0;
#pragma unroll
      for (int k = 1; k < 8; ++k) kc += t >= tm.kcoff[k] ? 1 : 0;
      const int n = t - tm.kcoff[kc];
      const int i0 = base + (n & (g - 1)) + g * (64 * (n >> lg) + 8 * kc);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int idx = min(i0 + g * e, lim);
        if constexpr (V == 4) {
          const float4 w = __ldg(reinterpret_cast<const float4*>(src + idx));
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int j = (k + rot) & 3;
            v[e][k] = (j & 2) ? ((j & 1) ? w.w : w.z) : ((j & 1) ? w.y : w.x);
          }
        } else {
          const float2 w = __ldg(reinterpret_cast<const float2*>(src + idx));
          v[e][0] = rot ? w.y : w.x; v[e][1] = rot ? w.x : w.y;
        }
      }
    }
  };
  auto store = [&](int b, const float (&v)[8][V]) {
    const int q = tc + kTcsConvThreads * b;
    if (q < nq) {
      const int t = q * V;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_bf16x2(v[2 * e][k], v[2 * e + 1][k], hi[e], lo[e]);
        const int r = t + ((k + rot) & (V - 1));                // register slot k holds row (k + rot) % V
        *reinterpret_cast<uint4*>(buf + (size_t)r * 16) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(buf + (size_t)(brows + r) * 16) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
  };
  const int nb = (nq + kTcsConvThreads - 1) / kTcsConvThreads;
  float v[G][8][V];
#pragma unroll
  for (int k = 0; k < G; ++k) load(k, v[k]);
  TC_TWAIT(bempty, par ^ 1, w_be);
  for (int b0 = 0; b0 < nb; b0 += G) {
    if (b0 > 0) {
#pragma unroll
      for (int k = 0; k < G; ++k) load(b0 + k, v[k]);
    }
#pragma unroll
    for (int k = 0; k < G; ++k) store(b0 + k, v[k]);
  }
  fence_proxy_async_smem();
  mbar_arrive(bfull);
}

// Epilogue of one term for 16 shifts p0 .. p0 + 15 of data row n = blk g + r (TMEM lane n):
// D = v + w (the hi.hi + lo.hi and hi.lo accumulators, columns (2 p + c)), acc (+)= D (eq. (4):
// acc = corr_{i+1} + D_i = corr_i), corr_i stores, running peak (lags increase with p: the
// first maximum wins).
template <int LG>
__device__ __forceinline__ void tcs_epi16(const uint32_t (&v)[32], const uint32_t (&w)[32], int n, int p0, bool first,
                                          float2* acc, float2* cur, PeakF& best) {
  constexpr int g = 1 << LG;
  const int tau0 = (n & (g - 1)) + g * (64 * (n >> LG) + p0);
  const int b = tcs_pad(tau0);
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {                              // 8 shifts at a time: loads, then stores
    float2 d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      d[i] = make_float2(__uint_as_float(v[16 * hh + 2 * i]) + __uint_as_float(w[16 * hh + 2 * i]),
                         __uint_as_float(v[16 * hh + 2 * i + 1]) + __uint_as_float(w[16 * hh + 2 * i + 1]));
    const int ii = 8 * hh;
    if (!first) {
      float2 a[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = acc[b + g * (ii + i) + ((g * (ii + i)) >> 6)];
#pragma unroll
      for (int i = 0; i < 8; ++i) { d[i].x += a[i].x; d[i].y += a[i].y; }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[b + g * (ii + i) + ((g * (ii + i)) >> 6)] = d[i];
    if (cur) {
#pragma unroll
      for (int i = 0; i < 8; ++i) __stcs(cur + tau0 + g * (ii + i), d[i]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float m2 = mag2f(d[i].x, d[i].y);
      if (m2 > best.m2) { best.m2 = m2; best.tau = tau0 + g * (ii + i); best.re = d[i].x; best.im = d[i].y; }
    }
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
  uint64_t* bfull = aempty + S;                                   // [kTcsSlots]
  uint64_t* bempty = bfull + kTcsSlots;                           // [kTcsSlots]
  uint64_t* dfull = bempty + kTcsSlots;                           // [2]
  uint64_t* dempty = dfull + 2;                                   // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dempty + 2);
  PeakF* red = reinterpret_cast<PeakF*>(smem_raw + 512);          // [2][8] epilogue warp partials
  unsigned char* ring = smem_raw + L.ring;
  unsigned char* bbuf = smem_raw + L.bbuf;
  float2* acc = reinterpret_cast<float2*>(smem_raw + L.acc);      // [tcs_pad(N) + 2], padded
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nterms = p.J + 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&afull[i], 1); mbar_init(&aempty[i], 1); }
    for (int i = 0; i < kTcsSlots; ++i) { mbar_init(&bfull[i], kTcsConvThreads); mbar_init(&bempty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], kTcsEpiThreads); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tslot, 512);                          // two accumulators of 256 columns
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  // register budget by role (whole warpgroups 0-1 loader / MMA / converters, 2-3 epilogue; setmaxnreg
  // at the head of each arm so that the arm's allocation follows it)
  if (warp < kTcsFirstEpi) {
  set_max_regs<kTcsRegsProd>();
  if (warp == 0) {
    // ---------------- template operand producer
    if (lane == 0) {
      uint32_t q = 0;
      long long w_a = 0;
      for (long long row = blockIdx.x; row < p.rows; row += gridDim.x)
        for (int step = 0; step < nterms; ++step) {
          const TcsTerm& tm = p.term[step];
          const int nsp = tcs_nsp(tm.ksteps);
          {                                                       // the band segments two terms ahead -> L2
            long long nrow = row;
            int nstep = step + 2;
            if (nstep >= nterms) { nstep -= nterms; nrow += gridDim.x; }
            if (nrow < p.rows) {
              const TcsTerm& tn = p.term[nstep];
              const float* b0 = bands + ((size_t)nrow * (p.J + 1) + tn.band) * 2 * p.stride + tn.pf_a4;
              prefetch_l2(b0, (uint32_t)tn.pf_len * 4u);
              prefetch_l2(b0 + p.stride, (uint32_t)tn.pf_len * 4u);
            }
          }
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
    const uint32_t idesc_base = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t idesc256 = idesc_base | ((uint32_t)(256 >> 3) << 17);
    const uint32_t idesc128 = idesc_base | ((uint32_t)(128 >> 3) << 17);
    uint32_t q = 0, qt = 0;
    long long w_d = 0, w_af = 0, w_bf = 0;
    const long long t_start = TC_CLOCK();
    const uint32_t ring0 = smem_u32(ring), bbuf0 = smem_u32(bbuf);
    const uint64_t dT = smem_desc(ring0, 128, 256);              // template: K-major, 8-row groups 256 B apart
    const uint64_t dD0 = smem_desc(0, 0, 128);                   // data: fixed fields (LBO and start per K step)
    for (long long row = blockIdx.x; row < p.rows; row += gridDim.x)
      for (int step = 0; step < nterms; ++step, ++qt) {
        const TcsTerm& tm = p.term[step];
        const int ksteps = tm.ksteps, g = 1 << tm.lg;
        const uint32_t brows16 = (uint32_t)tm.kcoff[8];        // lo block offset in 16-byte units
        const uint32_t db = qt & 1, dph = (qt >> 1) & 1;
        TC_TWAIT(&dempty[db], dph ^ 1, w_d);
        tc_fence_after();
        const uint32_t dt = tmem + db * 256;
        for (int pl = 0; pl < 2; ++pl) {
          const uint32_t sidx = 2 * qt + pl, bs = sidx % kTcsSlots;       // term-plane sidx, its buffer
          TC_TWAIT(&bfull[bs], (sidx / kTcsSlots) & 1, w_bf);
          tc_fence_after();
          const uint32_t b16 = (bbuf0 + bs * (uint32_t)L.bslot) >> 4;
          uint32_t slot = 0;
          for (int ks = 0; ks < ksteps; ++ks) {
            if ((ks & 1) == 0) {
              slot = q % S;
              TC_TWAIT(&afull[slot], (q / S) & 1, w_af);
              tc_fence_after();
            }
            const int i2 = 2 * (ks & 3), X = ks >> 2;
            const uint32_t row0 = (uint32_t)(tm.kcoff[i2] + X * g);
            const uint32_t lbo16 = (uint32_t)(tm.kcoff[i2 + 1] - tm.kcoff[i2]);
            const uint64_t ahi = dD0 | ((uint64_t)lbo16 << 16) | (uint64_t)(b16 + row0);
            const uint64_t alo = ahi + brows16;
            const uint64_t thi = dT + (uint64_t)((slot * kTcsAStage + (ks & 1) * (kTcsAStage / 2)) >> 4);
            const bool last_of_stage = (ks & 1) || ks == ksteps - 1;
            if (elect_one_sync()) {
              umma_bf16(dt, ahi, thi, idesc256, (pl > 0 || ks > 0) ? 1u : 0u);   // [hi.hi | hi.lo]
              umma_bf16(dt, alo, thi, idesc128, 1u);                             // + lo.hi
              if (last_of_stage) umma_commit(&aempty[slot]);
            }
            __syncwarp();
            if (last_of_stage) ++q;
          }
          if (elect_one_sync()) umma_commit(&bempty[bs]);
          __syncwarp();
        }
        if (elect_one_sync()) umma_commit(&dfull[db]);
        __syncwarp();
      }
    if (p.prof && blockIdx.x == 0 && lane == 0)
      printf("tcs cta0 mma: total %lld wait dempty %lld afull %lld bfull %lld\n", TC_CLOCK() - t_start, w_d, w_af, w_bf);
  } else if (warp < kTcsFirstEpi) {
    // ---------------- converters: warps 2-4 the re plane, 5-7 the im plane
    const int pl = (warp - kTcsFirstConv) / 3;
    const int tc = threadIdx.x - 32 * kTcsFirstConv - kTcsConvThreads * pl;
    uint32_t qt = 0;
    long long w_be = 0;
    for (long long row = blockIdx.x; row < p.rows; row += gridDim.x)
      for (int step = 0; step < nterms; ++step, ++qt) {
        const TcsTerm& tm = p.term[step];
        const float* src = bands + (((size_t)row * (p.J + 1) + tm.band) * 2 + pl) * p.stride;
        const uint32_t sidx = 2 * qt + pl, bs = sidx % kTcsSlots;         // term-plane sidx, its buffer
        unsigned char* buf = bbuf + (size_t)bs * L.bslot;
        const uint32_t par = (sidx / kTcsSlots) & 1;
        if (tm.lg >= 2) tcs_convert<4>(p, tm, tc, src, buf, &bfull[bs], &bempty[bs], par, w_be);
        else tcs_convert<2>(p, tm, tc, src, buf, &bfull[bs], &bempty[bs], par, w_be);
      }
    if (p.prof && blockIdx.x == 0 && tc == 0) printf("tcs cta0 converter %d: wait bempty %lld\n", pl, w_be);
  }
  } else {
    set_max_regs<kTcsRegsEpi>();
    // ---------------- epilogue (256 threads): TMEM lane quarter = warp % 4 (data rows n),
    // half h = shifts p in [32 h, 32 h + 32)
    const int te = threadIdx.x - 32 * kTcsFirstEpi;
    const int quarter = warp & 3, h = (warp - kTcsFirstEpi) >> 2;
    const int n = 32 * quarter + lane;                            // TMEM lane = data row
    const bool live = n < p.ncols;
    uint32_t qt = 0;
    long long w_df = 0, t_epi = 0, t_b = 0;
    for (long long row = blockIdx.x; row < p.rows; row += gridDim.x) {
      for (int step = 0; step < nterms; ++step, ++qt) {
        const TcsTerm& tm = p.term[step];
        const int ti = p.J - step;
        const uint32_t db = qt & 1, dph = (qt >> 1) & 1;
        float2* cur = p.want_corr ? corr + ((size_t)row * (p.J + 1) + ti) * p.N : nullptr;
        const bool first = step == 0;
        TC_TWAIT(&dfull[db], dph, w_df);
        const long long t_e0 = TC_CLOCK();
        tc_fence_after();
        PeakF best; best.m2 = -1.f; best.tau = 0; best.re = 0.f; best.im = 0.f;
#pragma unroll 1
        for (int s2 = 0; s2 < 2; ++s2) {
          const int p0 = 32 * h + 16 * s2;
          const uint32_t ta = tmem + db * 256 + ((uint32_t)(32 * quarter) << 16) + 2 * p0;
          uint32_t v[32], w[32];
          tmem_ld32_nowait(ta, v);
          tmem_ld32_nowait(ta + 128, w);
          tmem_wait_ld(v);
          tmem_wait_ld(w);
          if (s2 == 1) { tc_fence_before(); mbar_arrive(&dempty[db]); }   // this thread's TMEM reads are done
          if (live) {
            switch (tm.lg) {
              case 1: tcs_epi16<1>(v, w, n, p0, first, acc, cur, best); break;
              case 2: tcs_epi16<2>(v, w, n, p0, first, acc, cur, best); break;
              case 3: tcs_epi16<3>(v, w, n, p0, first, acc, cur, best); break;
              case 4: tcs_epi16<4>(v, w, n, p0, first, acc, cur, best); break;
              case 5: tcs_epi16<5>(v, w, n, p0, first, acc, cur, best); break;
              case 6: tcs_epi16<6>(v, w, n, p0, first, acc, cur, best); break;
              default: tcs_epi16<7>(v, w, n, p0, first, acc, cur, best); break;
            }
          }
        }
        // warp argmax (largest |.|^2, then smallest lag), then the 8 warps (red double-buffered
        // by term parity: te 0 reads it after the barrier, the next term writes the other half)
        const unsigned mb = best.m2 >= 0.f ? __float_as_uint(best.m2) : 0u;   // m2 >= 0: bit order = value order
        const unsigned mmax = __reduce_max_sync(0xffffffffu, mb);
        const unsigned tmin = __reduce_min_sync(0xffffffffu, (best.m2 >= 0.f && mb == mmax) ? (unsigned)best.tau : 0xffffffffu);
        PeakF* rd = red + (qt & 1) * kTcsEpiWarps;
        if (lane == 0) rd[warp - kTcsFirstEpi].tau = -1;
        __syncwarp();
        if (best.m2 >= 0.f && mb == mmax && (unsigned)best.tau == tmin) rd[warp - kTcsFirstEpi] = best;
        const long long t_c = TC_CLOCK();
        // every lag of corr_i is in acc before the next term adds to it; the partials are complete
        named_bar(2, kTcsEpiThreads);
        t_b += TC_CLOCK() - t_c;
        if (te == 0 && lag) {
          PeakF b; b.tau = -1; b.m2 = 0.f; b.re = 0.f; b.im = 0.f;
          for (int w2 = 0; w2 < kTcsEpiWarps; ++w2) {
            const PeakF o = rd[w2];
            if (o.tau >= 0 && (b.tau < 0 || o.m2 > b.m2 || (o.m2 == b.m2 && o.tau < b.tau))) b = o;
          }
          const size_t e = (size_t)row * (p.J + 1) + ti;
          lag[e] = b.tau;
          if (val) val[e] = make_float2(b.re, b.im);
        }
        t_epi += TC_CLOCK() - t_e0;
      }
    }
    if (p.prof && blockIdx.x == 0 && te == 0)
      printf("tcs cta0 epilogue: wait dfull %lld work %lld (barrier %lld)\n", w_df, t_epi, t_b);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace sidwt
