// corr_i8.cu -- integer-family correlation (a5-a7) on the tensor cores, sm_100a.
//
// Reversible integer 5/3 (reading R-INT): bands W_1..W_J, U_J are exact int32 and the
// correlation is the exact integer reduced mod 2^32, so no rounding may
// enter.  Term i (band W at stride g = 2^lg, taps t[k] at support kmin + k, k < n):
//     D[tau] = sum_k conj(t[k]) W[tau + g (kmin + k)]               (a5)
//
// Exact integer GEMM by digits.  Every band value x lies in the static bound of its band
// (interval arithmetic through the integer lifting program from int16 rows: |U_s| <= 2^s 32768,
// |W_s| <= 2^(s-1) 65535), so x = sum_b 256^b d_b with d_b the bytes of its two's complement
// (d_b unsigned for b < D-1, the top digit signed), D = 3 for J <= 8; D = 2 whenever a term's
// staged values all fit in int16 (checked per row and term by the builders).  The template
// coefficients are split into balanced signed digits t = sum_a 256^a t_a.  Each digit product
// d_b t_a is an int8 tensor-core MMA (tcgen05.mma kind::i8) with int32 accumulation -- exact,
// the sums stay far below 2^31 -- and the epilogue forms sum_{a,b} 256^(a+b) acc_{a,b} mod 2^32.
//
// GEMM shape (natural lag order, no Toeplitz matrix of the data is formed):
//   M = 128 rows = 128 lag blocks of 16 consecutive lags (tile of 2048 lags): row c, K byte j
//       reads the digit stream at byte 16 c + j -- a Hankel view of one byte plane of the band
//       (K-major, no swizzle, core matrices of 8 rows x 16 bytes overlapping at a 16-byte row
//       pitch: SBO = 128 B).
//   N = 32 Tn columns = (output component re/im) x (template digit a) x (shift p = 0..15).
//   K: dense terms (g < 16): consecutive 32-byte steps of the stream; B[j][p] = t_k where
//       j - p - sh = g k.  Strided terms (g >= 16): each 16-byte K half holds one tap -- the
//       A descriptor's leading byte offset is g, so the two halves of a K step are the
//       16-byte windows of taps 2ks and 2ks+1 -- and B is diagonal (j mod 16 = p).
//   conj(t) w = (tr wr + ti wi) + i (tr wi - ti wr): the wr stream meets B columns
//   (re: tr, im: -ti), the wi stream (re: ti, im: tr); both accumulate into the same TMEM.
//   Data digit b's MMAs write at TMEM column offset 32 b, so the products of equal weight
//   256^(a+b) land in the same 32-column group: the tensor core forms the digit groups
//   c = a + b itself (D + Tn - 1 groups of [128 lanes][32] int32), TMEM double-buffered by tile.
//
// Eq. (4): one CTA owns a whole row (persistent over rows), terms coarsest
// first; every epilogue thread owns the same 16 lags (one lag block of one 2048-lag tile) for all
// terms, so the running corr_i = corr_{i+1} + D_i lives in its registers; each corr_i goes
// straight to HBM (128 contiguous bytes per thread) and the row's peak per scale (a7) is reduced
// in the epilogue -- no partials, no finalize kernel.
//
// Roles (512 threads, whole warpgroups so that setmaxnreg can move registers to the epilogue):
// warp 0 bulk-copy loader (band segments of both components, B images); warps 1, 2 MMA issuers
// (whole warp, one elected lane issues; one tile each); warp 3 idle; warps 4-7 builders (int32
// band segment -> byte-digit planes, range flag); warps 8-15 epilogue, one per TMEM lane quarter
// (warp % 4) and tile (the row's two tiles in parallel), a thread takes all 16 shifts of its lag
// block; corr leaves through swizzled staging and one 4 KB TMA store per warp and term.
#define SIDWT_NO_KERNELS
#include "kernels.cuh"
#include "corr_tc.cuh"
#include "corr_i8.h"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace sidwt {

// epilogue: one warp per TMEM lane quarter and tile; a thread owns a whole lag block (16 lags) of
// its tile, so the per-tile fixed work (waits, fence, TMA issue) is paid once per 16 lags; the two
// tiles of a row are taken by two groups of four warps in parallel (measured before the epilogue
// had its own register budget: two warps per quarter with 8 lags each, both tiles in sequence)
constexpr int kI8HW = 1, kI8PL = 16 / kI8HW;
constexpr int kI8TileGroups = 2;                   // tiles of a row handled in parallel (ntiles <= 2)
// roles by warpgroup (setmaxnreg moves registers between warpgroups): warps 0-3 loader, two MMA
// issuers and one idle warp; warps 4-7 builders; warps 8-15 epilogue
constexpr int kI8FirstBuild = 4, kI8BuildWarps = 4, kI8FirstEpi = 8, kI8EpiWarps = 4 * kI8TileGroups;
constexpr int kI8Mma2 = 2;                               // second MMA-issuing warp
constexpr int kI8Warps = kI8FirstEpi + kI8EpiWarps;
constexpr int kI8RegsCtl = 56, kI8RegsBuild = 72, kI8RegsEpi = 192;   // per thread, after setmaxnreg
static_assert(kI8FirstBuild % 4 == 0 && kI8FirstEpi % 4 == 0 && kI8Warps % 4 == 0, "roles are whole warpgroups");
static_assert(kI8FirstBuild * kI8RegsCtl + kI8BuildWarps * kI8RegsBuild + kI8EpiWarps * kI8RegsEpi <= 2048,
              "register budget: 64 K registers per SM");
constexpr int kI8Threads = 32 * kI8Warps;
constexpr int kI8BuildThreads = 32 * kI8BuildWarps;
// TMEM: 512 columns, two accumulator buffers of 256 (tile t+1's MMAs overlap tile t's epilogue)
// when dmax * ncol <= 256, else one buffer of 512
constexpr int kI8TmemCols = 512;

struct I8Smem { size_t red, cand, cmeta, wscr, stg, band, stream, img, total; };
constexpr int kI8RowBytes = 8 * kI8PL;             // one lane's corr slice: kI8PL lags x 8 B (32, 64 or 128: TMA swizzle span)
constexpr int kI8StgBytes = 32 * kI8RowBytes;       // per epilogue warp and buffer: 32 lag blocks
__host__ __device__ inline I8Smem i8_layout(const I8Params& p) {
  I8Smem L;
  const size_t nterms = (size_t)p.J + 1;
  L.red = 1024;                                                         // [2 rows][J+1][kI8EpiWarps] warp peak candidates
  L.cand = L.red + 2 * nterms * kI8EpiWarps * 24;                       // [2 rows][J+1][16 lags] int2: the key holder's corr values
  L.cmeta = L.cand + 2 * nterms * 16 * 8;                               // [2 rows][J+1] (taken, first lag)
  L.wscr = (L.cmeta + 2 * nterms * 8 + 15) & ~(size_t)15;               // [kI8EpiWarps][16 lags] int2: scratch of the rare tie path
  L.stg = (L.wscr + (size_t)kI8EpiWarps * 16 * 8 + 1023) & ~(size_t)1023;   // swizzled TMA staging
  L.band = L.stg + (size_t)kI8EpiWarps * kI8StgBytes;
  L.stream = (L.band + (size_t)p.nband * 2 * p.seg_alloc * 4 + 127) & ~(size_t)127;
  L.img = L.stream + (size_t)p.nstream * 2 * p.dmax * p.plane;
  L.total = L.img + (size_t)p.nimg * p.img_alloc;
  return L;
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t saddr, int x0, int x1, int x2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\n"
               :: "l"(map), "r"(saddr), "r"(x0), "r"(x1), "r"(x2) : "memory");
}
__device__ __forceinline__ void bulk_wait_read_le1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }

// D[tmem] (+)= A[smem] . B[smem], kind::i8 (int8 inputs, int32 accumulate)
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n" : "=r"(pred));
  return pred != 0;
}

// 32 lanes x 8 consecutive 32-bit columns -> 8 registers per thread (no wait); the wait for all
// of a thread's outstanding loads is tmem_wait_ld_all (memory clobber orders the uses)
__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld_all() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// NC consecutive accumulator columns (NC a multiple of 4): x8 pieces, then an x4 tail
template <int NC>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[NC]) {
#pragma unroll
  for (int o = 0; o + 8 <= NC; o += 8) {
    uint32_t* x = r + o;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7])
                 : "r"(taddr + o) : "memory");
  }
  if constexpr (NC % 8 == 4) {
    uint32_t* x = r + NC - 4;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "r"(taddr + NC - 4) : "memory");
  }
}
template <int NR>
__device__ __forceinline__ void tie_regs(uint32_t (&r)[NR]) {   // uses of r are ordered after the preceding wait
#pragma unroll
  for (int i = 0; i < NR; ++i) asm volatile("" : "+r"(r[i]));
}

// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread (no wait)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld16(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :: "memory");
}

// B operand images: for each processing step, K step ks, data component x (0: wr, 1: wi), an
// [ncol][32 bytes] K-major no-swizzle block, element (n, j) at (n/8)*256 + (j/16)*128 + (n%8)*16
// + j%16; column n = 32 a + 16 (p / 8) + 8 oc + p % 8 holds digit a of the coefficient that multiplies
// the x stream for output component oc at shift p.  One thread per (step, ks, x, n).
__global__ void k_i8_images(const int2* __restrict__ taps, I8Params p, const int* toff_by_term, int total,
                            unsigned char* __restrict__ img) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= total) return;
  const int n = gid % p.ncol;
  int rest = gid / p.ncol;
  const int x = rest & 1;
  rest >>= 1;                                         // global K-step index
  int step = 0, base = 0;
  while (step <= p.J && rest >= base + p.term[step].ksteps) { base += p.term[step].ksteps; ++step; }
  const I8Term tm = p.term[step];
  const int ks = rest - base;
  const int ti = p.J - step;
  const int a = n / 32, oc = (n / 8) & 1, pp = 8 * ((n / 16) & 1) + (n % 8);
  const int g = 1 << tm.lg;
  unsigned char* blk = img + tm.img_ofs + (size_t)(ks * 2 + x) * p.ncol * 32;
  for (int j = 0; j < 32; ++j) {
    int k = -1;
    if (tm.strided) {
      if ((j & 15) == pp) k = 2 * ks + (j >> 4);
    } else {
      const int d = 32 * ks + j - pp - tm.sh;
      if (d >= 0 && d % g == 0) k = d / g;
    }
    int dig = 0;
    if (k >= 0 && k < tm.ntap) {
      const int2 t = taps[toff_by_term[ti] + k];
      // conj(t) w: wr meets (re: tr, im: -ti), wi meets (re: ti, im: tr)
      int v = (x == 0) ? (oc == 0 ? t.x : -t.y) : (oc == 0 ? t.y : t.x);
      for (int q = 0; q <= a; ++q) {                   // balanced base-256 digit a
        dig = ((v + 128) & 255) - 128;
        v = (v - dig) >> 8;
      }
    }
    blk[(n >> 3) * 256 + (j >> 4) * 128 + (n & 7) * 16 + (j & 15)] = (unsigned char)(signed char)dig;
  }
}

// The MMAs of one 2048-lag tile: for data component x and K step ks, data digit b's products go
// to TMEM column offset 32 b (equal-weight digit products sum in the same 32-column group); at
// the first K step the group a digit reaches first (c = b + TN - 1) starts fresh.  A signedness:
// the top digit signed, the others unsigned.  D (digits in use) is a template parameter so the
// issue sequence is straight-line.
template <int TN, int D>
__device__ __forceinline__ void i8_issue_tile(uint32_t dt, uint64_t a_t, uint64_t bdesc0, uint32_t idesc0, int ksteps,
                                              int kadv16, uint32_t xstride16, uint32_t plane16) {
  constexpr uint32_t kNsplit = ((uint32_t)(32 * (TN > 1 ? TN - 1 : 1)) >> 3) << 17;
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    uint64_t ad = a_t + (uint64_t)(x * xstride16);
    uint64_t bd = bdesc0 + (uint64_t)(x * 64 * TN);
    for (int ks = 0; ks < ksteps; ++ks, ad += (uint64_t)kadv16, bd += (uint64_t)(128 * TN)) {
      const bool first = (x | ks) == 0;
#pragma unroll
      for (int b = 0; b < D; ++b) {
        const uint32_t idb = idesc0 | (b == D - 1 ? (1u << 7) : 0u);
        if (b > 0 && TN > 1 && first) {
          umma_i8(dt + 32 * b, ad + b * plane16, bd, (idb & ~(0x3Fu << 17)) | kNsplit, 1u);
          umma_i8(dt + 32 * (b + TN - 1), ad + b * plane16, bd + (uint64_t)(64 * (TN - 1)),
                  (idb & ~(0x3Fu << 17)) | (4u << 17), 0u);
        } else {
          umma_i8(dt + 32 * b, ad + b * plane16, bd, idb, first ? 0u : 1u);
        }
      }
    }
  }
}

template <int TN>
__global__ void __launch_bounds__(kI8Threads, 1)
k_correlate_i8(const int* __restrict__ bands, const unsigned char* __restrict__ img, int2* __restrict__ corr,
               int32_t* __restrict__ lag, int2* __restrict__ val, const __grid_constant__ I8Params p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const I8Smem L = i8_layout(p);
  const int NB = p.nband, NS = p.nstream, NI = p.nimg;
  uint64_t* bandfull = reinterpret_cast<uint64_t*>(smem_raw);        // [NB]
  uint64_t* bandempty = bandfull + 4;                                 // [NB]
  uint64_t* sfull = bandempty + 4;                                    // [NS]
  uint64_t* sempty = sfull + 4;                                       // [NS]
  uint64_t* imgfull = sempty + 4;                                     // [NI]
  uint64_t* imgempty = imgfull + 4;                                   // [NI]
  uint64_t* dfull = imgempty + 4;                                     // [2]
  uint64_t* dempty = dfull + 2;                                       // [2]
  uint64_t* hkey = dempty + 2;                                        // peak keys of a term posted (one arrival per epilogue warp)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem_raw + 256);
  int* dcnt = reinterpret_cast<int*>(smem_raw + 264);                 // [2] digits used per TMEM buffer
  int* sflag = reinterpret_cast<int*>(smem_raw + 288);                // [4 stages][4 builder warps]
  unsigned* hkeys = reinterpret_cast<unsigned*>(smem_raw + 384);      // [2 terms][kI8EpiWarps] warp maxima of the peak keys
  PeakI* red = reinterpret_cast<PeakI*>(smem_raw + L.red);            // [2][J+1][kI8EpiWarps]
  int2* cand = reinterpret_cast<int2*>(smem_raw + L.cand);            // [2][J+1][16]
  int* cmeta = reinterpret_cast<int*>(smem_raw + L.cmeta);            // [2][J+1][2]
  int2* wscr = reinterpret_cast<int2*>(smem_raw + L.wscr);            // [kI8EpiWarps][16]
  unsigned char* stg = smem_raw + L.stg;                              // [kI8EpiWarps][kI8StgBytes]
  int* band = reinterpret_cast<int*>(smem_raw + L.band);
  unsigned char* stream = smem_raw + L.stream;
  unsigned char* imgs = smem_raw + L.img;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nterms = p.J + 1;
  constexpr int NCOL = 32 * TN;

  // accumulator span: digit-weight groups c = a + b = 0 .. dmax + TN - 2, 32 columns each
  const int NBUF = (p.dmax + TN - 1) * 32 <= kI8TmemCols / 2 ? 2 : 1;
  const uint32_t bufcols = kI8TmemCols / NBUF;
  // two MMA-issuing warps (one tile each) when a row has two tiles and TMEM is double-buffered
  const int nmma = (p.ntiles >= 2 && NBUF == 2) ? 2 : 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) { mbar_init(&bandfull[i], 1); mbar_init(&bandempty[i], kI8BuildThreads); }
    for (int i = 0; i < NS; ++i) { mbar_init(&sfull[i], kI8BuildThreads); mbar_init(&sempty[i], nmma); }
    for (int i = 0; i < NI; ++i) { mbar_init(&imgfull[i], 1); mbar_init(&imgempty[i], nmma); }
    for (int i = 0; i < 2; ++i) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], 32 * 4); }
    mbar_init(hkey, kI8EpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = threadIdx.x; i < 4 * nterms; i += blockDim.x) cmeta[i] = 0;
  if (warp == 1) tmem_alloc(tslot, kI8TmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  // register budget by role (one setmaxnreg per warpgroup, inside the role's branch so that the
  // allocation of that branch follows it): the epilogue keeps both tiles' running sums, the
  // accumulator groups and its addresses in registers; loader / MMA / builder warps need few
  if (warp < kI8FirstBuild) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" :: "n"(kI8RegsCtl));
  if (warp == 0) {
    // ---------------- loader: band segments (both components) and the term's B images
    if (lane == 0) {
      uint32_t u = 0;
      for (long long row = blockIdx.x; row < p.rows; row += gridDim.x)
        for (int step = 0; step < nterms; ++step, ++u) {
          const I8Term& tm = p.term[step];
          const uint32_t bs = u % NB, is = u % NI;
          mbar_wait(&bandempty[bs], ((u / NB) & 1) ^ 1);
          const uint32_t bytes = (uint32_t)tm.seg_len * 4u;
          mbar_expect_tx(&bandfull[bs], 2 * bytes);
          const int* src = bands + ((size_t)row * nterms + tm.band) * 2 * p.stride + tm.seg_a4;
          int* dst = band + (size_t)bs * 2 * p.seg_alloc;
          bulk_load_g2s(dst, src, bytes, &bandfull[bs]);
          bulk_load_g2s(dst + p.seg_alloc, src + p.stride, bytes, &bandfull[bs]);
          mbar_wait(&imgempty[is], ((u / NI) & 1) ^ 1);
          const uint32_t ib = (uint32_t)tm.ksteps * 2 * NCOL * 32;
          mbar_expect_tx(&imgfull[is], ib);
          bulk_load_g2s(imgs + (size_t)is * p.img_alloc, img + tm.img_ofs, ib, &imgfull[is]);
        }
    }
  } else if (warp == 1 || warp == kI8Mma2) {
    // ---------------- MMA issuers: two warps, warp k issues the MMAs of tiles t = k (mod 2) (one
    // tile per warp for N = 4096), so the two tiles' issue latencies overlap.  The whole warp runs
    // the loop (uniform values in uniform registers); one elected lane issues MMAs and commits.
    const int mw = warp == 1 ? 0 : 1;
    const uint32_t idesc0 = (2u << 4) | (1u << 10) | ((uint32_t)(NCOL >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t st0 = smem_u32(stream), im0 = smem_u32(imgs);
    const uint32_t plane16 = (uint32_t)p.plane >> 4;
    uint32_t u = 0, q = 0;
    for (long long row = blockIdx.x; row < p.rows; row += gridDim.x)
      for (int step = 0; step < nterms; ++step, ++u) {
        const int ksteps = p.term[step].ksteps, kadv16 = p.term[step].kadv >> 4, dig = p.term[step].dig;
        const uint32_t ss = u % NS, is = u % NI;
        if (mw >= nmma) continue;                                          // single issuer: the second warp idles
        mbar_wait(&sfull[ss], (u / NS) & 1);
        mbar_wait(&imgfull[is], (u / NI) & 1);
        tc_fence_after();
        bool fits = true;
        for (int w = 0; w < kI8BuildWarps; ++w) fits = fits && sflag[ss * 4 + w] != 0;
        const int D = (fits && dig > 2) ? 2 : dig;
        const uint64_t bdesc0 = smem_desc(im0 + is * p.img_alloc, 128, 256);
        const uint64_t adesc0 = smem_desc(st0 + ss * 2 * p.dmax * p.plane, (uint32_t)p.term[step].lbo, 128);
        for (int t = 0; t < p.ntiles; ++t, ++q) {
          if (t % nmma != mw) continue;
          const uint32_t buf = q % NBUF;
          mbar_wait(&dempty[buf], ((q / NBUF) & 1) ^ 1);
          tc_fence_after();
          if (lane == 0) dcnt[buf] = D;
          __syncwarp();
          const uint32_t dt = tmem + buf * bufcols;
          if (elect_one()) {
            const uint64_t a_t = adesc0 + (uint64_t)(128 * t);
            switch (D) {
              case 2: i8_issue_tile<TN, 2>(dt, a_t, bdesc0, idesc0, ksteps, kadv16, p.dmax * plane16, plane16); break;
              case 3: i8_issue_tile<TN, 3>(dt, a_t, bdesc0, idesc0, ksteps, kadv16, p.dmax * plane16, plane16); break;
              default: i8_issue_tile<TN, 4>(dt, a_t, bdesc0, idesc0, ksteps, kadv16, p.dmax * plane16, plane16); break;
            }
            umma_commit(&dfull[buf]);
          }
          __syncwarp();
        }
        if (elect_one()) {
          umma_commit(&sempty[ss]);
          umma_commit(&imgempty[is]);
        }
        __syncwarp();
      }
  }
  } else if (warp < kI8FirstEpi) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" :: "n"(kI8RegsBuild));
    // ---------------- builders: int32 band segment -> byte-digit planes (natural order)
    const int tb = threadIdx.x - 32 * kI8FirstBuild;
    uint32_t u = 0;
    for (long long row = blockIdx.x; row < p.rows; row += gridDim.x)
      for (int step = 0; step < nterms; ++step, ++u) {
        const I8Term& tm = p.term[step];
        const uint32_t bs = u % NB, ss = u % NS;
        mbar_wait(&bandfull[bs], (u / NB) & 1);
        mbar_wait(&sempty[ss], ((u / NS) & 1) ^ 1);
        const int nd = tm.dig;
        const int n4 = tm.seg_len >> 2;
        unsigned range = 0;
        // pass 1: digit planes 0 and 1 and the range of the staged values (4 loads in flight)
        for (int x = 0; x < 2; ++x) {
          const int4* __restrict__ src = reinterpret_cast<const int4*>(band + ((size_t)bs * 2 + x) * p.seg_alloc);
          unsigned* __restrict__ d0 = reinterpret_cast<unsigned*>(stream + ((size_t)ss * 2 + x) * p.dmax * p.plane);
          unsigned* __restrict__ d1 = d0 + p.plane / 4;
          for (int i0 = tb; i0 < n4; i0 += 4 * kI8BuildThreads) {
            int4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int i = i0 + k * kI8BuildThreads;
              v[k] = i < n4 ? src[i] : make_int4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int i = i0 + k * kI8BuildThreads;
              range |= ((unsigned)v[k].x + 32768u) | ((unsigned)v[k].y + 32768u) | ((unsigned)v[k].z + 32768u) |
                       ((unsigned)v[k].w + 32768u);
              const unsigned p01 = __byte_perm(v[k].x, v[k].y, 0x5140), p23 = __byte_perm(v[k].z, v[k].w, 0x5140);
              if (i < n4) {
                d0[i] = __byte_perm(p01, p23, 0x5410);
                d1[i] = __byte_perm(p01, p23, 0x7632);
              }
            }
          }
        }
        // every staged value in [-32768, 32767]: two digits suffice for this (row, term)
        const unsigned any_big = __any_sync(0xffffffffu, (range >> 16) != 0u);
        if (lane == 0) sflag[ss * 4 + (warp - kI8FirstBuild)] = any_big ? 0 : 1;
        if (nd > 2) {
          named_bar(3, kI8BuildThreads);
          bool big = false;
          for (int w = 0; w < kI8BuildWarps; ++w) big = big || sflag[ss * 4 + w] == 0;
          // pass 2 (rare): the digit planes >= 2 for the MMA's three- or four-digit products
          if (big)
            for (int x = 0; x < 2; ++x) {
              const int4* __restrict__ src = reinterpret_cast<const int4*>(band + ((size_t)bs * 2 + x) * p.seg_alloc);
              unsigned* __restrict__ d2 = reinterpret_cast<unsigned*>(stream + ((size_t)ss * 2 + x) * p.dmax * p.plane) +
                                          2 * (p.plane / 4);
              for (int i = tb; i < n4; i += kI8BuildThreads) {
                const int4 v = src[i];
                const unsigned q01 = __byte_perm(v.x, v.y, 0x7362), q23 = __byte_perm(v.z, v.w, 0x7362);
                d2[i] = __byte_perm(q01, q23, 0x5410);
                if (nd > 3) d2[i + p.plane / 4] = __byte_perm(q01, q23, 0x7632);
              }
            }
        }
        fence_proxy_async_smem();                   // digit planes -> visible to the tensor core
        mbar_arrive(&sfull[ss]);
        mbar_arrive(&bandempty[bs]);
      }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" :: "n"(kI8RegsEpi));
    // ---------------- epilogue: TMEM -> digits recombined -> eq. (4) running sums -> corr, peaks.
    // Warp (quarter, tg): TMEM lanes 32 quarter .. +31 of tile tg; lane = one lag block, all 16
    // shifts: accumulator columns 32 c + 16 half + 8 oc + i of digit-weight group c.
    //
    // Peak search (a7) in two stages.  Stage 1, every lag: the high word of the exact 64-bit
    // |corr|^2 is a monotone key (m1 >= m2 => hi(m1) >= hi(m2)), so the row's maximum lies among
    // the lags whose key equals the largest key; each thread keeps the largest key of its 16 lags
    // (a max tree, no index tracking), the warp maximum is posted to shared memory and hkey (an
    // mbarrier, one arrival per epilogue warp and term) is signalled.  Stage 2, once the term's
    // eight warp keys are posted: the first thread of the first warp holding the largest key copies
    // its 16 running sums (corr_ti at its lags) to the term's candidate slot -- they still hold
    // corr_ti because stage 2 runs before the next term's D is added (after its accumulator loads,
    // which hides the wait) -- and the exact comparison (64-bit |.|^2, smallest lag among ties)
    // over those 16 lags is done once per row in the final combine.  Further threads with the
    // same key (rare: equal high words) are compared exactly in their warp (16 lanes per holder)
    // and post a warp candidate; every other warp posts an empty one.
    constexpr int PL = kI8PL;
    const int te = threadIdx.x - 32 * kI8FirstEpi;
    const int we = warp - kI8FirstEpi;
    const int quarter = warp & 3, tg = we >> 2;
    const int c = 32 * quarter + lane;                                  // TMEM lane = lag block of the tile
    const int N = p.N, ntiles = p.ntiles;
    const bool want_corr = p.want_corr != 0, tma = p.tma_store != 0;
    const bool mine = tg < ntiles;                                      // this warp's tile exists
    const int tauA = 2048 * tg + 16 * c;                                // this thread's first lag
    const bool valid = mine && tauA < N;                                // N % 16 == 0: a block is all in or all out
    // staging addresses, computed once and kept in registers (opaque to rematerialisation)
    constexpr int CH = kI8RowBytes / 16;                                // 16-byte chunks per row
    uint32_t sb_base = smem_u32(stg + (size_t)we * kI8StgBytes), stg_row = sb_base + kI8RowBytes * lane, stg_off[CH];
    {
      const int sw = ((lane * kI8RowBytes) >> 7) & (CH - 1);
#pragma unroll
      for (int k = 0; k < CH; ++k) { stg_off[k] = 16 * (k ^ sw); asm volatile("" : "+r"(stg_off[k])); }
      asm volatile("" : "+r"(sb_base));
      asm volatile("" : "+r"(stg_row));
    }
    uint32_t q = (uint32_t)tg, hn = 0;                                  // q: this warp's tile in the MMA order
    int par = 0;
    for (long long row = blockIdx.x; row < p.rows; row += gridDim.x) {
      // running corr (mod 2^32) of the thread's 16 lags, interleaved (re, im): the staging stores
      // take four consecutive registers
      unsigned run[2 * PL];
#pragma unroll
      for (int i = 0; i < 2 * PL; ++i) run[i] = 0u;
      unsigned wh_prev = 0, hm_prev = 0;                                // warp / thread key of the previous term
      PeakI* rrow = red + (size_t)par * nterms * kI8EpiWarps;
      const int rowblk = (int)row * nterms * (N >> 4);                  // first lag block of the row's corr
      auto dump16 = [&](int2* dst) {                                    // this thread's corr_ti at its 16 lags
        int4* cs = reinterpret_cast<int4*>(dst);
#pragma unroll
        for (int k = 0; k < PL / 2; ++k)
          cs[k] = make_int4((int)run[4 * k], (int)run[4 * k + 1], (int)run[4 * k + 2], (int)run[4 * k + 3]);
      };
      // stage 2 for term tip (the term posted last: phase hn - 1 of hkey)
      auto resolve = [&](int tip) {
        mbar_wait(hkey, (hn - 1) & 1);
        // the term's largest key; the first warp holding it fills the candidate slot
        const uint4* hp = reinterpret_cast<const uint4*>(hkeys + kI8EpiWarps * ((hn - 1) & 1));
        const uint4 ka = hp[0], kb = hp[1];
        const unsigned kk[8] = {ka.x, ka.y, ka.z, ka.w, kb.x, kb.y, kb.z, kb.w};
        const unsigned gmax = max(max(max(ka.x, ka.y), max(ka.z, ka.w)), max(max(kb.x, kb.y), max(kb.z, kb.w)));
        PeakI* rp = rrow + (size_t)tip * kI8EpiWarps + we;
        bool posted = false;
        if (wh_prev == gmax) {
          unsigned bal = __ballot_sync(0xffffffffu, hm_prev == gmax);   // non-zero: the warp key is some lane's key
          bool lower = false;                                           // a lower-numbered warp holds the same key
#pragma unroll
          for (int w = 0; w < kI8EpiWarps - 1; ++w) lower = lower || (w < we && kk[w] == gmax);
          if (!lower) {
            // the term's key holder: first such lane of the first such warp fills the candidate slot
            const int src = __ffs(bal) - 1;
            bal &= bal - 1;
            if (lane == src) {
              const int slot = par * nterms + tip;
              dump16(cand + (size_t)slot * 16);
              cmeta[2 * slot + 1] = tauA;
              cmeta[2 * slot] = 1;
            }
          }
          if (bal) {
            // rare (equal high words): the other holders' lags, exact, 16 lanes per holder
            PeakI wb;
            wb.m2 = 0; wb.tau = -1; wb.re = 0; wb.im = 0; wb.pad = 0;
            int2* ws = wscr + we * 16;
            while (bal) {
              const int src = __ffs(bal) - 1;
              bal &= bal - 1;
              if (lane == src) dump16(ws);
              __syncwarp();
              const int tau = 2048 * tg + 16 * (32 * quarter + src) + lane;
              const bool ok = lane < PL && tau < N && mine;
              const int2 v = ok ? ws[lane] : make_int2(0, 0);
              const unsigned long long m = mag2i(v.x, v.y);
              const unsigned hi = ok ? (unsigned)(m >> 32) : 0u, lo = ok ? (unsigned)m : 0u;
              const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
              const unsigned mlo = __reduce_max_sync(0xffffffffu, (ok && hi == mhi) ? lo : 0u);
              const unsigned cnd = (ok && hi == mhi && lo == mlo) ? (unsigned)tau : 0xffffffffu;
              const unsigned tmin = __reduce_min_sync(0xffffffffu, cnd);
              if (tmin != 0xffffffffu) {
                const unsigned long long mm = ((unsigned long long)mhi << 32) | mlo;
                if (wb.tau < 0 || beats(mm, (int)tmin, wb.m2, wb.tau)) {
                  const int wl = __ffs(__ballot_sync(0xffffffffu, cnd == tmin)) - 1;
                  wb.m2 = mm; wb.tau = (int)tmin;
                  wb.re = __shfl_sync(0xffffffffu, v.x, wl);
                  wb.im = __shfl_sync(0xffffffffu, v.y, wl);
                }
              }
              __syncwarp();
            }
            if (lane == 0) *rp = wb;
            posted = true;
          }
        }
        if (!posted && lane == 0) {
          PeakI e; e.m2 = 0; e.tau = -1; e.re = 0; e.im = 0; e.pad = 0;
          *rp = e;
        }
      };
      for (int step = 0; step < nterms; ++step) {
        const int ti = p.J - step;
        unsigned hmax = 0;                                              // stage 1: largest key of this thread's lags
        unsigned re[PL], im[PL];
        if (mine) {
          // this warp's tile: D_ti (digits recombined mod 2^32)
          const uint32_t buf = q % NBUF;
          // a single TMEM buffer alternates between the two tile groups: pass the other group's phase first
          if (NBUF == 1 && ntiles > 1 && q > 0) mbar_wait(&dfull[0], (q - 1) & 1);
          mbar_wait(&dfull[buf], (q / NBUF) & 1);
          tc_fence_after();
          const int D = dcnt[buf];
          const uint32_t tb0 = tmem + ((uint32_t)(32 * quarter) << 16) + buf * bufcols;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            // digit-weight group c, half hf at columns 32 c + 16 hf + [oc 8 + i]: one x16 load per group;
            // groups 0, 1 always exist (D >= 2), group 2 whenever TN >= 2
            uint32_t g0[16], g1[16], g2[16];
            tmem_ld_cols<16>(tb0 + 16 * hf, g0);
            tmem_ld_cols<16>(tb0 + 16 * hf + 32, g1);
            if constexpr (TN >= 2) tmem_ld_cols<16>(tb0 + 16 * hf + 64, g2);
            tmem_wait_ld_all();
            tie_regs(g0); tie_regs(g1);
            if constexpr (TN >= 2) tie_regs(g2);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              re[8 * hf + i] = g0[i] + (g1[i] << 8);
              im[8 * hf + i] = g0[8 + i] + (g1[8 + i] << 8);
              if constexpr (TN >= 2) { re[8 * hf + i] += g2[i] << 16; im[8 * hf + i] += g2[8 + i] << 16; }
            }
          }
          for (int cq = TN >= 2 ? 3 : 2; cq < D + TN - 1; ++cq) {      // rare: higher digit-weight groups
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              uint32_t g[16];
              tmem_ld_cols<16>(tb0 + 16 * hf + 32 * cq, g);
              tmem_wait_ld_all();
              tie_regs(g);
#pragma unroll
              for (int i = 0; i < 8; ++i) { re[8 * hf + i] += g[i] << (8 * cq); im[8 * hf + i] += g[8 + i] << (8 * cq); }
            }
          }
          tc_fence_before();
          mbar_arrive(&dempty[buf]);
          q += (uint32_t)ntiles;
        }
        // the previous term's stage 2 reads the running sums before this term is added
        if (step > 0) resolve(ti + 1);
        if (mine) {
#pragma unroll
          for (int i = 0; i < PL; ++i) {
            if (step == 0) { run[2 * i] = re[i]; run[2 * i + 1] = im[i]; }
            else { run[2 * i] += re[i]; run[2 * i + 1] += im[i]; }
          }
          if (want_corr && !tma && valid) {
            int4* dst = reinterpret_cast<int4*>(corr + ((size_t)row * nterms + ti) * N + tauA);
#pragma unroll
            for (int i = 0; i < PL / 2; ++i)
              dst[i] = make_int4((int)run[4 * i], (int)run[4 * i + 1], (int)run[4 * i + 2], (int)run[4 * i + 3]);
          }
          if (want_corr && tma) {
            // corr_ti of this warp's 32 lag blocks (4 KB contiguous in HBM) -> swizzled staging (the
            // TMA map's swizzle span = one lane's row) -> one TMA tensor store; the previous term's
            // store must have read the staging buffer
            if (lane == 0) bulk_wait_read_all();
            __syncwarp();
#pragma unroll
            for (int k = 0; k < CH; ++k)
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n"
                           :: "r"(stg_row + stg_off[k]), "r"(run[4 * k]), "r"(run[4 * k + 1]), "r"(run[4 * k + 2]), "r"(run[4 * k + 3])
                           : "memory");
          }
          if (valid) {
            // stage 1: keys of this tile's lags (max tree); independent work under the staging stores
            unsigned k16[PL];
#pragma unroll
            for (int i = 0; i < PL; ++i) k16[i] = (unsigned)(mag2i((int)run[2 * i], (int)run[2 * i + 1]) >> 32);
#pragma unroll
            for (int w = PL / 2; w >= 1; w >>= 1)
#pragma unroll
              for (int i = 0; i < w; ++i) k16[i] = max(k16[i], k16[i + w]);
            hmax = k16[0];
          }
          if (want_corr && tma) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && 2048 * tg + 512 * quarter < N) {   // N % 512 == 0: a warp's 32 blocks all in or all out
              // lag-block coordinate of (row, ti, tile, quarter); the tensor's block count fits 32 bits
              const int blk = (rowblk + ti * (N >> 4)) + 128 * tg + 32 * quarter;
              tma_store_3d(&p.cmap, sb_base, 0, 0, blk);
              bulk_commit();
            }
          }
        }
        // post this warp's key for the term
        const unsigned wh = __reduce_max_sync(0xffffffffu, hmax);
        if (lane == 0) {
          hkeys[kI8EpiWarps * (hn & 1) + we] = wh;
          mbar_arrive(hkey);
        }
        ++hn;
        wh_prev = wh;
        hm_prev = valid ? hmax : 0xffffffffu;                           // a thread without lags never holds the key
        if (step == nterms - 1) resolve(ti);                            // the row's last term: no later tile hides the wait
      }
      // every scale of the row: combine the candidates (one barrier per row)
      named_bar(2, 32 * kI8EpiWarps);
      // 16 lanes per term: lane j takes the key holder's lag j (exact |.|^2) and, for j < 8, warp j's
      // tie candidate; half-warp argmax (largest |.|^2, smallest lag among ties)
      for (int tt = te >> 4; tt < nterms; tt += 2 * kI8EpiWarps) {
        const int j = lane & 15;
        const unsigned hmask = 0xffffu << (lane & 16);
        unsigned long long m = 0;
        int tau = -1, vre = 0, vim = 0;
        int* cm = cmeta + 2 * (par * nterms + tt);
        if (cm[0]) {
          const int tj = cm[1] + j;
          if (tj < N) {
            const int2 v = cand[(size_t)(par * nterms + tt) * 16 + j];
            m = mag2i(v.x, v.y); tau = tj; vre = v.x; vim = v.y;
          }
        }
        if (j < kI8EpiWarps) {
          const PeakI o = rrow[(size_t)tt * kI8EpiWarps + j];
          if (o.tau >= 0 && (tau < 0 || beats(o.m2, o.tau, m, tau))) { m = o.m2; tau = o.tau; vre = o.re; vim = o.im; }
        }
        const bool ok = tau >= 0;
        const unsigned hi = ok ? (unsigned)(m >> 32) : 0u, lo = ok ? (unsigned)m : 0u;
        const unsigned mhi = __reduce_max_sync(hmask, hi);
        const unsigned mlo = __reduce_max_sync(hmask, (ok && hi == mhi) ? lo : 0u);
        const unsigned cnd = (ok && hi == mhi && lo == mlo) ? (unsigned)tau : 0xffffffffu;
        const unsigned tmin = __reduce_min_sync(hmask, cnd);
        __syncwarp(hmask);
        if (j == 0) cm[0] = 0;
        if (lag && ((ok && (unsigned)tau == tmin) || (j == 0 && tmin == 0xffffffffu))) {
          const size_t e = (size_t)row * nterms + tt;
          lag[e] = tmin == 0xffffffffu ? -1 : tau;
          if (val) val[e] = tmin == 0xffffffffu ? make_int2(0, 0) : make_int2(vre, vim);
        }
      }
      par ^= 1;
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kI8TmemCols);
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static int digits_for(long long lo, long long hi) {
  for (int d = 1; d <= 4; ++d) {
    const long long lim = 1LL << (8 * d - 1);
    if (lo >= -lim && hi <= lim - 1) return d;
  }
  return 5;
}

bool i8_configure(I8Params& p, int N, int J, int stride, int ML, const int* kmin, const int* cnt, const int* toff,
                  const int2* taps) {
  p = I8Params{};
  if (N % 16 != 0 || N > 4096 || (ML & 3) != 0 || J + 1 > kI8MaxTerms) return false;
  p.N = N; p.J = J; p.stride = stride; p.ML = ML;
  p.ntiles = (N + 2047) / 2048;
  // template digits (balanced, signed): every coefficient and its negation
  long long tmax = 0;
  for (int i = 0; i <= J; ++i)
    for (int k = 0; k < cnt[i]; ++k) {
      const int2 t = taps[toff[i] + k];
      tmax = std::max<long long>(tmax, std::max<long long>(std::llabs((long long)t.x), std::llabs((long long)t.y)));
    }
  int tn = 1;
  while (tn <= 4 && tmax > 127LL * ((1LL << (8 * tn)) - 1) / 255) ++tn;
  if (tn > 4) return false;
  p.tn = tn; p.ncol = 32 * tn;
  // static bound of each band from int16 rows through the integer dual program (R-INT):
  // e += floor((o_k + o_{k-1}) / 2) -> U_s in [2 lo, 2 hi]; o -= floor((e_k + e_{k+1} + 2) / 4) ->
  // W_s in [lo - hi, hi - lo], (lo, hi) the bound of U_{s-1}
  long long ulo = -32768, uhi = 32767;
  int bdig[kI8MaxTerms];
  for (int s = 1; s <= J; ++s) {
    bdig[s - 1] = digits_for(ulo - uhi, uhi - ulo);
    ulo *= 2; uhi *= 2;
    if (s == J) bdig[J] = digits_for(ulo, uhi);
  }
  int dmax = 2, kwin = 0, seg_alloc = 0, img = 0;
  for (int step = 0; step <= J; ++step) {
    const int ti = J - step;
    I8Term& tm = p.term[step];
    tm.band = ti;
    tm.lg = ti < J ? ti + 1 : J;
    tm.kmin = kmin[ti];
    tm.ntap = cnt[ti];
    tm.dig = std::max(2, bdig[ti]);
    if (tm.dig > 4) return false;
    dmax = std::max(dmax, tm.dig);
    const int g = 1 << tm.lg;
    const int gk = g * tm.kmin;
    tm.strided = g >= 16;
    if (tm.strided) {
      tm.sh = 0;
      tm.P0 = gk;                                            // multiple of 16
      tm.ksteps = (tm.ntap + 1) / 2;
      tm.kadv = 2 * g;
      tm.lbo = g;
      kwin = std::max(kwin, (tm.ksteps - 1) * 2 * g + g + 16);
    } else {
      tm.sh = ((gk + ML) % 4 + 4) % 4;
      tm.P0 = gk - tm.sh;
      tm.ksteps = (16 + g * (tm.ntap - 1) + tm.sh + 31) / 32;
      tm.kadv = 32;
      tm.lbo = 16;
      kwin = std::max(kwin, 32 * tm.ksteps);
    }
    tm.seg_a4 = tm.P0 + ML;
    if (tm.seg_a4 < 0 || (tm.seg_a4 & 3) != 0) return false;
    const long long need = (long long)N + (long long)g * (tm.ntap - 1) + tm.sh + 1;   // stream bytes with nonzero weight
    const long long have = (long long)stride - tm.seg_a4;
    tm.seg_len = (int)((std::min(need, have) + 3) & ~3LL);
    if (tm.seg_len > have) tm.seg_len = (int)(have & ~3LL);
    seg_alloc = std::max(seg_alloc, tm.seg_len);
    tm.img_ofs = img;
    img += tm.ksteps * 2 * p.ncol * 32;
  }
  p.dmax = dmax;
  if ((dmax + tn - 1) * 32 > kI8TmemCols) return false;
  p.seg_alloc = (seg_alloc + 3) & ~3;
  p.plane = (int)((std::max(2048 * p.ntiles - 16 + kwin, seg_alloc) + 127) & ~127);
  int img_alloc = 0;
  for (int step = 0; step <= J; ++step) img_alloc = std::max(img_alloc, p.term[step].ksteps * 2 * p.ncol * 32);
  p.img_alloc = (img_alloc + 127) & ~127;
  // ring depths: as many staged band segments as fit (>= 2), two digit-stream stages (one for
  // deep plans whose planes are long, e.g. J = 10), two B-image stages
  const size_t budget = 227 * 1024;
  for (p.nimg = 2; p.nimg >= 1; --p.nimg)
    for (p.nstream = 2; p.nstream >= 1; --p.nstream)
      for (p.nband = 4; p.nband >= 2; --p.nband)
        if (i8_layout(p).total <= budget) {
          if (std::getenv("SIDWT_I8_VERBOSE")) {
            const I8Smem L = i8_layout(p);
            fprintf(stderr, "[i8] tn %d dmax %d rings: band %d x %d B, stream %d x %d B, img %d x %d B; staging at %zu, total %zu B\n",
                    p.tn, p.dmax, p.nband, 2 * p.seg_alloc * 4, p.nstream, 2 * p.dmax * p.plane, p.nimg, p.img_alloc, L.stg, L.total);
          }
          return true;
        }
  return false;
}

size_t i8_image_bytes(const I8Params& p) {
  size_t b = 0;
  for (int step = 0; step <= p.J; ++step) b += (size_t)p.term[step].ksteps * 2 * p.ncol * 32;
  return b;
}

size_t i8_smem_bytes(const I8Params& p) { return i8_layout(p).total; }

cudaError_t i8_build_images(const I8Params& p, const int2* d_taps, const int* toff, unsigned char* d_img) {
  int total_ks = 0;
  for (int step = 0; step <= p.J; ++step) total_ks += p.term[step].ksteps;
  int* d_toff = nullptr;
  cudaError_t e = cudaMalloc(&d_toff, kI8MaxTerms * sizeof(int));
  if (e == cudaSuccess) e = cudaMemcpy(d_toff, toff, (p.J + 1) * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const int total = total_ks * 2 * p.ncol;
    k_i8_images<<<(total + 127) / 128, 128>>>(d_taps, p, d_toff, total, d_img);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (d_toff) cudaFree(d_toff);
  return e;
}

// corr [rows][J+1][N] int2 as a 3-D TMA tensor of 8-byte elements: [lag blocks of 16][kI8HW parts][kI8PL
// lags]; box = kI8PL lags x 1 part x 32 blocks (one epilogue warp's tile slice), swizzle span = one row
static bool encode_corr_map_i8(CUtensorMap* map, void* corr, long long rows, const I8Params& p) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }
  const cuuint64_t dims[3] = {kI8PL, kI8HW, (cuuint64_t)rows * (p.J + 1) * (p.N / 16)};
  const cuuint64_t strides[2] = {kI8RowBytes, 128};
  const cuuint32_t box[3] = {kI8PL, 1, 32};
  const CUtensorMapSwizzle sw = kI8RowBytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                : (kI8RowBytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, corr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t i8_launch(const I8Params& p0, const int* bands, const unsigned char* img, int2* corr, int32_t* lag,
                      int2* val, int grid, cudaStream_t s) {
  I8Params p = p0;
  p.tma_store = (p.N % 512 == 0) ? 1 : 0;
  if (corr && p.tma_store && !encode_corr_map_i8(&p.cmap, corr, p.rows, p)) return cudaErrorInvalidValue;
  const size_t smem = i8_layout(p).total;
  void (*kern)(const int*, const unsigned char*, int2*, int32_t*, int2*, const I8Params);
  switch (p.tn) {
    case 1: kern = k_correlate_i8<1>; break;
    case 2: kern = k_correlate_i8<2>; break;
    case 3: kern = k_correlate_i8<3>; break;
    default: kern = k_correlate_i8<4>; break;
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kI8Threads, smem, s>>>(bands, img, corr, lag, val, p);
  return cudaGetLastError();
}

}  // namespace sidwt
