// fused.cuh -- SURVEY.md section 8(f) NEXT 1: analyze -> correlate -> peaks in one kernel,
// without the band round trip through HBM.
//
// One CTA per (row, TT-lag tile), single template.  The extended input segment of the tile
// plus the correlation reach and the lifting halo is loaded once (both components); the
// J levels of the SIDWT lifting run on chip exactly as in k_analyze (same level code, so
// the bands are bit-identical); after level s the correlation term of W_s (D_s, eq. (4))
// is computed from the on-chip detail plane with the same register sliding window as
// k_correlate and parked in shared memory, and W_s is overwritten by the next level.  The
// approximation term A_J follows the last level.  The suffix sums corr_s = corr_{s+1} +
// D_{s+1} (same operands and order as k_correlate, hence bit-identical results), the
// corr stores (optional: peaks-only mode) and the per-tile peak partials close the tile.
#pragma once
#include "kernels.cuh"

namespace sidwt {

struct FusParams {
  int N, J, ext, TT, ntiles, fML, halo_l, lbuf, padl, padr, taps_per_t;
  long long rows;
  Lift lift;
  int want_corr, want_peaks;
  Term term[kMaxTerms];                // indexed by term (i < J: W_{i+1}, i = J: U_J)
  uint2 ctap[kCTaps];                  // template taps (one template)
};

// levels LH .. J-1 of both components, each followed by its correlation term
template <int FAM, int RV, int LH, int Q>
__device__ __forceinline__ void fused_levels(const FusParams& p, typename Dual<FAM>::T* U0, typename Dual<FAM>::T* W0,
                                             typename Dual<FAM>::T* U1, typename Dual<FAM>::T* W1,
                                             typename std::conditional<FAM == FI53, int2, float2>::type* D, int tau0);

template <int FAM, int Q>
__device__ __forceinline__ void fused_term(const FusParams& p, int ti, const typename Dual<FAM>::T* P0,
                                           const typename Dual<FAM>::T* P1,
                                           typename std::conditional<FAM == FI53, int2, float2>::type* D, int tau0) {
  constexpr bool INT = FAM == FI53;
  typedef typename std::conditional<INT, int2, float2>::type T2;
  typedef typename std::conditional<INT, unsigned, float>::type A;
  typedef typename Dual<FAM>::T T;
  const Term tm = p.term[ti];
  const int g = 1 << tm.lg;
  const int TT = p.TT;
  const int nq = TT >> tm.lg;
  const int nqb = (nq + Q - 1) / Q;
  // band value of fine-grid position tau0 + g kmin sits at buffer index fML + halo_l + g kmin
  const T* sb = P0 + p.fML + p.halo_l + g * tm.kmin;
  const int plane = (int)(P1 - P0);
  const T2* tp = reinterpret_cast<const T2*>(p.ctap) + tm.toff;
  T2* Dt = D + (size_t)ti * TT;
  for (int w = threadIdx.x; w < g * nqb; w += blockDim.x) {
    const int r = w & (g - 1);
    const int q0 = (w >> tm.lg) * Q;
    A ar[Q], ai[Q];
    corr_item<INT, Q>(sb, plane, tp, tm.ntap, r, tm.lg, q0, ar, ai);
    T2* pn = Dt + r + (q0 << tm.lg);
    const int nj = min(Q, nq - q0);
#pragma unroll
    for (int j = 0; j < Q; ++j)
      if (j < nj) { T2 o; o.x = (T)ar[j]; o.y = (T)ai[j]; pn[j * g] = o; }
  }
}

template <int FAM, int RV, int LH, int Q>
__device__ __forceinline__ void fused_levels(const FusParams& p, typename Dual<FAM>::T* U0, typename Dual<FAM>::T* W0,
                                             typename Dual<FAM>::T* U1, typename Dual<FAM>::T* W1,
                                             typename std::conditional<FAM == FI53, int2, float2>::type* D, int tau0) {
  if constexpr (LH < 16) {
    if (LH >= p.J) return;
    analyze_level<FAM, RV, LH, false>(U0, W0, p.lbuf, p.lift);
    analyze_level<FAM, RV, LH, false>(U1, W1, p.lbuf, p.lift);
    fused_term<FAM, Q>(p, LH, W0, W1, D, tau0);                // D_{LH+1} from W_{LH+1}
    // the next level reads U only and writes W after its first barrier
    fused_levels<FAM, RV, LH + 1, Q>(p, U0, W0, U1, W1, D, tau0);
  }
}

template <int FAM, int RV, int Q, int NT>
__global__ void __launch_bounds__(NT, 2) k_fused(const void* __restrict__ rows_in, void* __restrict__ corr,
                                                 void* __restrict__ partials, const __grid_constant__ FusParams p) {
  constexpr bool INT = FAM == FI53;
  typedef typename Dual<FAM>::T T;
  typedef typename std::conditional<INT, int2, float2>::type T2;
  typedef typename std::conditional<INT, PeakI, PeakF>::type PK;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int per = p.padl + 2 * (p.lbuf + p.padr);             // one component: pads, U, W
  T* U0 = reinterpret_cast<T*>(smem_raw) + p.padl;
  T* W0 = U0 + p.lbuf + p.padr;
  T* U1 = U0 + per;
  T* W1 = W0 + per;
  T2* D = reinterpret_cast<T2*>(smem_raw + (((size_t)2 * per * sizeof(T) + 15) & ~(size_t)15));   // [J+1][TT]
  constexpr int kWarps = NT / 32;
  __shared__ PK red[kMaxTerms][kWarps];

  const int tile = blockIdx.x % p.ntiles;
  const long long row = blockIdx.x / p.ntiles;
  const int tau0 = tile * p.TT;
  const long long A = (long long)tau0 - p.fML - p.halo_l;     // position of buffer index 0

  // zero pads; load both components of the extended row segment [A, A + lbuf)
  for (int c = 0; c < 2; ++c) {
    T* U = c ? U1 : U0;
    for (int u = threadIdx.x; u < p.padl; u += NT) U[u - p.padl] = T(0);
    for (int u = threadIdx.x; u < p.padr; u += NT) U[p.lbuf + u] = T(0);
  }
  {
    const int N = p.N;
    constexpr int B = 4;
    for (int u0 = threadIdx.x; u0 < p.lbuf; u0 += B * NT) {
      T v0[B], v1[B];
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int u = u0 + k * NT;
        const int idx = u < p.lbuf ? ext_index((int)(A + u), N, p.ext) : 0;
        if constexpr (INT) {
          const int16_t* src = static_cast<const int16_t*>(rows_in) + ((size_t)row * N + idx) * 2;
          const int pr = u < p.lbuf ? __ldg(reinterpret_cast<const int*>(src)) : 0;
          v0[k] = (T)(int16_t)(pr & 0xffff);
          v1[k] = (T)(int16_t)(pr >> 16);
        } else {
          const float2 z = u < p.lbuf ? __ldg(static_cast<const float2*>(rows_in) + (size_t)row * N + idx) : make_float2(0.f, 0.f);
          v0[k] = z.x;
          v1[k] = z.y;
        }
      }
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int u = u0 + k * NT;
        if (u < p.lbuf) { U0[u] = v0[k]; U1[u] = v1[k]; }
      }
    }
  }
  __syncthreads();

  fused_levels<FAM, RV, 0, Q>(p, U0, W0, U1, W1, D, tau0);
  fused_term<FAM, Q>(p, p.J, U0, U1, D, tau0);                 // A_J from U_J
  __syncthreads();

  // eq. (4) suffix sums in place (D[ti] = D[ti] + corr_{ti+1}), corr stores, peak partials
  const int TT = p.TT;
  for (int ti = p.J; ti >= 0; --ti) {
    T2* a = D + (size_t)ti * TT;
    if (ti < p.J) {
      const T2* prev = D + (size_t)(ti + 1) * TT;
      for (int tl = threadIdx.x; tl < TT; tl += NT) {
        T2 x = a[tl];
        const T2 y = prev[tl];
        if constexpr (INT) { x.x = (int)((unsigned)y.x + (unsigned)x.x); x.y = (int)((unsigned)y.y + (unsigned)x.y); }
        else { x.x = y.x + x.x; x.y = y.y + x.y; }
        a[tl] = x;
      }
      __syncthreads();
    }
    T2* dst = p.want_corr ? static_cast<T2*>(corr) + ((size_t)row * (p.J + 1) + ti) * p.N + tau0 : nullptr;
    PK best;
    best.m2 = 0; best.tau = -1; best.re = 0; best.im = 0;
    for (int tl = threadIdx.x; tl < TT; tl += NT) {
      const T2 v = a[tl];
      if (dst) dst[tl] = v;
      if (p.want_peaks) {
        if constexpr (INT) {
          const unsigned long long m = mag2i(v.x, v.y);
          if (best.tau < 0 || m > best.m2) { best.m2 = m; best.tau = tau0 + tl; best.re = v.x; best.im = v.y; }
        } else {
          const float m = mag2f(v.x, v.y);
          if (best.tau < 0 || m > best.m2) { best.m2 = m; best.tau = tau0 + tl; best.re = v.x; best.im = v.y; }
        }
      }
    }
    if (p.want_peaks) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        PK o;
        o.m2 = __shfl_down_sync(0xffffffffu, best.m2, off);
        o.tau = __shfl_down_sync(0xffffffffu, best.tau, off);
        o.re = __shfl_down_sync(0xffffffffu, best.re, off);
        o.im = __shfl_down_sync(0xffffffffu, best.im, off);
        if (o.tau >= 0 && (best.tau < 0 || beats(o.m2, o.tau, best.m2, best.tau))) best = o;
      }
      if ((threadIdx.x & 31) == 0) red[ti][threadIdx.x >> 5] = best;
    }
  }
  if (p.want_peaks) {
    __syncthreads();
    for (int ti = threadIdx.x; ti <= p.J; ti += NT) {
      PK b = red[ti][0];
      for (int w = 1; w < kWarps; ++w) {
        const PK o = red[ti][w];
        if (o.tau >= 0 && (b.tau < 0 || beats(o.m2, o.tau, b.m2, b.tau))) b = o;
      }
      static_cast<PK*>(partials)[((size_t)row * (p.J + 1) + ti) * p.ntiles + tile] = b;
    }
  }
}

}  // namespace sidwt
