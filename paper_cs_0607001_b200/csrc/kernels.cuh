// kernels.cuh -- sm_100a kernels of libsidwt.
//   k_template_pyramid : analysis pyramid of the template bank (fp64 / int64)
//   k_analyze          : fused J-level dual-analysis lifting of one (row, component,
//                        tile), all levels on chip, bands stored by TMA bulk copies
//   k_correlate        : per-scale correlation (eq. (4) suffix sums), register-blocked
//                        sliding window, fused per-tile peak partials
//   k_peaks / k_peaks_finalize : argmax over lags (smallest lag on ties)
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>

#include "lifting.cuh"

namespace sidwt {

constexpr int kMaxTerms = 17;   // J + 1 <= SIDWT_MAX_LEVELS + 1

// ---------------------------------------------------------------------------
// PTX helpers: bulk async copy smem -> global (TMA engine, SASS UBLKCP).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_store_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
               :: "l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Extension of the received row (DESIGN.md R-D6): periodic or whole-sample symmetric.
// General form (any n); the kernels use a branch-only fast path when the range allows.
__device__ __forceinline__ int ext_index(int n, int N, int ext) {
  if (ext == 0) return n & (N - 1);                 // N is a power of two
  if (N == 1) return 0;
  const int P = 2 * N - 2;
  int m = n % P;
  if (m < 0) m += P;
  return m < N ? m : P - m;
}

// ---------------------------------------------------------------------------
// K0: template pyramid.  One thread per (template, component); analysis lifting
// programs on the zero-extended template, critically sampled, in fp64 (int64).
// ---------------------------------------------------------------------------
struct PyrParams {
  int fam, J, T, n_t, taps_per_t;
  int klo[kMaxTerms], cnt[kMaxTerms], off[kMaxTerms];   // term i: b_{i+1} (i<J), a_J (i=J)
  int npad[kMaxTerms];                                  // residue stride of a term (paper orientation)
  int scratch_len;                                      // per-thread scratch length (doubles)
  int nres;                                             // 1, or 2^J residues (paper orientation)
  Lift64 lift;                                          // 9/7 analysis constants
};

template <typename V>
__device__ __forceinline__ V getz(const V* a, long lo, long hi, long n) {
  return (n < lo || n > hi) ? V(0) : a[n - lo];
}

template <typename V>
__device__ void analysis_level(int fam, const Lift64& L, const V* cur, long lo, long hi, V* e, V* o, long klo, long khi) {
  // fill e/o over [klo, khi]; conv A: (x[2k], x[2k+1]); causal D4 (R-D1): (x[2k], x[2k-1])
  for (long k = klo; k <= khi; ++k) {
    e[k - klo] = getz(cur, lo, hi, 2 * k);
    o[k - klo] = getz(cur, lo, hi, fam == FD4 ? 2 * k - 1 : 2 * k + 1);
  }
  const long n = khi - klo + 1;
  auto E = [&](long i) -> V { return (i < 0 || i >= n) ? V(0) : e[i]; };
  auto O = [&](long i) -> V { return (i < 0 || i >= n) ? V(0) : o[i]; };
  if (fam == F53) {
    for (long i = 0; i < n; ++i) o[i] = o[i] - V(0.5) * (E(i) + E(i + 1));
    for (long i = n - 1; i >= 0; --i) e[i] = e[i] + V(0.25) * (O(i) + O(i - 1));
    for (long i = 0; i < n; ++i) o[i] = V(0.5) * o[i];
  } else if (fam == F97) {      // PAPER.md:238, reading R-D3
    for (long i = 0; i < n; ++i) o[i] = o[i] + V(L.a) * (E(i) + E(i + 1));
    for (long i = n - 1; i >= 0; --i) e[i] = e[i] + V(L.b) * (O(i) + O(i - 1));
    for (long i = 0; i < n; ++i) o[i] = o[i] + V(L.g) * (E(i) + E(i + 1));
    for (long i = n - 1; i >= 0; --i) e[i] = e[i] + V(L.d) * (O(i) + O(i - 1));
    for (long i = 0; i < n; ++i) { e[i] = V(L.z) * e[i]; o[i] = o[i] / V(L.z); }
  } else if (fam == FD4) {      // eq. (17)
    for (long i = 0; i < n; ++i) o[i] = o[i] - V(kSqrt3) * e[i];
    for (long i = n - 1; i >= 0; --i) e[i] = e[i] + V(kD4c1) * O(i) + V(kD4c2) * O(i - 1);
    for (long i = n - 1; i >= 0; --i) o[i] = E(i) + O(i - 1);
    for (long i = 0; i < n; ++i) { e[i] = V(kD4K1) * e[i]; o[i] = V(kD4K2) * o[i]; }
  }
}

__device__ inline void analysis_level_int(const int64_t* cur, long lo, long hi, int64_t* e, int64_t* o, long klo, long khi) {
  for (long k = klo; k <= khi; ++k) {
    e[k - klo] = getz(cur, lo, hi, 2 * k);
    o[k - klo] = getz(cur, lo, hi, 2 * k + 1);
  }
  const long n = khi - klo + 1;
  // o -= (e_k + e_{k+1}) >> 1 ; e += (o_{k-1} + o_k + 2) >> 2   (reading R-INT)
  for (long i = 0; i < n; ++i) o[i] -= (e[i] + (i + 1 < n ? e[i + 1] : 0)) >> 1;
  for (long i = n - 1; i >= 0; --i) e[i] += ((i > 0 ? o[i - 1] : 0) + o[i] + 2) >> 2;
}

__host__ __device__ inline long fl_div2(long a) { return a >= 0 ? a / 2 : -((-a + 1) / 2); }
__host__ __device__ inline long cl_div2(long a) { return -fl_div2(-a); }

#ifndef SIDWT_NO_KERNELS   // non-template kernels: defined in the one TU that launches them (sidwt.cu)
// table: [n_t][taps_per_t] float2 (or int2); scratch: per thread 4 * scratch_len values
// nres > 1 (the paper's orientation, template carries the redundant tree): thread residue
// rho pyramids the template delayed by rho (support [rho, rho + T)); term i keeps the
// residues rho < 2^{lg_i} at table offset off[i] + rho * npad[i] + (k - klo[i]).
__global__ void k_template_pyramid(const void* __restrict__ x, void* __restrict__ table,
                                   double* __restrict__ scratch, PyrParams p) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= 2 * p.n_t * p.nres) return;
  const int rho = gid / (2 * p.n_t);
  const int t = (gid >> 1) % p.n_t, comp = gid & 1;
  const Supp sp = analysis_support(p.fam);
  const bool isint = (p.fam == FI53);
  double* base = scratch + (size_t)gid * 4 * p.scratch_len;
  long lo = rho, hi = rho + p.T - 1;
  auto slot = [&](int ti) -> int {                          // -1: this residue does not feed term ti
    if (p.nres == 1) return p.off[ti];
    const int lg = ti < p.J ? ti + 1 : p.J;
    return rho < (1 << lg) ? p.off[ti] + rho * p.npad[ti] : -1;
  };
  if (!isint) {
    double* cur = base;
    double* nxt = base + p.scratch_len;
    double* e = base + 2 * p.scratch_len;
    double* o = base + 3 * p.scratch_len;
    const float* xf = static_cast<const float*>(x) + (size_t)t * p.T * 2;
    for (int n = 0; n < p.T; ++n) cur[n] = (double)xf[2 * n + comp];
    float* tab = static_cast<float*>(table) + (size_t)t * p.taps_per_t * 2;
    for (int s = 1; s <= p.J; ++s) {
      const long alo = cl_div2(lo + sp.lLo), ahi = fl_div2(hi + sp.lHi);
      const long blo = cl_div2(lo + sp.hLo), bhi = fl_div2(hi + sp.hHi);
      const long klo = (alo < blo ? alo : blo) - 2, khi = (ahi > bhi ? ahi : bhi) + 2;
      analysis_level<double>(p.fam, p.lift, cur, lo, hi, e, o, klo, khi);
      const int ti = s - 1;
      const int sl = slot(ti);
      if (sl >= 0)
        for (long k = blo; k <= bhi; ++k) tab[2 * (sl + (k - p.klo[ti])) + comp] = (float)o[k - klo];
      for (long k = alo; k <= ahi; ++k) nxt[k - alo] = e[k - klo];
      double* tmp = cur; cur = nxt; nxt = tmp;
      lo = alo; hi = ahi;
    }
    const int sl = slot(p.J);
    for (long k = lo; k <= hi; ++k) tab[2 * (sl + (k - p.klo[p.J])) + comp] = (float)cur[k - lo];
  } else {
    int64_t* cur = reinterpret_cast<int64_t*>(base);
    int64_t* nxt = cur + p.scratch_len;
    int64_t* e = cur + 2 * p.scratch_len;
    int64_t* o = cur + 3 * p.scratch_len;
    const int16_t* xi = static_cast<const int16_t*>(x) + (size_t)t * p.T * 2;
    for (int n = 0; n < p.T; ++n) cur[n] = xi[2 * n + comp];
    int* tab = static_cast<int*>(table) + (size_t)t * p.taps_per_t * 2;
    for (int s = 1; s <= p.J; ++s) {
      const long alo = cl_div2(lo + sp.lLo), ahi = fl_div2(hi + sp.lHi);
      const long blo = cl_div2(lo + sp.hLo), bhi = fl_div2(hi + sp.hHi);
      const long klo = (alo < blo ? alo : blo) - 2, khi = (ahi > bhi ? ahi : bhi) + 2;
      analysis_level_int(cur, lo, hi, e, o, klo, khi);
      const int ti = s - 1;
      for (int i = 0; i < p.cnt[ti]; ++i) tab[2 * (p.off[ti] + i) + comp] = (int)o[p.klo[ti] + i - klo];
      for (long k = alo; k <= ahi; ++k) nxt[k - alo] = e[k - klo];
      int64_t* tmp = cur; cur = nxt; nxt = tmp;
      lo = alo; hi = ahi;
    }
    for (int i = 0; i < p.cnt[p.J]; ++i) tab[2 * (p.off[p.J] + i) + comp] = (int)cur[p.klo[p.J] + i - lo];
  }
}

#endif  // SIDWT_NO_KERNELS

// ---------------------------------------------------------------------------
// K1: fused multi-level SIDWT lifting of one (row, component, tile).
//
// smem: U[padl + lbuf + padr] (in-place working band, fine-grid positions
// A .. A+lbuf at U[padl ..]) and Wst[lbuf + padr] (detail staging, same
// indexing).  Level s (stride h = 2^{s-1}): thread w owns a run of RV
// consecutive pairs j0..j0+RV-1 of branch rho = w mod h (fine-grid positions
// rho + h j), loads RV + HL + HR values, lifts in registers, then (after a
// barrier) writes U_s in place and W_s into staging; one thread stores the
// staging plane with a bulk async copy (TMA engine) while the next level
// computes.  The level stride is a compile-time constant (one instantiation per
// level) so every shared-memory access is one instruction with an immediate
// offset; the zeroed pads absorb the reads and writes that run past the buffer
// ends, so there are no index clamps or store predicates: positions whose value
// depends on the pads lie inside the halo, which is never stored.  Each input
// sample is read from HBM once per component; every band byte is written once.
// Bank-conflict free: RV odd.
// ---------------------------------------------------------------------------
struct AnaParams {
  int N, J, ext, stride, ML;
  int tile_len, ntiles, halo_l, lbuf;
  int padl, padr;
  long long rows;
  Lift lift;
};

template <int FAM, int RV, int LH, bool BULK = true>
__device__ __forceinline__ void analyze_level(typename Dual<FAM>::T* __restrict__ U, typename Dual<FAM>::T* __restrict__ Wst,
                                              int lbuf, const Lift& L) {
  typedef typename Dual<FAM>::T T;
  constexpr int HL = Dual<FAM>::HL, HR = Dual<FAM>::HR, WIN = RV + HL + HR;
  constexpr int h = 1 << LH;
  const int w = threadIdx.x;
  const int rho = w & (h - 1);
  const int j0 = (w >> LH) * RV;
  const int len = (lbuf - rho + h - 1) >> LH;     // positions rho + h j < lbuf
  const bool active = j0 < len;
  const int u0 = rho + (j0 << LH);
  T c[RV], d[RV];
  if (active) {
    const T* src = U + u0 - HL * h;
    T v[WIN];
#pragma unroll
    for (int i = 0; i < WIN; ++i) v[i] = src[i * h];
    Dual<FAM>::template run<RV>(v, c, d, L);
  }
  if (BULK && threadIdx.x == 0 && LH > 0) bulk_wait_read_all();   // staging free again
  __syncthreads();
  if (active) {
#pragma unroll
    for (int i = 0; i < RV; ++i) {
      U[u0 + i * h] = c[i];
      Wst[u0 + i * h] = d[i];
    }
  }
  if (BULK) fence_proxy_async_smem();
  __syncthreads();
}

// Levels LH = 0 .. J-1 as straight-line code (compile-time stride per level), each
// followed by the bulk store of its detail plane.
template <int FAM, int RV, int LH>
__device__ __forceinline__ void analyze_levels(int J, typename Dual<FAM>::T* U, typename Dual<FAM>::T* Wst, int lbuf,
                                               typename Dual<FAM>::T* plane0, size_t band_step, int halo_l, int out_len,
                                               const Lift& L) {
  if constexpr (LH < 16) {
    if (LH >= J) return;
    analyze_level<FAM, RV, LH>(U, Wst, lbuf, L);
    if (threadIdx.x == 0) {
      bulk_store_s2g(plane0 + (size_t)LH * band_step, Wst + halo_l, (uint32_t)(out_len * sizeof(typename Dual<FAM>::T)));
      bulk_commit();
    }
    analyze_levels<FAM, RV, LH + 1>(J, U, Wst, lbuf, plane0, band_step, halo_l, out_len, L);
  }
}

template <int FAM, int RV>
__global__ void __launch_bounds__(512) k_analyze(const void* __restrict__ rows_in, void* __restrict__ bands, AnaParams p) {
  typedef typename Dual<FAM>::T T;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* Ubuf = reinterpret_cast<T*>(smem_raw);
  T* U = Ubuf + p.padl;
  T* Wst = Ubuf + p.padl + p.lbuf + p.padr;

  const int tile = blockIdx.x % p.ntiles;
  const long long rc = blockIdx.x / p.ntiles;
  const int comp = (int)(rc & 1);
  const long long row = rc >> 1;
  const int tstart = tile * p.tile_len;
  const int out_len = min(p.tile_len, p.stride - tstart);
  const long long A = (long long)(-p.ML + tstart) - p.halo_l;

  // zero the pads (reads past the buffer ends see finite values); 16-byte stores (padl, padr,
  // lbuf are multiples of 4)
  {
    typedef typename std::conditional<FAM == FI53, int4, float4>::type T4;
    T4 z;
    z.x = T(0); z.y = T(0); z.z = T(0); z.w = T(0);
    for (int u = threadIdx.x; u < (p.padl >> 2); u += blockDim.x) reinterpret_cast<T4*>(Ubuf)[u] = z;
    for (int u = threadIdx.x; u < (p.padr >> 2); u += blockDim.x) reinterpret_cast<T4*>(U + p.lbuf)[u] = z;
  }
  // load the extended row segment (one component); 8 independent loads in flight per thread
  {
    const int N = p.N;
    const long long A_hi = A + p.lbuf - 1;
    const bool fast = (p.ext == 0) ? (A >= -N && A_hi < 2LL * N) : (A >= -(N - 1) && A_hi <= 2LL * N - 2);
    const int Ai = (int)A;
    auto src_index = [&](int u) -> int {
      const int n = Ai + u;
      if (fast) {
        if (p.ext == 0) return n < 0 ? n + N : (n >= N ? n - N : n);
        return n < 0 ? -n : (n >= N ? 2 * N - 2 - n : n);
      }
      return ext_index(n, N, p.ext);
    };
    constexpr int B = 8;
    // interior positions [0, N) of the segment: 16-byte vector loads of 4 consecutive samples
    // (both components) and one 16-byte shared store of this component's 4 values; the
    // extension margins at the ends take the per-sample path below (needs Ai = 0 mod 4)
    int v_lo = 0, v_hi = 0;
    if ((Ai & 3) == 0) {
      v_lo = (max(0, -Ai) + 3) & ~3;
      v_hi = min(p.lbuf, N - Ai) & ~3;
      if (v_hi < v_lo) v_hi = v_lo;
      const int ngrp = (v_hi - v_lo) >> 2;
      constexpr int G = 4;
      for (int g0 = threadIdx.x; g0 < ngrp; g0 += G * blockDim.x) {
        T x[G][4];
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const int gi = g0 + k * blockDim.x;
          const int u = v_lo + 4 * gi;
          if (gi < ngrp) {
            if constexpr (FAM == FI53) {
              const int4 w = __ldg(reinterpret_cast<const int4*>(static_cast<const int16_t*>(rows_in) +
                                                              ((size_t)row * p.N + (Ai + u)) * 2));
              const int ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) x[k][e] = comp ? (ww[e] >> 16) : (int)(int16_t)(ww[e] & 0xffff);
            } else {
              const float4* q = reinterpret_cast<const float4*>(static_cast<const float*>(rows_in) +
                                                                ((size_t)row * p.N + (Ai + u)) * 2);
              const float4 a = __ldg(q), b = __ldg(q + 1);
              x[k][0] = comp ? a.y : a.x; x[k][1] = comp ? a.w : a.z;
              x[k][2] = comp ? b.y : b.x; x[k][3] = comp ? b.w : b.z;
            }
          }
        }
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const int gi = g0 + k * blockDim.x;
          if (gi < ngrp) {
            typedef typename std::conditional<FAM == FI53, int4, float4>::type T4;
            T4 o;
            o.x = x[k][0]; o.y = x[k][1]; o.z = x[k][2]; o.w = x[k][3];
            *reinterpret_cast<T4*>(U + v_lo + 4 * gi) = o;
          }
        }
      }
    }
    // the rest (extension margins, or everything when Ai is not a multiple of 4): per sample
    const int nrest = p.lbuf - (v_hi - v_lo);
    auto rest_u = [&](int i) -> int { return i < v_lo ? i : i + (v_hi - v_lo); };
    if constexpr (FAM == FI53) {
      const int16_t* src = static_cast<const int16_t*>(rows_in) + (size_t)row * p.N * 2 + comp;
      for (int i0 = threadIdx.x; i0 < nrest; i0 += B * blockDim.x) {
        T v[B];
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const int i = i0 + k * blockDim.x;
          v[k] = i < nrest ? (T)__ldg(src + 2 * (size_t)src_index(rest_u(i))) : T(0);
        }
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const int i = i0 + k * blockDim.x;
          if (i < nrest) U[rest_u(i)] = v[k];
        }
      }
    } else {
      const float* src = static_cast<const float*>(rows_in) + (size_t)row * p.N * 2 + comp;
      for (int i0 = threadIdx.x; i0 < nrest; i0 += B * blockDim.x) {
        T v[B];
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const int i = i0 + k * blockDim.x;
          v[k] = i < nrest ? __ldg(src + 2 * (size_t)src_index(rest_u(i))) : T(0);
        }
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const int i = i0 + k * blockDim.x;
          if (i < nrest) U[rest_u(i)] = v[k];
        }
      }
    }
  }
  __syncthreads();

  T* plane0 = static_cast<T*>(bands) + ((size_t)row * (p.J + 1) * 2 + comp) * p.stride + tstart;
  const size_t band_step = (size_t)2 * p.stride;

  analyze_levels<FAM, RV, 0>(p.J, U, Wst, p.lbuf, plane0, band_step, p.halo_l, out_len, p.lift);
  if (threadIdx.x == 0) {
    bulk_store_s2g(plane0 + (size_t)p.J * band_step, U + p.halo_l, (uint32_t)(out_len * sizeof(T)));
    bulk_commit();
    bulk_wait_all();
  }
}

// ---------------------------------------------------------------------------
// K4: synthesis (inverse lifting, eq. (21); PR property PAPER.md:61-63,
// 173-179): U_level over fine-grid positions [0, N) from U_J and W_J .. W_{level+1},
// coarse to fine.  One CTA per (row, component, tile of TL positions); the buffer holds
// the tile plus the accumulated inverse reach; level l needs U_l, W_l at tau + 2h m.
// ---------------------------------------------------------------------------
struct SynParams {
  int N, J, ext, stride, ML, level, TL, ntiles, halo_l, halo_r, lbuf;
  long long rows;
  Lift lift;
};

template <int FAM>
__global__ void __launch_bounds__(256) k_synthesize(const void* __restrict__ bands, void* __restrict__ out, SynParams p) {
  typedef typename Inverse<FAM>::T T;
  constexpr int SL = Inverse<FAM>::SL, SR = Inverse<FAM>::SR, W = SL + SR + 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* A = reinterpret_cast<T*>(smem_raw);
  T* B = A + p.lbuf;
  T* C = B + p.lbuf;
  const int tile = blockIdx.x % p.ntiles;
  const long long rc = blockIdx.x / p.ntiles;
  const int comp = (int)(rc & 1);
  const long long row = rc >> 1;
  const int t0 = tile * p.TL;
  const int P0 = t0 - p.halo_l;                                  // position of buffer index 0
  const T* brow = static_cast<const T*>(bands) + (size_t)row * (p.J + 1) * 2 * p.stride + (size_t)comp * p.stride;
  // stored index of fine-grid position pos of band `band` (b < J: W_{b+1}, b = J: U_J)
  auto bidx = [&](int band, int pos) -> int {
    if (p.ext == 0) return pos & (p.N - 1);
    const int lo = -p.ML, hi = p.stride - p.ML;                  // stored positions [lo, hi)
    if (pos >= lo && pos < hi) return pos + p.ML;
    // symmetric families (host-guaranteed for 5/3, 9/7, int 5/3): period 2N-2, then
    // reflection of U about 0 / of W_{b+1} about -2^b
    const int P = 2 * p.N - 2;
    int m = pos % P;
    if (m < 0) m += P;
    if (m < hi) return m + p.ML;
    if (m - P >= lo) return m - P + p.ML;
    int q = (band == p.J) ? P - m : -(2 << band) - m;
    while (q < lo) q += P;
    while (q >= hi) q -= P;
    return q + p.ML;
  };
  auto load_band = [&](int band, T* dst) {
    const T* src = brow + (size_t)band * 2 * p.stride;
    for (int u = threadIdx.x; u < p.lbuf; u += blockDim.x) dst[u] = src[bidx(band, P0 + u)];
  };
  load_band(p.J, A);                                              // U_J
  int lo = 0, hi = p.lbuf;                                        // valid range of A
  for (int l = p.J; l > p.level; --l) {
    const int st = 1 << l;                                        // pair step 2h, h = 2^{l-1}
    load_band(l - 1, B);                                          // W_l
    __syncthreads();
    const int nlo = lo + SL * st, nhi = hi - SR * st;
    for (int u = nlo + threadIdx.x; u < nhi; u += blockDim.x) {
      T c[W], d[W];
#pragma unroll
      for (int m = 0; m < W; ++m) { c[m] = A[u + (m - SL) * st]; d[m] = B[u + (m - SL) * st]; }
      C[u] = Inverse<FAM>::e(c, d, p.lift);
    }
    __syncthreads();
    T* tmp = A; A = C; C = tmp;
    lo = nlo; hi = nhi;
  }
  const int n = min(p.TL, p.N - t0);
  T* o = static_cast<T*>(out) + (size_t)row * p.N * 2 + comp;
  for (int i = threadIdx.x; i < n; i += blockDim.x) o[(size_t)(t0 + i) * 2] = A[p.halo_l + i];
}

// ---------------------------------------------------------------------------
// Peak partial record (per row, template, scale, lag tile).
// ---------------------------------------------------------------------------
struct PeakF { float m2; int tau; float re, im; };
struct PeakI { unsigned long long m2; int tau; int re, im, pad; };

__device__ __forceinline__ float mag2f(float re, float im) { return __fmaf_rn(re, re, __fmul_rn(im, im)); }
__device__ __forceinline__ unsigned long long mag2i(int re, int im) {
  return (unsigned long long)((long long)re * re) + (unsigned long long)((long long)im * im);
}
// a beats b: larger magnitude, or equal magnitude and smaller lag
template <typename M>
__device__ __forceinline__ bool beats(M ma, int ta, M mb, int tb) { return ma > mb || (ma == mb && ta < tb); }

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy global -> shared (TMA engine, SASS UBLKCP.S.G).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               :: "r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------------------
// K2: correlation.  One CTA per (row, template, lag tile of TT).  Terms are taken
// coarsest first: A_J (band J, stride 2^J), then D_J .. D_1 (band i-1, stride 2^i).
// After term i the accumulator holds corr_i (eq. (4) suffix sum) and is stored.
// Per term, thread item (r, qb) computes Q consecutive outputs of residue class r
// (lags tau = r + g q) as a sliding window over the taps: 4 FFMA (or 4 IMAD) per
// tap per output, one smem load pair per tap per item, taps broadcast from smem.
// Band tiles are double buffered: the next term's tile is fetched by two bulk
// async copies (TMA engine, mbarrier completion) while the current term computes
// (symmetric extension: contiguous ranges); periodic bands wrap and use batched
// cooperative loads instead.
// ---------------------------------------------------------------------------
struct Term { int band, lg, kmin, npad, ntap, toff; };
constexpr int kCTaps = 1536;     // template taps carried in the kernel parameters (constant cache)
struct CorParams {
  int N, J, ext, stride, ML, n_t, TT, ntiles, taps_per_t, balloc, nbuf;
  long long rows;
  int want_corr, want_peaks;
  Term term[kMaxTerms];
  uint2 ctap[kCTaps];            // [n_t][taps_per_t] float2 / int2 bits when n_t * taps_per_t <= kCTaps
};

// One chunk of REM taps (REM = Q except in an item's last chunk).  Step kk: every output
// j consumes slot (j + kk) % Q; afterwards slot kk is refilled with the value Q taps
// ahead.  In the last chunk only the refills consumed within the chunk (kk <= REM - 2)
// are issued.
// REAL: every template tap has a zero imaginary part (e.g. the Barker code of C2), so the
// two FMAs with t.y are exact no-ops and are skipped (same results, half the FMAs).
template <int Q, int REM, bool LAST, bool REAL = false>
__device__ __forceinline__ void corr_chunk_f(const float* __restrict__ pr, int plane, int g, const float2* __restrict__ tp,
                                             float (&wr)[Q], float (&wi)[Q], float (&ar)[Q], float (&ai)[Q]) {
#pragma unroll
  for (int kk = 0; kk < REM; ++kk) {
    const float2 t = tp[kk];
    const float nty = -t.y;
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const int sl = (j + kk) % Q;
      ar[j] = fmaf(t.x, wr[sl], ar[j]);
      if (!REAL) ar[j] = fmaf(t.y, wi[sl], ar[j]);
      ai[j] = fmaf(t.x, wi[sl], ai[j]);
      if (!REAL) ai[j] = fmaf(nty, wr[sl], ai[j]);
    }
    if (!LAST || kk < REM - 1) {
      const float* q = pr + kk * g;
      wr[kk] = q[0];
      wi[kk] = q[plane];
    }
  }
}

// Integer family: conj(t) w = (tx wr + ty wi) + i (tx wi - ty wr) with three multiplies,
// k = tx (wr + wi):  re = k + (ty - tx) wi,  im = k - (tx + ty) wr  (exact in the ring of
// integers mod 2^32, so bit-identical to the four-multiply form); ws = wr + wi is kept
// alongside the window, so per complex MAC: 1 IMUL + 2 IMAD on the multiply pipe (half
// rate on sm_100) and 2 IADD on the integer ALU pipe, instead of 4 IMAD.
template <int Q, int REM, bool LAST, bool REAL = false>
__device__ __forceinline__ void corr_chunk_i(const int* __restrict__ pr, int plane, int g, const int2* __restrict__ tp,
                                             unsigned (&wr)[Q], unsigned (&wi)[Q], unsigned (&ws)[Q],
                                             unsigned (&ar)[Q], unsigned (&ai)[Q]) {
#pragma unroll
  for (int kk = 0; kk < REM; ++kk) {
    const int2 t = tp[kk];
    const unsigned tx = (unsigned)t.x, ty = (unsigned)t.y;
    const unsigned d1 = ty - tx, d2 = 0u - tx - ty;
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const int sl = (j + kk) % Q;
      if (REAL) {
        ar[j] += tx * wr[sl];
        ai[j] += tx * wi[sl];
      } else {
        const unsigned k = tx * ws[sl];
        ar[j] += k + d1 * wi[sl];                    // wrap-around int32 (exact mod 2^32)
        ai[j] += k + d2 * wr[sl];
      }
    }
    if (!LAST || kk < REM - 1) {
      const int* q = pr + kk * g;
      wr[kk] = (unsigned)q[0];
      wi[kk] = (unsigned)q[plane];
      if (!REAL) ws[kk] = wr[kk] + wi[kk];
    }
  }
}

template <bool INT, int Q, int REM, bool REAL = false>
__device__ __forceinline__ void corr_chunk(const typename std::conditional<INT, int, float>::type* pr, int plane, int g,
                                           const typename std::conditional<INT, int2, float2>::type* tp,
                                           typename std::conditional<INT, unsigned, float>::type (&wr)[Q],
                                           typename std::conditional<INT, unsigned, float>::type (&wi)[Q],
                                           typename std::conditional<INT, unsigned, float>::type (&ws)[Q],
                                           typename std::conditional<INT, unsigned, float>::type (&ar)[Q],
                                           typename std::conditional<INT, unsigned, float>::type (&ai)[Q]) {
  if constexpr (INT) corr_chunk_i<Q, REM, true, REAL>(pr, plane, g, tp, wr, wi, ws, ar, ai);
  else corr_chunk_f<Q, REM, true, REAL>(pr, plane, g, tp, wr, wi, ar, ai);
}

// Last chunk of an item: REM = rem taps (1..Q), dispatched to a compile-time length.
template <bool INT, int Q, int R, bool REAL = false>
__device__ __forceinline__ void corr_last(int rem, const typename std::conditional<INT, int, float>::type* pr, int plane, int g,
                                          const typename std::conditional<INT, int2, float2>::type* tp,
                                          typename std::conditional<INT, unsigned, float>::type (&wr)[Q],
                                          typename std::conditional<INT, unsigned, float>::type (&wi)[Q],
                                          typename std::conditional<INT, unsigned, float>::type (&ws)[Q],
                                          typename std::conditional<INT, unsigned, float>::type (&ar)[Q],
                                          typename std::conditional<INT, unsigned, float>::type (&ai)[Q]) {
  if constexpr (R >= Q) {
    corr_chunk<INT, Q, Q, REAL>(pr, plane, g, tp, wr, wi, ws, ar, ai);
  } else {
    if (rem == R) corr_chunk<INT, Q, R, REAL>(pr, plane, g, tp, wr, wi, ws, ar, ai);
    else corr_last<INT, Q, R + 1, REAL>(rem, pr, plane, g, tp, wr, wi, ws, ar, ai);
  }
}

// One item: Q outputs q0..q0+Q-1 of residue r; band tile value for output q, tap k' at
// sb[r + g (q + k')] (re plane) and sb[... + plane] (im plane).  No index clamps: the
// tile holds every value the valid outputs need; outputs past the residue's end (the
// ragged last q-block) read at most g (Q-1) values past the tile, inside the buffer.
template <bool INT, int Q, bool PAPER = false, bool REAL = false>
__device__ __forceinline__ void corr_item(const typename std::conditional<INT, int, float>::type* sb, int plane,
                                          const typename std::conditional<INT, int2, float2>::type* tp, int ntap,
                                          int r, int lg, int q0,
                                          typename std::conditional<INT, unsigned, float>::type (&ar)[Q],
                                          typename std::conditional<INT, unsigned, float>::type (&ai)[Q]) {
  typedef typename std::conditional<INT, unsigned, float>::type A;
  const int g = 1 << lg;
  A wr[Q], wi[Q], ws[Q];
  // received-tree orientation: outputs r + g q read W[r + g (q + k)]; the paper's orientation
  // (template tree) reads the critically sampled received band W[g (q + k)] with the
  // template's residue-r taps
  const auto* base = sb + (PAPER ? 0 : r) + (q0 << lg);
#pragma unroll
  for (int m = 0; m < Q; ++m) {
    wr[m] = (A)base[m << lg];
    wi[m] = (A)base[(m << lg) + plane];
    if constexpr (INT) ws[m] = wr[m] + wi[m];
    ar[m] = A(0);
    ai[m] = A(0);
  }
  const auto* pr = base + (Q << lg);
  const int nfull = (ntap - 1) / Q;          // full chunks; the last chunk has 1..Q taps
  for (int c = 0; c < nfull; ++c, pr += Q * g, tp += Q) {
    if constexpr (INT) corr_chunk_i<Q, Q, false, REAL>(pr, plane, g, tp, wr, wi, ws, ar, ai);
    else corr_chunk_f<Q, Q, false, REAL>(pr, plane, g, tp, wr, wi, ar, ai);
  }
  corr_last<INT, Q, 1, REAL>(ntap - nfull * Q, pr, plane, g, tp, wr, wi, ws, ar, ai);
}

// Real-template item with packed FP32 pairs: the window holds (wr, wi) pairs and the
// accumulator (ar, ai) pairs, and every tap is one fma.rn.f32x2 (FFMA2) per output instead
// of two FFMAs -- each lane of the pair is the same fused multiply-add, so results are
// bit-identical (the tap's real part is duplicated into both lanes).
__device__ __forceinline__ unsigned long long f2pack(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void f2unpack(unsigned long long v, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}
__device__ __forceinline__ void ffma2(unsigned long long& a, unsigned long long t, unsigned long long w) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(t), "l"(w));
}

template <int Q, int REM, bool LAST>
__device__ __forceinline__ void corr_chunk_r2(const float* __restrict__ pr, int plane, int g,
                                              const float2* __restrict__ tp,
                                              unsigned long long (&w)[Q], unsigned long long (&a)[Q]) {
#pragma unroll
  for (int kk = 0; kk < REM; ++kk) {
    const float tx = tp[kk].x;                                 // constant cache
    const unsigned long long t = f2pack(tx, tx);
#pragma unroll
    for (int j = 0; j < Q; ++j) ffma2(a[j], t, w[(j + kk) % Q]);
    if (!LAST || kk < REM - 1) {
      const float* q = pr + kk * g;
      w[kk] = f2pack(q[0], q[plane]);
    }
  }
}

template <int Q, int R>
__device__ __forceinline__ void corr_last_r2(int rem, const float* pr, int plane, int g, const float2* tp,
                                             unsigned long long (&w)[Q], unsigned long long (&a)[Q]) {
  if constexpr (R >= Q) {
    corr_chunk_r2<Q, Q, true>(pr, plane, g, tp, w, a);
  } else {
    if (rem == R) corr_chunk_r2<Q, R, true>(pr, plane, g, tp, w, a);
    else corr_last_r2<Q, R + 1>(rem, pr, plane, g, tp, w, a);
  }
}

template <int Q>
__device__ __forceinline__ void corr_item_r2(const float* sb, int plane, const float2* tp, int ntap, int r, int lg,
                                             int q0, float (&ar)[Q], float (&ai)[Q]) {
  const int g = 1 << lg;
  unsigned long long w[Q], a[Q];
  const float* base = sb + r + (q0 << lg);
#pragma unroll
  for (int m = 0; m < Q; ++m) {
    w[m] = f2pack(base[m << lg], base[(m << lg) + plane]);
    a[m] = 0ull;
  }
  const float* pr = base + (Q << lg);
  const int nfull = (ntap - 1) / Q;
  for (int c = 0; c < nfull; ++c, pr += Q * g, tp += Q) corr_chunk_r2<Q, Q, false>(pr, plane, g, tp, w, a);
  corr_last_r2<Q, 1>(ntap - nfull * Q, pr, plane, g, tp, w, a);
#pragma unroll
  for (int m = 0; m < Q; ++m) f2unpack(a[m], ar[m], ai[m]);
}

// All items of one term: thread item (r, qb) computes Q outputs of residue r, then the
// eq. (4) suffix sum corr_ti = corr_{ti+1} + term into the other accumulator buffer.
// LG >= 0: g = 2^LG is a compile-time constant; LG = -1: runtime lg.
template <bool INT, int Q, bool PAPER, bool REAL, int LG>
__device__ __forceinline__ void corr_term(const typename std::conditional<INT, int, float>::type* sb, int plane,
                                          const typename std::conditional<INT, int2, float2>::type* tp, const Term& tm,
                                          int lg_rt, int TT, const typename std::conditional<INT, int2, float2>::type* aprev,
                                          typename std::conditional<INT, int2, float2>::type* anew, bool first) {
  typedef typename std::conditional<INT, int, float>::type T;
  typedef typename std::conditional<INT, int2, float2>::type T2;
  typedef typename std::conditional<INT, unsigned, float>::type A;
  const int lg = LG >= 0 ? LG : lg_rt;
  const int g = 1 << lg;
  const int nq = TT >> lg;
  const int nqb = (nq + Q - 1) / Q;
  for (int w = threadIdx.x; w < g * nqb; w += blockDim.x) {
    const int r = w & (g - 1);
    const int q0 = (w >> lg) * Q;
    A ar[Q], ai[Q];
    if constexpr (!INT && REAL && !PAPER) corr_item_r2<Q>(sb, plane, tp, tm.ntap, r, lg, q0, ar, ai);
    else corr_item<INT, Q, PAPER, REAL>(sb, plane, tp + (PAPER ? r * tm.npad : 0), tm.ntap, r, lg, q0, ar, ai);
    // eq. (4) suffix sum: corr_ti = corr_{ti+1} + term (outputs r + g (q0 + j))
    const int base = r + (q0 << lg);
    const T2* pp = aprev + base;
    T2* pn = anew + base;
    const int nj = min(Q, nq - q0);
    if (first) {
#pragma unroll
      for (int j = 0; j < Q; ++j)
        if (j < nj) { T2 o; o.x = (T)ar[j]; o.y = (T)ai[j]; pn[j * g] = o; }
    } else if (nj == Q) {
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        const T2 v = pp[j * g];
        T2 o; o.x = (T)((A)v.x + ar[j]); o.y = (T)((A)v.y + ai[j]);
        pn[j * g] = o;
      }
    } else {
#pragma unroll
      for (int j = 0; j < Q; ++j)
        if (j < nj) {
          const T2 v = pp[j * g];
          T2 o; o.x = (T)((A)v.x + ar[j]); o.y = (T)((A)v.y + ai[j]);
          pn[j * g] = o;
        }
    }
  }
}

template <bool INT, int Q, int NT, int MINB, bool CT, bool PAPER = false, bool REAL = false>
__global__ void __launch_bounds__(NT, MINB) k_correlate(const void* __restrict__ bands, const void* __restrict__ taps,
                                                   void* __restrict__ corr, void* __restrict__ partials,
                                                   const __grid_constant__ CorParams p) {
  typedef typename std::conditional<INT, int, float>::type T;
  typedef typename std::conditional<INT, int2, float2>::type T2;
  typedef typename std::conditional<INT, unsigned, float>::type A;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw);                 // [2]
  T2* stap = reinterpret_cast<T2*>(smem_raw + 16);
  T* sbuf = reinterpret_cast<T*>(smem_raw + 16 + (((size_t)p.taps_per_t * sizeof(T2) + 127) & ~(size_t)127));  // [2][2][balloc]
  T2* acc = reinterpret_cast<T2*>(sbuf + 2 * (size_t)p.nbuf * p.balloc);   // [2 buffers][TT] complex (re, im)
  constexpr int kWarps = NT / 32;
  typedef typename std::conditional<INT, PeakI, PeakF>::type PK;
  __shared__ PK red[kMaxTerms][kWarps];

  const int tile = blockIdx.x % p.ntiles;
  const long long bt = blockIdx.x / p.ntiles;
  const int t = (int)(bt % p.n_t);
  const long long row = bt / p.n_t;
  const int tau0 = tile * p.TT;
  const int TT = p.TT;
  const int plane = p.balloc;
  const bool tma = (p.ext != 0);
  const T* brow = static_cast<const T*>(bands) + (size_t)row * (p.J + 1) * 2 * p.stride;

  // tile of term `ti` starts at band index a (symmetric: pos + ML >= 0, always in range)
  auto issue = [&](int step, int b) {
    const Term tm = p.term[p.J - step];
    const int g = 1 << tm.lg;
    const int blen = TT + g * (tm.ntap - 1);
    const int a = tau0 + g * tm.kmin + p.ML;
    const int a4 = a & ~3;
    const uint32_t bytes = (uint32_t)(((a - a4) + blen + 3) & ~3) * 4u;
    const T* src = brow + (size_t)tm.band * 2 * p.stride + a4;
    T* dst = sbuf + (size_t)b * 2 * p.balloc;
    mbar_expect_tx(&mbar[b], 2 * bytes);
    bulk_load_g2s(dst, src, bytes, &mbar[b]);
    bulk_load_g2s(dst + p.balloc, src + p.stride, bytes, &mbar[b]);
  };

  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const T2* tsrc = static_cast<const T2*>(taps) + (size_t)t * p.taps_per_t;
  if (!CT)
    for (int i = threadIdx.x; i < p.taps_per_t; i += blockDim.x) stap[i] = tsrc[i];
  const T2* tbase = CT ? reinterpret_cast<const T2*>(p.ctap) + (size_t)t * p.taps_per_t : stap;
  __syncthreads();
  if (tma && threadIdx.x == 0) issue(0, 0);
  const bool dbl = p.nbuf == 2;

  int cur = 0;
  for (int step = 0; step <= p.J; ++step) {
    const int ti = p.J - step;
    const Term tm = p.term[ti];
    const int g = 1 << tm.lg;
    const int b = dbl ? (step & 1) : 0;
    T* sb = sbuf + (size_t)b * 2 * p.balloc;
    if (tma) {
      // double buffer: prefetch the next term now; single buffer: after this compute
      if (dbl && threadIdx.x == 0 && step < p.J) issue(step + 1, b ^ 1);
      mbar_wait(&mbar[b], (uint32_t)(dbl ? ((step >> 1) & 1) : (step & 1)));
      const int a = tau0 + g * tm.kmin + p.ML;
      sb += (a & 3);
    } else {
      // periodic: wrapped positions, batched cooperative loads (8 in flight per thread)
      const int blen = TT + g * (tm.ntap - 1);
      const int pos0 = tau0 + g * tm.kmin;
      const T* pre = brow + (size_t)tm.band * 2 * p.stride;
      for (int x0 = threadIdx.x; x0 < blen; x0 += 8 * blockDim.x) {
        T vr[8], vi[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int xx = x0 + k * blockDim.x;
          const int idx = (pos0 + xx) & (p.N - 1);
          vr[k] = xx < blen ? __ldg(pre + idx) : T(0);
          vi[k] = xx < blen ? __ldg(pre + p.stride + idx) : T(0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int xx = x0 + k * blockDim.x;
          if (xx < blen) { sb[xx] = vr[k]; sb[plane + xx] = vi[k]; }
        }
      }
      __syncthreads();
    }
    // compute term, accumulate into acc[cur^1] = acc[cur] + term; the band stride g = 2^lg
    // is dispatched to a compile-time constant (immediate shared-memory offsets in the tap loop)
    const T2* aprev = acc + (size_t)cur * TT;
    T2* anew = acc + (size_t)(cur ^ 1) * TT;
    const T2* tp = tbase + tm.toff;
    switch (tm.lg) {
      case 1: corr_term<INT, Q, PAPER, REAL, 1>(sb, plane, tp, tm, 1, TT, aprev, anew, step == 0); break;
      case 2: corr_term<INT, Q, PAPER, REAL, 2>(sb, plane, tp, tm, 2, TT, aprev, anew, step == 0); break;
      case 3: corr_term<INT, Q, PAPER, REAL, 3>(sb, plane, tp, tm, 3, TT, aprev, anew, step == 0); break;
      case 4: corr_term<INT, Q, PAPER, REAL, 4>(sb, plane, tp, tm, 4, TT, aprev, anew, step == 0); break;
      case 5: corr_term<INT, Q, PAPER, REAL, 5>(sb, plane, tp, tm, 5, TT, aprev, anew, step == 0); break;
      case 6: corr_term<INT, Q, PAPER, REAL, 6>(sb, plane, tp, tm, 6, TT, aprev, anew, step == 0); break;
      default: corr_term<INT, Q, PAPER, REAL, -1>(sb, plane, tp, tm, tm.lg, TT, aprev, anew, step == 0); break;
    }
    __syncthreads();
    if (tma && !dbl && threadIdx.x == 0 && step < p.J) issue(step + 1, 0);
    cur ^= 1;
    // store corr_ti (4 lags per thread-iteration, 2 x 16-byte stores) and reduce this tile's
    // peak partial: lags increase within a thread, so a strict '>' keeps the smallest lag.
    const T2* a = acc + (size_t)cur * TT;
    T2* dst = p.want_corr ? static_cast<T2*>(corr) + (((size_t)row * p.n_t + t) * (p.J + 1) + ti) * p.N + tau0 : nullptr;
    PK best;
    best.m2 = 0; best.tau = -1; best.re = 0; best.im = 0;
    auto consider = [&](T re, T im, int tau) {
      if constexpr (INT) {
        const unsigned long long m = mag2i(re, im);
        const bool bt = (best.tau < 0) || (m > best.m2);
        best.m2 = bt ? m : best.m2; best.tau = bt ? tau : best.tau; best.re = bt ? re : best.re; best.im = bt ? im : best.im;
      } else {
        const float m = mag2f(re, im);
        const bool bt = (best.tau < 0) || (m > best.m2);
        best.m2 = bt ? m : best.m2; best.tau = bt ? tau : best.tau; best.re = bt ? re : best.re; best.im = bt ? im : best.im;
      }
    };
    if ((TT & 1) == 0) {
      // two lags per 16-byte load / store, straight copy of the interleaved accumulator
      typedef typename std::conditional<INT, int4, float4>::type T4;
      for (int tl = threadIdx.x * 2; tl < TT; tl += blockDim.x * 2) {
        const T4 v = *reinterpret_cast<const T4*>(a + tl);
        if (dst) *reinterpret_cast<T4*>(dst + tl) = v;
        if (p.want_peaks) {
          if constexpr (INT) {
            // pair maximum first (ties keep the earlier lag), then one compare with the best
            const unsigned long long m0 = mag2i(v.x, v.y), m1 = mag2i(v.z, v.w);
            const bool k0 = m0 >= m1;
            const unsigned long long mx = k0 ? m0 : m1;
            if (best.tau < 0 || mx > best.m2) {
              best.m2 = mx; best.tau = tau0 + tl + (k0 ? 0 : 1);
              best.re = k0 ? v.x : v.z; best.im = k0 ? v.y : v.w;
            }
          } else {
            const float m0 = mag2f(v.x, v.y), m1 = mag2f(v.z, v.w);
            const float mx = fmaxf(m0, m1);
            if (best.tau < 0 || mx > best.m2) {
              const bool k0 = m0 == mx;
              best.m2 = mx; best.tau = tau0 + tl + (k0 ? 0 : 1);
              best.re = k0 ? v.x : v.z; best.im = k0 ? v.y : v.w;
            }
          }
        }
      }
    } else {
      for (int tl = threadIdx.x; tl < TT; tl += blockDim.x) {
        const T2 v = a[tl];
        if (dst) dst[tl] = v;
        if (p.want_peaks) consider(v.x, v.y, tau0 + tl);
      }
    }
    if (p.want_peaks) {
      if constexpr (INT) {
        // warp argmax of the 64-bit |.|^2 by three hardware reductions: the largest high word,
        // the largest low word among those lanes, then the smallest lag attaining both
        const bool ok = best.tau >= 0;
        const unsigned hi = ok ? (unsigned)(best.m2 >> 32) : 0u, lo = ok ? (unsigned)best.m2 : 0u;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, (ok && hi == mhi) ? lo : 0u);
        const unsigned cand = (ok && hi == mhi && lo == mlo) ? (unsigned)best.tau : 0xffffffffu;
        const unsigned tmin = __reduce_min_sync(0xffffffffu, cand);
        if (ok && (unsigned)best.tau == tmin) red[ti][threadIdx.x >> 5] = best;
        else if ((threadIdx.x & 31) == 0 && tmin == 0xffffffffu) { PK e; e.m2 = 0; e.tau = -1; e.re = 0; e.im = 0; e.pad = 0; red[ti][threadIdx.x >> 5] = e; }
      } else {
        // warp argmax by two hardware reductions: the largest |.|^2 (float bits of a
        // non-negative float order like unsigned ints), then the smallest lag attaining it
        const unsigned mb = best.tau >= 0 ? __float_as_uint(best.m2) : 0u;
        const unsigned mmax = __reduce_max_sync(0xffffffffu, mb);
        const unsigned cand = (best.tau >= 0 && mb == mmax) ? (unsigned)best.tau : 0xffffffffu;
        const unsigned tmin = __reduce_min_sync(0xffffffffu, cand);
        if (best.tau >= 0 && (unsigned)best.tau == tmin) red[ti][threadIdx.x >> 5] = best;
        else if ((threadIdx.x & 31) == 0 && tmin == 0xffffffffu) { PK e; e.m2 = 0; e.tau = -1; e.re = 0; e.im = 0; red[ti][threadIdx.x >> 5] = e; }
      }
    }
  }
  if (p.want_peaks) {
    __syncthreads();
    for (int ti = threadIdx.x; ti <= p.J; ti += blockDim.x) {
      PK b = red[ti][0];
      for (int w = 1; w < kWarps; ++w) {
        const PK o = red[ti][w];
        if (o.tau >= 0 && (b.tau < 0 || beats(o.m2, o.tau, b.m2, b.tau))) b = o;
      }
      static_cast<PK*>(partials)[(((size_t)row * p.n_t + t) * (p.J + 1) + ti) * p.ntiles + tile] = b;
    }
  }
}

// Combine per-tile peak partials (tiles ordered by lag: ties keep the earlier tile; the
// comparison carries the lag, so the combination order does not matter).  One warp per
// (row, template, scale): coalesced reads of its partials, shuffle reduction.
template <bool INT>
__global__ void __launch_bounds__(256) k_peaks_finalize(const void* __restrict__ partials, int ntiles, long long count,
                                                        int32_t* __restrict__ lag, void* __restrict__ val) {
  typedef typename std::conditional<INT, PeakI, PeakF>::type PK;
  typedef typename std::conditional<INT, int2, float2>::type T2;
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= count) return;
  const PK* pp = static_cast<const PK*>(partials) + (size_t)i * ntiles;
  PK b;
  b.m2 = 0; b.tau = -1; b.re = 0; b.im = 0;
  for (int k = lane; k < ntiles; k += 32) {
    const PK o = pp[k];
    if (o.tau >= 0 && (b.tau < 0 || beats(o.m2, o.tau, b.m2, b.tau))) b = o;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    PK o;
    o.m2 = __shfl_down_sync(0xffffffffu, b.m2, off);
    o.tau = __shfl_down_sync(0xffffffffu, b.tau, off);
    o.re = __shfl_down_sync(0xffffffffu, b.re, off);
    o.im = __shfl_down_sync(0xffffffffu, b.im, off);
    if (o.tau >= 0 && (b.tau < 0 || beats(o.m2, o.tau, b.m2, b.tau))) b = o;
  }
  if (lane == 0) {
    lag[i] = b.tau;
    if (val) { T2 v; v.x = b.re; v.y = b.im; static_cast<T2*>(val)[i] = v; }
  }
}

// K3: standalone peak search over a stored correlation [count][N].
template <bool INT>
__global__ void __launch_bounds__(256) k_peaks(const void* __restrict__ corr, int N, int32_t* __restrict__ lag,
                                               void* __restrict__ val) {
  typedef typename std::conditional<INT, PeakI, PeakF>::type PK;
  typedef typename std::conditional<INT, int2, float2>::type T2;
  __shared__ PK red[8];
  const T2* c = static_cast<const T2*>(corr) + (size_t)blockIdx.x * N;
  PK best;
  best.m2 = 0; best.tau = 0x7fffffff; best.re = 0; best.im = 0;
  for (int tau = threadIdx.x; tau < N; tau += blockDim.x) {
    const T2 v = c[tau];
    if constexpr (INT) {
      const unsigned long long m = mag2i(v.x, v.y);
      if (best.tau == 0x7fffffff || beats(m, tau, best.m2, best.tau)) { best.m2 = m; best.tau = tau; best.re = v.x; best.im = v.y; }
    } else {
      const float m = mag2f(v.x, v.y);
      if (best.tau == 0x7fffffff || beats(m, tau, best.m2, best.tau)) { best.m2 = m; best.tau = tau; best.re = v.x; best.im = v.y; }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    PK o;
    o.m2 = __shfl_down_sync(0xffffffffu, best.m2, off);
    o.tau = __shfl_down_sync(0xffffffffu, best.tau, off);
    o.re = __shfl_down_sync(0xffffffffu, best.re, off);
    o.im = __shfl_down_sync(0xffffffffu, best.im, off);
    if (o.tau != 0x7fffffff && (best.tau == 0x7fffffff || beats(o.m2, o.tau, best.m2, best.tau))) best = o;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    PK b = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      const PK o = red[w];
      if (o.tau != 0x7fffffff && (b.tau == 0x7fffffff || beats(o.m2, o.tau, b.m2, b.tau))) b = o;
    }
    lag[blockIdx.x] = b.tau;
    if (val) { T2 v; v.x = b.re; v.y = b.im; static_cast<T2*>(val)[blockIdx.x] = v; }
  }
}

}  // namespace sidwt
