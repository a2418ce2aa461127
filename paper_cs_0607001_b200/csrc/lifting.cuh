// lifting.cuh -- the paper's lifting programs, as register-resident in-place
// step sequences.  Two uses:
//   * Dual-analysis programs (received signal, fp32 / int32) applied to a run of
//     RV consecutive pairs of one level-(s-1) branch, the fine-grid form of the
//     SIDWT tree: pair j = (v_j, v_{j+1}) (or
//     (v_j, v_{j-1}) for causal D4), lifting neighbours j +- 2.
//   * Analysis programs (template, fp64 / int64) on a zero-extended finite
//     sequence, critically sampled ("stored").
// Constants: Table I; eq. (17) (reading R-D2).
#pragma once
#include <cstdint>

namespace sidwt {

enum Family { F53 = 0, F97 = 1, FD4 = 2, FI53 = 3 };

// Table I, t = 5/4.
constexpr double kAlpha = -1.5, kBeta = -0.0625, kGamma = 0.8, kDelta = 0.46875;
constexpr double kZeta = 1.1313708498984760390;      // 4 sqrt(2) / 5

// 9/7 lifting constants as kernel parameters.  The paper's free-variable family
// (the finite-precision 9/7 of its ref. [10]):
//   alpha = (1 - 2t) / (4 (t - 1)), beta = -(t - 1)^2, gamma = 1 / (4 t (t - 1)),
//   delta = t^3 - 7/4 t^2 + t, zeta = sqrt(2) / t,
// with t = 5/4 giving Table I and t = 1.2301741... the irrational CDF 9/7 of ref. [28].
// The other families ignore them.
struct Lift64 { double a, b, g, d, z; };
struct Lift { float a, b, g, d, z, iz; };
__host__ inline Lift64 lift97_t(double t) {
  if (t == 1.25) return {kAlpha, kBeta, kGamma, kDelta, kZeta};
  return {(1.0 - 2.0 * t) / (4.0 * (t - 1.0)), -(t - 1.0) * (t - 1.0), 1.0 / (4.0 * t * (t - 1.0)),
          t * t * t - 1.75 * t * t + t, 1.4142135623730950488 / t};
}
__host__ inline Lift lift_f32(const Lift64& k) {
  return {(float)k.a, (float)k.b, (float)k.g, (float)k.d, (float)k.z, (float)(1.0 / k.z)};
}
// eq. (17)
constexpr double kSqrt3 = 1.7320508075688772935;
constexpr double kD4c1 = 0.43301270189221932338;     // sqrt3 / 4
constexpr double kD4c2 = -0.066987298107780676618;   // (sqrt3 - 2) / 4
constexpr double kD4K1 = 1.9318516525781365735;      // (sqrt3 + 1) / sqrt2
constexpr double kD4K2 = 0.51763809020504152470;     // (sqrt3 - 1) / sqrt2

// ---------------------------------------------------------------------------
// Dual-analysis programs on a run.  v[0..WIN) holds v_j for j = j0 - HL + i.
// Outputs c[i], d[i] for pairs j = j0 + i, i in [0, RV).
// ---------------------------------------------------------------------------
template <int FAM> struct Dual;

// LeGall 5/3, P^T(z^-1) = diag(1,2) [1,0; -1/4(1+z),1] [1, 1/2(1+z^-1); 0,1]
// (reading R-D4): e += 1/2 (o_k + o_{k-1}); o -= 1/4 (e_k + e_{k+1}); d = 2 o.
template <> struct Dual<F53> {
  typedef float T;
  static constexpr int HL = 1, HR = 3;
  template <int RV>
  __device__ __forceinline__ static void run(const float (&v)[RV + HL + HR], float (&c)[RV], float (&d)[RV], const Lift& L) {
    float e1[RV + 2];
#pragma unroll
    for (int a = 0; a < RV + 2; ++a) e1[a] = fmaf(0.5f, v[a] + v[a + 2], v[a + 1]);
#pragma unroll
    for (int a = 0; a < RV; ++a) {
      c[a] = e1[a];
      d[a] = 2.0f * fmaf(-0.25f, e1[a] + e1[a + 2], v[a + 2]);
    }
  }
};

// CDF 9/7 dual analysis (reading R-D3, mechanical dual of the analysis program):
// e += -alpha(o_k + o_{k-1}); o += -beta(e_k + e_{k+1}); e += -gamma(..); o += -delta(..);
// c = e / zeta, d = zeta o.
template <> struct Dual<F97> {
  typedef float T;
  static constexpr int HL = 3, HR = 5;
  template <int RV>
  __device__ __forceinline__ static void run(const float (&v)[RV + HL + HR], float (&c)[RV], float (&d)[RV], const Lift& L) {
    const float na = -L.a, nb = -L.b, ng = -L.g, nd = -L.d;
    float e1[RV + 6], o1[RV + 4], e2[RV + 2];
#pragma unroll
    for (int a = 0; a < RV + 6; ++a) e1[a] = fmaf(na, v[a] + v[a + 2], v[a + 1]);      // j = j0-2+a
#pragma unroll
    for (int a = 0; a < RV + 4; ++a) o1[a] = fmaf(nb, e1[a] + e1[a + 2], v[a + 2]);    // j = j0-2+a
#pragma unroll
    for (int b = 0; b < RV + 2; ++b) e2[b] = fmaf(ng, o1[b + 2] + o1[b], e1[b + 2]);   // j = j0+b
#pragma unroll
    for (int b = 0; b < RV; ++b) {
      const float o2 = fmaf(nd, e2[b] + e2[b + 2], o1[b + 2]);
      c[b] = e2[b] * L.iz;
      d[b] = o2 * L.z;
    }
  }
};

// Causal Daubechies-4, eq. (17), pairs (x[2k], x[2k-1]) (reading R-D1):
// o -= sqrt3 e; e += c1 o_k + c2 o_{k-1}; o <- e_k + o_{k-1}; a = K1 e, b = K2 o.
template <> struct Dual<FD4> {
  typedef float T;
  static constexpr int HL = 3, HR = 0;
  template <int RV>
  __device__ __forceinline__ static void run(const float (&v)[RV + HL + HR], float (&c)[RV], float (&d)[RV], const Lift& L) {
    float o1[RV + 2];
#pragma unroll
    for (int a = 0; a < RV + 2; ++a) o1[a] = fmaf(-(float)kSqrt3, v[a + 1], v[a]);      // j = j0-2+a
#pragma unroll
    for (int b = 0; b < RV; ++b) {
      const float e1 = fmaf((float)kD4c2, o1[b], fmaf((float)kD4c1, o1[b + 2], v[b + 3]));
      c[b] = (float)kD4K1 * e1;
      d[b] = (float)kD4K2 * (e1 + o1[b]);
    }
  }
};

// Reversible integer 5/3 (reading R-INT): e += (o_k + o_{k-1}) >> 1;
// o -= (e_k + e_{k+1} + 2) >> 2; c = e, d = o.  >> is an arithmetic shift (floor).
template <> struct Dual<FI53> {
  typedef int T;
  static constexpr int HL = 1, HR = 3;
  template <int RV>
  __device__ __forceinline__ static void run(const int (&v)[RV + HL + HR], int (&c)[RV], int (&d)[RV], const Lift&) {
    int e1[RV + 2];
#pragma unroll
    for (int a = 0; a < RV + 2; ++a) e1[a] = v[a + 1] + ((v[a] + v[a + 2]) >> 1);
#pragma unroll
    for (int a = 0; a < RV; ++a) {
      c[a] = e1[a];
      d[a] = v[a + 2] - ((e1[a] + e1[a + 2] + 2) >> 2);
    }
  }
};

// ---------------------------------------------------------------------------
// Inverse dual-analysis programs (synthesis, eq. (21): the finer
// approximation from the coarser (approximation, detail) pair by the inverse lifting
// steps).  On the fine grid: U_{s-1}[tau] = e of the pair at tau, from c = U_s and
// d = W_s at tau + 2h m (h = 2^{s-1}); c[i], d[i] hold m = i - SL.
// ---------------------------------------------------------------------------
template <int FAM> struct Inverse;

// 5/3: o_k = d_k / 2 + (c_k + c_{k+1}) / 4 ; e_k = c_k - (o_k + o_{k-1}) / 2
template <> struct Inverse<F53> {
  typedef float T;
  static constexpr int SL = 1, SR = 1;
  __device__ __forceinline__ static float e(const float (&c)[3], const float (&d)[3], const Lift&) {
    const float ok = fmaf(0.5f, d[1], 0.25f * (c[1] + c[2]));
    const float om = fmaf(0.5f, d[0], 0.25f * (c[0] + c[1]));
    return fmaf(-0.5f, ok + om, c[1]);
  }
};

// CDF 9/7 (reading R-D3): e4 = zeta c, o4 = d / zeta; o3 = o4 + delta (e4_k + e4_{k+1});
// e2 = e4 + gamma (o3_k + o3_{k-1}); o1 = o3 + beta (e2_k + e2_{k+1}); e = e2 + alpha (o1_k + o1_{k-1})
template <> struct Inverse<F97> {
  typedef float T;
  static constexpr int SL = 2, SR = 2;
  __device__ __forceinline__ static float e(const float (&c)[5], const float (&d)[5], const Lift& L) {
    const float z = L.z, iz = L.iz;
    float e4[5], o4[4], o3[4], e2[3], o1[2];
#pragma unroll
    for (int i = 0; i < 5; ++i) e4[i] = z * c[i];          // m = i - 2
#pragma unroll
    for (int i = 0; i < 4; ++i) o4[i] = iz * d[i];         // m = i - 2
#pragma unroll
    for (int i = 0; i < 4; ++i) o3[i] = fmaf(L.d, e4[i] + e4[i + 1], o4[i]);   // m = i - 2
#pragma unroll
    for (int i = 0; i < 3; ++i) e2[i] = fmaf(L.g, o3[i + 1] + o3[i], e4[i + 1]);  // m = i - 1
#pragma unroll
    for (int i = 0; i < 2; ++i) o1[i] = fmaf(L.b, e2[i] + e2[i + 1], o3[i + 1]);   // m = i - 1
    return fmaf(L.a, o1[1] + o1[0], e2[1]);
  }
};

// causal D4 (eq. (17), reading R-D1): e1 = c / K1, o2 = d / K2, o1_k = o2_{k+1} - e1_{k+1},
// e_k = e1_k - c1 o1_k - c2 o1_{k-1} with o1_{k-1} = o2_k - e1_k
template <> struct Inverse<FD4> {
  typedef float T;
  static constexpr int SL = 0, SR = 1;
  __device__ __forceinline__ static float e(const float (&c)[2], const float (&d)[2], const Lift&) {
    const float ik1 = (float)(1.0 / kD4K1), ik2 = (float)(1.0 / kD4K2);
    const float e1k = ik1 * c[0], e1n = ik1 * c[1];
    const float o1k = fmaf(ik2, d[1], -e1n), o1m = fmaf(ik2, d[0], -e1k);
    return fmaf(-(float)kD4c2, o1m, fmaf(-(float)kD4c1, o1k, e1k));
  }
};

// reversible integer 5/3 (reading R-INT): o_k = d_k + ((c_k + c_{k+1} + 2) >> 2);
// e_k = c_k - ((o_k + o_{k-1}) >> 1)  -- the exact inverse of the received program
template <> struct Inverse<FI53> {
  typedef int T;
  static constexpr int SL = 1, SR = 1;
  __device__ __forceinline__ static int e(const int (&c)[3], const int (&d)[3], const Lift&) {
    const int ok = d[1] + ((c[1] + c[2] + 2) >> 2);
    const int om = d[0] + ((c[0] + c[1] + 2) >> 2);
    return c[1] - ((ok + om) >> 1);
  }
};

__host__ __device__ inline void inverse_reach(int fam, int& sl, int& sr) {
  switch (fam) {
    case F97: sl = 2; sr = 2; break;
    case FD4: sl = 0; sr = 1; break;
    default:  sl = 1; sr = 1; break;
  }
}

// Reach of one level in units of the level stride h = 2^{s-1}: the approximation at
// tau reads U over [tau - lowL h, tau + lowR h]; the detail over [tau - hiL h, tau + hiR h].
struct Reach { int lowL, lowR, hiL, hiR; };
__host__ __device__ inline Reach dual_reach(int fam) {
  switch (fam) {
    case F97: return {3, 3, 3, 5};
    case FD4: return {3, 0, 3, 0};
    default:  return {1, 1, 1, 3};   // 5/3 and integer 5/3
  }
}

// Analysis (template) program supports, as Mallat ranges: out[k] depends on
// in[2k - m] for m in [lLo, lHi] (approximation) / [hLo, hHi] (detail); obtained
// from the dependency structure of the analysis lifting programs.
struct Supp { int lLo, lHi, hLo, hHi; };
__host__ __device__ inline Supp analysis_support(int fam) {
  switch (fam) {
    case F97: return {-4, 4, -4, 2};
    case FD4: return {0, 3, 0, 3};
    default:  return {-2, 2, -2, 0};
  }
}

}  // namespace sidwt
