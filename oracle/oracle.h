/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, double-precision (int64 for the reversible integer family)
 * CPU oracle of the SIDWT multiresolution correlation of arXiv cs/0607001
 * (Bhattacharya & Mahapatra).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or generator with the CUDA library (include/sidwt.h,
 * paper_cs_0607001_b200/csrc); it is built from oracle/oracle.c alone.
 *
 * Route (deliberately different from the GPU's lifting + telescoped sums):
 *   filters  : the paper's printed filter polynomials (PAPER.md:161-163,
 *              189-199, 223-225) and Eq. (7) for the 9/7 highpass
 *   transform: Mallat convolution-and-downsample on periodic
 *              branch sequences, the even/odd shift tree of Fig. 1/5
 *
 *   corr     : approximation-domain direct cross-correlation (float families),
 *              eq. (4)-telescoped exact integer correlation (integer family)
 * See DESIGN.md section "Oracle" for every reading of the paper it encodes.
 */
#ifndef SIDWT_ORACLE_H
#define SIDWT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_LEGALL53 = 0, OR_CDF97 = 1, OR_DAUB4 = 2, OR_LEGALL53_INT = 3 };
enum { OR_ANALYSIS = 0, OR_DUAL = 1 };
enum { OR_LOWPASS = 0, OR_HIGHPASS = 1 };
enum { OR_PERIODIC = 0, OR_SYMMETRIC = 1 };

/* Filter f as "coefficient of z^-m", m in [*lo, *hi]; taps[m - *lo]. Returns 0 or -1. */
int oracle_filter(int family, int role, int which, int* lo, int* hi, double* taps);

/* CDF 9/7 free parameter t (default 5/4 = Table I, printed filters).  A
 * process-wide setting read by every OR_CDF97 call: set it before a run, not concurrently. */
void oracle_set_t97(double t);
double oracle_get_t97(void);
/* The 9/7 filter of parameter t derived from the lifting factorisation (any t, including
 * 5/4, where it must reproduce the printed listings).  Returns 0 or -1. */
int oracle_filter_t97(double t, int role, int which, int* lo, int* hi, double* taps);

/* Support [kmin, kmax] of the template pyramid at level s (1..J): which = lowpass (a_s) / highpass (b_s). */
int oracle_support(int family, int T, int s, int which, int* kmin, int* kmax);

/* One Mallat level on a P-periodic complex sequence v (float families):
 * out[k] = sum_m f[m] v[(2k - m) mod P], k in [0, Pout), Pout = P/2 (P even) or P (P odd). */
int oracle_mallat_level(int family, int role, int P, const double* v /*complex*/,
                        double* c /*complex[Pout]*/, double* d /*complex[Pout]*/);

/* One integer lifting level (family OR_LEGALL53_INT) on a P-periodic int64 sequence. */
int oracle_int_level(int role, int P, const int64_t* v, int64_t* c, int64_t* d);

/* Template pyramid for one template.  Float families: x complex [T]; out
 * a_s (s = 0..J) and b_s (s = 1..J) written into `pyr` in the order
 * b_1, ..., b_J, a_J, each over its support from oracle_support (complex).
 * Integer family: x int16 pairs [T][2], pyr int64 pairs.  Returns the number
 * of complex entries written, or -1. */
int oracle_template_pyramid(int family, int J, int T, const void* x, void* pyr);

/* Full path for rows [0, rows) (OpenMP over rows, nthreads <= 0 -> default).
 *  y    : float families complex double [rows][N]; integer family int16 [rows][N][2]
 *  x    : float families complex double [n_t][T];   integer family int16 [n_t][T][2]
 *  bands: optional (NULL to skip) [rows][J+1][p_hi - p_lo] complex double (int64 pairs
 *         for the integer family); band b < J holds W_{b+1}, band J holds U_J, at
 *         fine-grid positions p in [p_lo, p_hi)
 *  corr : optional [rows][n_t][J+1][N] complex double (int32 pairs, exact mod 2^32, for int)
 *  lag  : optional [rows][n_t][J+1] int32 ; val: optional, same shape, complex double / int32 pairs
 * Returns 0, or -1 on bad arguments. */
int oracle_run(int family, int J, int ext, int N, int rows, const void* y,
               int T, int n_t, const void* x, int p_lo, int p_hi, void* bands,
               void* corr, int32_t* lag, void* val, int nthreads);

/* Approximation band U_s (s >= 0; U_0 = the extended row) at fine-grid positions
 * [p_lo, p_hi) of each row, by the tree of oracle_run.  out: [rows][p_hi - p_lo] complex
 * double (int64 pairs for the integer family).  Returns 0 or -1. */
int oracle_approx(int family, int ext, int N, int rows, const void* y, int s, int p_lo, int p_hi, void* out,
                  int nthreads);

/* The paper's orientation (template carries the redundant tree, received row critically
 * sampled; eq. (20)): corr[rows][n_t][J+1][N] of
 * < A_s (x delayed by tau), C_s ybar > and its peaks, by the plain definition (one Mallat
 * pyramid of the delayed template per lag).  Float families only; -1 otherwise. */
int oracle_run_paper(int family, int J, int ext, int N, int rows, const void* y, int T, int n_t, const void* x,
                     void* corr, int32_t* lag, void* val, int nthreads);

int oracle_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
