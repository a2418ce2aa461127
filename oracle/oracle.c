/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A plain, slow, double / int64 implementation of what the SIDWT correlation
 * path of arXiv cs/0607001 computes.  Written to be checked against the paper
 * by eye; no blocking, no fusion, no reordering.  Readings of garbled or
 * silent passages are the ones listed in DESIGN.md ("Readings").
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC oracle.c -o liboracle.so -lm
 */
#include "oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

/* A filter as the coefficients of z^{-m}, m in [lo, hi]. */
typedef struct {
    int lo, hi;
    double c[24];
} filt_t;

static long imod(long a, long p) { long r = a % p; return r < 0 ? r + p : r; }
static long floordiv(long a, long b) {
    long q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
    return q;
}
static long ceildiv(long a, long b) { return -floordiv(-a, b); }
static double fget(const filt_t* f, int m) { return (m < f->lo || m > f->hi) ? 0.0 : f->c[m - f->lo]; }

/* ------------------------------------------------------------------------ */
/* Filters from the printed polynomials.                                     */
/* ------------------------------------------------------------------------ */

static void set_filt(filt_t* f, int lo, int hi, const double* v) {
    f->lo = lo; f->hi = hi;
    memset(f->c, 0, sizeof f->c);
    for (int m = lo; m <= hi; m++) f->c[m - lo] = v[m - lo];
}

/* 9/7 printed listings, read as symmetric filters listed
 * from the outermost tap to the centre tap (reading R-97L).
 * htilde[n], n = -4..4 ; h[n], n = -3..3 (coefficient of z^{-n}). */
static double ht97(int n) {
    static const double half[5] = {9.0 / 16, -6.0 / 16, -24.0 / 16, 86.0 / 16, 190.0 / 16};
    int a = n < 0 ? -n : n;
    if (a > 4) return 0.0;
    return half[4 - a] / 10.0 / sqrt(2.0);
}
static double h97(int n) {
    static const double half[4] = {-3.0 / 64, -1.0 / 32, 19.0 / 64, 18.0 / 32};
    int a = n < 0 ? -n : n;
    if (a > 3) return 0.0;
    return half[3 - a] * sqrt(2.0);
}

/* The paper's free-variable 9/7 family, t in [0.780, 1.852]:
 *   a = (-2t+1)/(4(t-1)), b = -(t-1)^2, g = 1/(4t(t-1)), d = t^3 - 7/4 t^2 + t, x = sqrt2/t.
 * t = 5/4 is Table I, whose filters are the printed listings above.
 * For any other t there are no printed filters; they are obtained here by expanding the
 * lifting factorisations -- the analysis matrix P~(z^-1) and the dual
 * P^T(z^-1), programs as in DESIGN.md reading R-D3 -- applied to unit
 * impulses: out[k] = sum_m f[m] x[2k - m] with x = delta_n gives f[2k - n]. */
static double g_t97 = 1.25;

void oracle_set_t97(double t) { g_t97 = t; }
double oracle_get_t97(void) { return g_t97; }

static void consts97(double t, double* a, double* b, double* g, double* d, double* x) {
    *a = (-2.0 * t + 1.0) / (4.0 * (t - 1.0));
    *b = -(t - 1.0) * (t - 1.0);
    *g = 1.0 / (4.0 * t * (t - 1.0));
    *d = t * t * t - 1.75 * t * t + t;
    *x = sqrt(2.0) / t;
}

/* Lifting program on pairs k = 0..n-1 (zero outside), e[k] = x[2k], o[k] = x[2k+1].
 * analysis (R-D3): o += a(e_k + e_{k+1}); e += b(o_k + o_{k-1});
 *   o += g(e_k + e_{k+1}); e += d(o_k + o_{k-1}); lowpass x e, highpass o / x.
 * dual (R-D3): e += -a(o_k + o_{k-1}); o += -b(e_k + e_{k+1});
 *   e += -g(o_k + o_{k-1}); o += -d(e_k + e_{k+1}); lowpass e / x, highpass x o. */
#define L97N 32
static void lift97_program(int role, double t, double* e, double* o) {
    double a, b, g, d, x;
    consts97(t, &a, &b, &g, &d, &x);
    double e2[L97N], o2[L97N];
#define EK(i) (((i) < 0 || (i) >= L97N) ? 0.0 : e[i])
#define OK(i) (((i) < 0 || (i) >= L97N) ? 0.0 : o[i])
    if (role == OR_ANALYSIS) {
        for (int k = 0; k < L97N; k++) o2[k] = o[k] + a * (EK(k) + EK(k + 1));
        memcpy(o, o2, sizeof o2);
        for (int k = 0; k < L97N; k++) e2[k] = e[k] + b * (OK(k) + OK(k - 1));
        memcpy(e, e2, sizeof e2);
        for (int k = 0; k < L97N; k++) o2[k] = o[k] + g * (EK(k) + EK(k + 1));
        memcpy(o, o2, sizeof o2);
        for (int k = 0; k < L97N; k++) e2[k] = e[k] + d * (OK(k) + OK(k - 1));
        memcpy(e, e2, sizeof e2);
        for (int k = 0; k < L97N; k++) { e[k] *= x; o[k] /= x; }
    } else {
        for (int k = 0; k < L97N; k++) e2[k] = e[k] - a * (OK(k) + OK(k - 1));
        memcpy(e, e2, sizeof e2);
        for (int k = 0; k < L97N; k++) o2[k] = o[k] - b * (EK(k) + EK(k + 1));
        memcpy(o, o2, sizeof o2);
        for (int k = 0; k < L97N; k++) e2[k] = e[k] - g * (OK(k) + OK(k - 1));
        memcpy(e, e2, sizeof e2);
        for (int k = 0; k < L97N; k++) o2[k] = o[k] - d * (EK(k) + EK(k + 1));
        memcpy(o, o2, sizeof o2);
        for (int k = 0; k < L97N; k++) { e[k] /= x; o[k] *= x; }
    }
#undef EK
#undef OK
}

/* Filter f[m], m in [lo, hi], of the t-family by impulse responses (n = 2*16 and 2*16+1). */
static void filter97_t(double t, int role, int which, filt_t* f) {
    int lo, hi;
    if (which == OR_LOWPASS) { lo = (role == OR_ANALYSIS) ? -4 : -3; hi = -lo; }
    else if (role == OR_ANALYSIS) { lo = -4; hi = 2; }
    else { lo = -5; hi = 3; }
    double v[24] = {0};
    for (int par = 0; par < 2; par++) {
        const int n = 2 * (L97N / 2) + par;            /* impulse position */
        double e[L97N] = {0}, o[L97N] = {0};
        if (par == 0) e[n / 2] = 1.0; else o[n / 2] = 1.0;
        lift97_program(role, t, e, o);
        for (int k = 0; k < L97N; k++) {
            const int m = 2 * k - n;
            if (m >= lo && m <= hi) v[m - lo] = (which == OR_LOWPASS) ? e[k] : o[k];
        }
    }
    set_filt(f, lo, hi, v);
}

int oracle_filter_t97(double t, int role, int which, int* lo, int* hi, double* taps) {
    filt_t f;
    if (!(t > 0.0) || t == 1.0) return -1;
    filter97_t(t, role, which, &f);
    *lo = f.lo; *hi = f.hi;
    for (int m = f.lo; m <= f.hi; m++) taps[m - f.lo] = f.c[m - f.lo];
    return 0;
}

/* Daubechies-4 closed form (textbook, ref [1]/[11]):
 * h0..h3 = (1+sqrt3, 3+sqrt3, 3-sqrt3, 1-sqrt3) / (4 sqrt2). */
static double hd4(int n) {
    const double r3 = sqrt(3.0), d = 4.0 * sqrt(2.0);
    switch (n) {
        case 0: return (1.0 + r3) / d;
        case 1: return (3.0 + r3) / d;
        case 2: return (3.0 - r3) / d;
        case 3: return (1.0 - r3) / d;
    }
    return 0.0;
}

/* Mallat filter f (out[k] = sum_m f[m] v[2k-m]) for (family, role, which). */
static int get_filter(int family, int role, int which, filt_t* f) {
    if (family == OR_LEGALL53 || family == OR_LEGALL53_INT) {
        if (role == OR_ANALYSIS) {
            /* PAPER.md:189  ht(z^-1) = -1/8 z^2 + 1/4 z + 3/4 + 1/4 z^-1 - 1/8 z^-2 */
            static const double lp[5] = {-1.0 / 8, 1.0 / 4, 3.0 / 4, 1.0 / 4, -1.0 / 8};
            /* PAPER.md:191  gt(z^-1) = -1/4 z^2 + 1/2 z - 1/4 */
            static const double hp[3] = {-1.0 / 4, 1.0 / 2, -1.0 / 4};
            if (which == OR_LOWPASS) set_filt(f, -2, 2, lp); else set_filt(f, -2, 0, hp);
        } else {
            /* Dual analysis P^T(z^-1) (eq. 12) of the synthesis
             * matrix scaled by 2: filters 2 h(z^-1), 2 g(z^-1), i.e.
             * f[m] = 2 h[-m] with the printed synthesis filters
             *   h(z) = 1/4 z + 1/2 + 1/4 z^-1                 (h[n], n=-1..1)
             *   g(z) = -1/8 z - 1/4 + 3/4 z^-1 - 1/4 z^-2 - 1/8 z^-3 (n=-1..3). */
            static const double h[3] = {1.0 / 4, 1.0 / 2, 1.0 / 4};
            static const double g[5] = {-1.0 / 8, -1.0 / 4, 3.0 / 4, -1.0 / 4, -1.0 / 8};
            double v[8];
            if (which == OR_LOWPASS) {
                for (int m = -1; m <= 1; m++) v[m + 1] = 2.0 * h[-m + 1];
                set_filt(f, -1, 1, v);
            } else {
                for (int m = -3; m <= 1; m++) v[m + 3] = 2.0 * g[-m + 1];
                set_filt(f, -3, 1, v);
            }
        }
        return 0;
    }
    if (family == OR_CDF97 && g_t97 != 1.25) {       /* another t: from the lifting factorisation */
        filter97_t(g_t97, role, which, f);
        return 0;
    }
    if (family == OR_CDF97) {
        double v[12];
        if (which == OR_LOWPASS) {
            /* analysis: ht(z^-1), f[m] = ht[-m] (symmetric); dual: h(z^-1), f[m] = h[-m]. */
            if (role == OR_ANALYSIS) { for (int m = -4; m <= 4; m++) v[m + 4] = ht97(-m); set_filt(f, -4, 4, v); }
            else                     { for (int m = -3; m <= 3; m++) v[m + 3] = h97(-m);  set_filt(f, -3, 3, v); }
        } else {
            /* Eq. (7): gt(z) = z^-1 h(-z^-1)  =>  gt(z^-1) = z h(-z),
             *   analysis highpass f[m] = (-1)^(m+1) h[m+1], m = -4..2;
             * ht(z) = -z^-1 g(-z^-1)  =>  g(z^-1) = z ht(-z),
             *   dual highpass f[m] = (-1)^(m+1) ht[m+1], m = -5..3. */
            if (role == OR_ANALYSIS) {
                for (int m = -4; m <= 2; m++) v[m + 4] = (((m + 1) & 1) ? -1.0 : 1.0) * h97(m + 1);
                set_filt(f, -4, 2, v);
            } else {
                for (int m = -5; m <= 3; m++) v[m + 5] = (((m + 1) & 1) ? -1.0 : 1.0) * ht97(m + 1);
                set_filt(f, -5, 3, v);
            }
        }
        return 0;
    }
    if (family == OR_DAUB4) {
        /* PAPER.md:161  ht(z^-1) = h0 + h1 z^-1 + h2 z^-2 + h3 z^-3
         * PAPER.md:163  gt'(z^-1) = -h3 + h2 z^-1 - h1 z^-2 + h0 z^-3  (causal)
         * PAPER.md:181  the same filters serve the received signal (orthogonal). */
        double v[4];
        if (which == OR_LOWPASS) { for (int m = 0; m < 4; m++) v[m] = hd4(m); }
        else { v[0] = -hd4(3); v[1] = hd4(2); v[2] = -hd4(1); v[3] = hd4(0); }
        set_filt(f, 0, 3, v);
        (void)role;
        return 0;
    }
    return -1;
}

int oracle_filter(int family, int role, int which, int* lo, int* hi, double* taps) {
    filt_t f;
    if (get_filter(family, role, which, &f)) return -1;
    *lo = f.lo; *hi = f.hi;
    for (int m = f.lo; m <= f.hi; m++) taps[m - f.lo] = f.c[m - f.lo];
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Supports of the critically sampled template pyramid (zero outside [0,T)). */
/* ------------------------------------------------------------------------ */
int oracle_support(int family, int T, int s, int which, int* kmin, int* kmax) {
    filt_t lp, hp;
    if (s < 1 || T < 1) return -1;
    if (get_filter(family, OR_ANALYSIS, OR_LOWPASS, &lp) || get_filter(family, OR_ANALYSIS, OR_HIGHPASS, &hp)) return -1;
    long lo = 0, hi = T - 1;
    for (int l = 1; l < s; l++) {
        long nlo = ceildiv(lo + lp.lo, 2), nhi = floordiv(hi + lp.hi, 2);
        lo = nlo; hi = nhi;
    }
    const filt_t* f = (which == OR_LOWPASS) ? &lp : &hp;
    *kmin = (int)ceildiv(lo + f->lo, 2);
    *kmax = (int)floordiv(hi + f->hi, 2);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* One Mallat level on a P-periodic sequence.              */
/* ------------------------------------------------------------------------ */
static int out_period(int P) { return (P % 2 == 0) ? P / 2 : P; }

static void mallat_periodic(const filt_t* f, const cplx* v, int P, cplx* out) {
    int Po = out_period(P);
    for (int k = 0; k < Po; k++) {
        cplx s = 0;
        for (int m = f->lo; m <= f->hi; m++) s += fget(f, m) * v[imod(2L * k - m, P)];
        out[k] = s;
    }
}

int oracle_mallat_level(int family, int role, int P, const double* v, double* c, double* d) {
    filt_t lp, hp;
    if (P < 1 || get_filter(family, role, OR_LOWPASS, &lp) || get_filter(family, role, OR_HIGHPASS, &hp)) return -1;
    mallat_periodic(&lp, (const cplx*)v, P, (cplx*)c);
    mallat_periodic(&hp, (const cplx*)v, P, (cplx*)d);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Reversible integer 5/3 (reading R-INT; refs [9],[25]). */
/* floor division written out (no reliance on shift semantics).              */
/* ------------------------------------------------------------------------ */
static int64_t fdiv64(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
    return q;
}

int oracle_int_level(int role, int P, const int64_t* v, int64_t* c, int64_t* d) {
    if (P < 1) return -1;
    int Po = out_period(P);
    int64_t* e = (int64_t*)malloc(sizeof(int64_t) * Po);
    int64_t* o = (int64_t*)malloc(sizeof(int64_t) * Po);
    for (int k = 0; k < Po; k++) { e[k] = v[imod(2L * k, P)]; o[k] = v[imod(2L * k + 1, P)]; }
    if (role == OR_DUAL) {
        /* received: e += floor((o_k + o_{k-1})/2) ; o -= floor((e_k + e_{k+1} + 2)/4) */
        for (int k = 0; k < Po; k++) c[k] = e[k] + fdiv64(o[k] + o[imod(k - 1, Po)], 2);
        for (int k = 0; k < Po; k++) d[k] = o[k] - fdiv64(c[k] + c[imod(k + 1, Po)] + 2, 4);
    } else {
        /* template: o -= floor((e_k + e_{k+1})/2) ; e += floor((o_{k-1} + o_k + 2)/4) */
        for (int k = 0; k < Po; k++) d[k] = o[k] - fdiv64(e[k] + e[imod(k + 1, Po)], 2);
        for (int k = 0; k < Po; k++) c[k] = e[k] + fdiv64(d[imod(k - 1, Po)] + d[k] + 2, 4);
    }
    free(e); free(o);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Template pyramid (critically sampled, zero-extended template, O3).        */
/* ------------------------------------------------------------------------ */
typedef struct {
    int J;
    int alo[20], ahi[20];   /* a_s support, s = 0..J */
    int blo[20], bhi[20];   /* b_s support, s = 1..J */
    cplx* a[20];            /* float families */
    cplx* b[20];
    int64_t* ai[20][2];     /* integer family: [s][re/im] */
    int64_t* bi[20][2];
} pyr_t;

static void pyr_free(pyr_t* p) {
    for (int s = 0; s <= p->J; s++) {
        free(p->a[s]); free(p->b[s]);
        for (int q = 0; q < 2; q++) { free(p->ai[s][q]); free(p->bi[s][q]); }
    }
}

static int build_pyramid(int family, int J, int T, const void* x, pyr_t* p) {
    memset(p, 0, sizeof *p);
    p->J = J;
    p->alo[0] = 0; p->ahi[0] = T - 1;
    if (family != OR_LEGALL53_INT) {
        filt_t lp, hp;
        get_filter(family, OR_ANALYSIS, OR_LOWPASS, &lp);
        get_filter(family, OR_ANALYSIS, OR_HIGHPASS, &hp);
        p->a[0] = (cplx*)malloc(sizeof(cplx) * T);
        memcpy(p->a[0], x, sizeof(cplx) * T);
        for (int s = 1; s <= J; s++) {
            int lo = p->alo[s - 1], hi = p->ahi[s - 1];
            const cplx* prev = p->a[s - 1];
            const filt_t* fs[2] = {&lp, &hp};
            for (int w = 0; w < 2; w++) {
                const filt_t* f = fs[w];
                int klo = (int)ceildiv(lo + f->lo, 2), khi = (int)floordiv(hi + f->hi, 2);
                cplx* out = (cplx*)calloc((size_t)(khi - klo + 1), sizeof(cplx));
                for (int k = klo; k <= khi; k++) {
                    cplx acc = 0;
                    for (int m = f->lo; m <= f->hi; m++) {
                        long n = 2L * k - m;
                        if (n >= lo && n <= hi) acc += fget(f, m) * prev[n - lo];
                    }
                    out[k - klo] = acc;
                }
                if (w == 0) { p->a[s] = out; p->alo[s] = klo; p->ahi[s] = khi; }
                else        { p->b[s] = out; p->blo[s] = klo; p->bhi[s] = khi; }
            }
        }
        return 0;
    }
    /* integer family: JPEG2000-style reversible analysis lifting on the
     * zero-extended template, Re and Im independently. */
    const int16_t* xi = (const int16_t*)x;
    for (int q = 0; q < 2; q++) {
        p->ai[0][q] = (int64_t*)malloc(sizeof(int64_t) * T);
        for (int n = 0; n < T; n++) p->ai[0][q][n] = xi[2 * n + q];
    }
    for (int s = 1; s <= J; s++) {
        int lo = p->alo[s - 1], hi = p->ahi[s - 1];
        /* linear supports of the 5/3 analysis filters: lowpass m -2..2, highpass -2..0 */
        int alo = (int)ceildiv(lo - 2, 2), ahi = (int)floordiv(hi + 2, 2);
        int blo = (int)ceildiv(lo - 2, 2), bhi = (int)floordiv(hi, 2);
        int klo = alo - 1, khi = ahi + 1;           /* work range with zero padding */
        int nk = khi - klo + 1;
        for (int q = 0; q < 2; q++) {
            const int64_t* prev = p->ai[s - 1][q];
            int64_t* e = (int64_t*)calloc(nk + 2, sizeof(int64_t));
            int64_t* o = (int64_t*)calloc(nk + 2, sizeof(int64_t));
            int64_t* d = (int64_t*)calloc(nk + 2, sizeof(int64_t));
            int64_t* c = (int64_t*)calloc(nk + 2, sizeof(int64_t));
#define AT(arr, k) (arr)[(k) - klo + 1]
            for (int k = klo - 1; k <= khi + 1; k++) {
                long n0 = 2L * k, n1 = 2L * k + 1;
                AT(e, k) = (n0 >= lo && n0 <= hi) ? prev[n0 - lo] : 0;
                AT(o, k) = (n1 >= lo && n1 <= hi) ? prev[n1 - lo] : 0;
            }
            for (int k = klo - 1; k <= khi; k++) AT(d, k) = AT(o, k) - fdiv64(AT(e, k) + AT(e, k + 1), 2);
            for (int k = klo; k <= khi; k++) AT(c, k) = AT(e, k) + fdiv64(AT(d, k - 1) + AT(d, k) + 2, 4);
            p->ai[s][q] = (int64_t*)calloc(ahi - alo + 1, sizeof(int64_t));
            p->bi[s][q] = (int64_t*)calloc(bhi - blo + 1, sizeof(int64_t));
            for (int k = alo; k <= ahi; k++) p->ai[s][q][k - alo] = AT(c, k);
            for (int k = blo; k <= bhi; k++) p->bi[s][q][k - blo] = AT(d, k);
#undef AT
            free(e); free(o); free(d); free(c);
        }
        p->alo[s] = alo; p->ahi[s] = ahi; p->blo[s] = blo; p->bhi[s] = bhi;
    }
    return 0;
}

int oracle_template_pyramid(int family, int J, int T, const void* x, void* out) {
    pyr_t p;
    if (J < 1 || T < 1) return -1;
    build_pyramid(family, J, T, x, &p);
    int n = 0;
    for (int s = 1; s <= J + 1; s++) {
        int isA = (s == J + 1), lev = isA ? J : s;
        int lo = isA ? p.alo[lev] : p.blo[lev], hi = isA ? p.ahi[lev] : p.bhi[lev];
        for (int k = lo; k <= hi; k++, n++) {
            if (family != OR_LEGALL53_INT) {
                ((cplx*)out)[n] = isA ? p.a[lev][k - lo] : p.b[lev][k - lo];
            } else {
                for (int q = 0; q < 2; q++)
                    ((int64_t*)out)[2 * n + q] = isA ? p.ai[lev][q][k - lo] : p.bi[lev][q][k - lo];
            }
        }
    }
    pyr_free(&p);
    return n;
}

/* ------------------------------------------------------------------------ */
/* Received signal: extension (O1) and the even/odd SIDWT tree (O4).         */
/* ------------------------------------------------------------------------ */

/* whole-sample symmetric (about 0 and N-1) or periodic extension of y */
static long ext_index(int ext, int N, long n) {
    if (ext == OR_PERIODIC || N == 1) return imod(n, N);
    long m = imod(n, 2L * N - 2);
    return m < N ? m : 2L * N - 2 - m;
}

/* Level-s tree storage: 2^s branches of period P; branch r at offset r*P. */
typedef struct {
    int s, P;
    cplx* c;        /* float families */
    int64_t* ci[2]; /* integer family, re/im */
} level_t;

static cplx band_at(const cplx* arr, int s, int P, long p) {
    long r = imod(p, 1L << s);
    long k = floordiv(p - r, 1L << s);
    return arr[r * P + imod(k, P)];
}
static int64_t band_at_i(const int64_t* arr, int s, int P, long p) {
    long r = imod(p, 1L << s);
    long k = floordiv(p - r, 1L << s);
    return arr[r * P + imod(k, P)];
}

/* One float row, all templates. */
static void run_row_float(int family, int J, int ext, int N, const cplx* y, int T, int n_t,
                          const pyr_t* pyr, int p_lo, int p_hi, cplx* bands, cplx* corr,
                          int32_t* lag, cplx* val) {
    filt_t lp, hp;
    get_filter(family, OR_DUAL, OR_LOWPASS, &lp);
    get_filter(family, OR_DUAL, OR_HIGHPASS, &hp);
    long nb = p_hi - p_lo;
    int P = (ext == OR_PERIODIC) ? N : (N == 1 ? 1 : 2 * N - 2);
    cplx* cur = (cplx*)malloc(sizeof(cplx) * P);
    for (int n = 0; n < P; n++) cur[n] = y[ext_index(ext, N, n)];
    cplx* cs = (cplx*)calloc((size_t)n_t * (J + 1) * N, sizeof(cplx));   /* corr_s */

    for (int s = 0; s <= J; s++) {
        if (s > 0) {
            /* build level s from level s-1 (branches of period P) */
            int Po = out_period(P);
            long nbr = 1L << (s - 1);
            cplx* nxt = (cplx*)malloc(sizeof(cplx) * (size_t)(2 * nbr) * Po);
            cplx* det = (cplx*)malloc(sizeof(cplx) * (size_t)(2 * nbr) * Po);
            cplx* vplus = (cplx*)malloc(sizeof(cplx) * P);
            for (long r = 0; r < nbr; r++) {
                const cplx* v = cur + r * P;
                /* even child r: DWT of v ; odd child r + 2^{s-1}: DWT of v+[k] = v[k+1] */
                mallat_periodic(&lp, v, P, nxt + r * Po);
                mallat_periodic(&hp, v, P, det + r * Po);
                for (int k = 0; k < P; k++) vplus[k] = v[imod(k + 1, P)];
                mallat_periodic(&lp, vplus, P, nxt + (r + nbr) * Po);
                mallat_periodic(&hp, vplus, P, det + (r + nbr) * Po);
            }
            free(vplus);
            free(cur);
            cur = nxt;
            P = Po;
            if (bands)
                for (long p = p_lo; p < p_hi; p++) bands[(long)(s - 1) * nb + (p - p_lo)] = band_at(det, s, P, p);
            free(det);
        }
        if (s == J && bands)
            for (long p = p_lo; p < p_hi; p++) bands[(long)J * nb + (p - p_lo)] = band_at(cur, s, P, p);
        /* O5: corr_s[tau] = sum_k conj(a_s[k]) U_s[tau + 2^s k]  (approximation domain) */
        for (int t = 0; t < n_t; t++) {
            const pyr_t* py = &pyr[t];
            for (long tau = 0; tau < N; tau++) {
                cplx acc = 0;
                for (int k = py->alo[s]; k <= py->ahi[s]; k++)
                    acc += conj(py->a[s][k - py->alo[s]]) * band_at(cur, s, P, tau + (1L << s) * k);
                cs[((long)t * (J + 1) + s) * N + tau] = acc;
            }
        }
    }
    free(cur);
    for (int t = 0; t < n_t; t++)
        for (int s = 0; s <= J; s++) {
            const cplx* c = cs + ((long)t * (J + 1) + s) * N;
            if (corr) memcpy(corr + ((long)t * (J + 1) + s) * N, c, sizeof(cplx) * N);
            /* O6: smallest tau attaining max |corr|^2 */
            long best = 0; double bv = -1.0;
            for (long tau = 0; tau < N; tau++) {
                double m = creal(c[tau]) * creal(c[tau]) + cimag(c[tau]) * cimag(c[tau]);
                if (m > bv) { bv = m; best = tau; }
            }
            if (lag) lag[t * (J + 1) + s] = (int32_t)best;
            if (val) val[t * (J + 1) + s] = c[best];
        }
    free(cs);
}

static int32_t wrap32(int64_t v) { return (int32_t)(uint32_t)(uint64_t)v; }

/* One integer row, all templates (telescoped exact correlation, eq. (4)). */
static void run_row_int(int J, int ext, int N, const int16_t* y, int n_t, const pyr_t* pyr,
                        int p_lo, int p_hi, int64_t* bands, int32_t* corr, int32_t* lag, int32_t* val) {
    long nb = p_hi - p_lo;
    int P = (ext == OR_PERIODIC) ? N : (N == 1 ? 1 : 2 * N - 2);
    int64_t* cur[2];
    for (int q = 0; q < 2; q++) {
        cur[q] = (int64_t*)malloc(sizeof(int64_t) * P);
        for (int n = 0; n < P; n++) cur[q][n] = y[2 * ext_index(ext, N, n) + q];
    }
    /* D[t][i][tau] (i = 1..J) and A[t][tau], exact */
    int64_t* D = (int64_t*)calloc((size_t)n_t * (J + 2) * N * 2, sizeof(int64_t));
#define DI(t, i, tau, q) D[((((long)(t) * (J + 2) + (i)) * N) + (tau)) * 2 + (q)]
    for (int s = 1; s <= J; s++) {
        int Po = out_period(P);
        long nbr = 1L << (s - 1);
        int64_t* nxt[2];
        int64_t* det[2];
        int64_t* vplus = (int64_t*)malloc(sizeof(int64_t) * P);
        for (int q = 0; q < 2; q++) {
            nxt[q] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * nbr) * Po);
            det[q] = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * nbr) * Po);
            for (long r = 0; r < nbr; r++) {
                const int64_t* v = cur[q] + r * P;
                oracle_int_level(OR_DUAL, P, v, nxt[q] + r * Po, det[q] + r * Po);
                for (int k = 0; k < P; k++) vplus[k] = v[imod(k + 1, P)];
                oracle_int_level(OR_DUAL, P, vplus, nxt[q] + (r + nbr) * Po, det[q] + (r + nbr) * Po);
            }
            free(cur[q]);
            cur[q] = nxt[q];
        }
        free(vplus);
        P = Po;
        if (bands)
            for (long p = p_lo; p < p_hi; p++)
                for (int q = 0; q < 2; q++)
                    bands[((long)(s - 1) * nb + (p - p_lo)) * 2 + q] = band_at_i(det[q], s, P, p);
        /* D_s[tau] = sum_k conj(b_s[k]) W_s[tau + 2^s k] */
        for (int t = 0; t < n_t; t++) {
            const pyr_t* py = &pyr[t];
            for (long tau = 0; tau < N; tau++) {
                int64_t re = 0, im = 0;
                for (int k = py->blo[s]; k <= py->bhi[s]; k++) {
                    int64_t br = py->bi[s][0][k - py->blo[s]], bi = py->bi[s][1][k - py->blo[s]];
                    long p = tau + (1L << s) * k;
                    int64_t wr = band_at_i(det[0], s, P, p), wi = band_at_i(det[1], s, P, p);
                    re += br * wr + bi * wi;
                    im += br * wi - bi * wr;
                }
                DI(t, s, tau, 0) = re; DI(t, s, tau, 1) = im;
            }
        }
        for (int q = 0; q < 2; q++) free(det[q]);
    }
    if (bands)
        for (long p = p_lo; p < p_hi; p++)
            for (int q = 0; q < 2; q++)
                bands[((long)J * nb + (p - p_lo)) * 2 + q] = band_at_i(cur[q], J, P, p);
    for (int t = 0; t < n_t; t++) {
        const pyr_t* py = &pyr[t];
        for (long tau = 0; tau < N; tau++) {
            int64_t re = 0, im = 0;
            for (int k = py->alo[J]; k <= py->ahi[J]; k++) {
                int64_t ar = py->ai[J][0][k - py->alo[J]], ai = py->ai[J][1][k - py->alo[J]];
                long p = tau + (1L << J) * k;
                int64_t ur = band_at_i(cur[0], J, P, p), ui = band_at_i(cur[1], J, P, p);
                re += ar * ur + ai * ui;
                im += ar * ui - ai * ur;
            }
            DI(t, J + 1, tau, 0) = re; DI(t, J + 1, tau, 1) = im;   /* A_J */
        }
        /* corr_J = A_J ; corr_s = A_J + sum_{i=s+1..J} D_i ; exact, then mod 2^32 */
        for (int s = 0; s <= J; s++) {
            int32_t* cc = corr ? corr + (((long)t * (J + 1) + s) * N) * 2 : NULL;
            long best = 0; uint64_t bv = 0; int first = 1;
            int32_t bre = 0, bim = 0;
            for (long tau = 0; tau < N; tau++) {
                int64_t re = DI(t, J + 1, tau, 0), im = DI(t, J + 1, tau, 1);
                for (int i = s + 1; i <= J; i++) { re += DI(t, i, tau, 0); im += DI(t, i, tau, 1); }
                int32_t r32 = wrap32(re), i32 = wrap32(im);
                if (cc) { cc[2 * tau] = r32; cc[2 * tau + 1] = i32; }
                uint64_t m = (uint64_t)((int64_t)r32 * r32) + (uint64_t)((int64_t)i32 * i32);
                if (first || m > bv) { bv = m; best = tau; bre = r32; bim = i32; first = 0; }
            }
            if (lag) lag[t * (J + 1) + s] = (int32_t)best;
            if (val) { val[2 * (t * (J + 1) + s)] = bre; val[2 * (t * (J + 1) + s) + 1] = bim; }
        }
    }
#undef DI
    for (int q = 0; q < 2; q++) free(cur[q]);
    free(D);
}

/* Approximation band U_s (s = 0..J) of one row at fine-grid positions [p_lo, p_hi), by the
 * same even/odd tree (O4) as oracle_run; U_0 is the extended row (O1).  Used to check the
 * GPU synthesis (inverse lifting, eq. (21)) against the forward tree. */
static void approx_row_float(int family, int ext, int N, const cplx* y, int s, int p_lo, int p_hi, cplx* out) {
    filt_t lp;
    get_filter(family, OR_DUAL, OR_LOWPASS, &lp);
    int P = (ext == OR_PERIODIC) ? N : (N == 1 ? 1 : 2 * N - 2);
    cplx* cur = (cplx*)malloc(sizeof(cplx) * P);
    for (int n = 0; n < P; n++) cur[n] = y[ext_index(ext, N, n)];
    for (int l = 1; l <= s; l++) {
        int Po = out_period(P);
        long nbr = 1L << (l - 1);
        cplx* nxt = (cplx*)malloc(sizeof(cplx) * (size_t)(2 * nbr) * Po);
        cplx* vplus = (cplx*)malloc(sizeof(cplx) * P);
        for (long r = 0; r < nbr; r++) {
            const cplx* v = cur + r * P;
            mallat_periodic(&lp, v, P, nxt + r * Po);
            for (int k = 0; k < P; k++) vplus[k] = v[imod(k + 1, P)];
            mallat_periodic(&lp, vplus, P, nxt + (r + nbr) * Po);
        }
        free(vplus);
        free(cur);
        cur = nxt;
        P = Po;
    }
    for (long p = p_lo; p < p_hi; p++) out[p - p_lo] = band_at(cur, s, P, p);
    free(cur);
}

static void approx_row_int(int ext, int N, const int16_t* y, int s, int p_lo, int p_hi, int64_t* out) {
    int P = (ext == OR_PERIODIC) ? N : (N == 1 ? 1 : 2 * N - 2);
    for (int q = 0; q < 2; q++) {
        int Pq = P;
        int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * Pq);
        for (int n = 0; n < Pq; n++) cur[n] = y[2 * ext_index(ext, N, n) + q];
        for (int l = 1; l <= s; l++) {
            int Po = out_period(Pq);
            long nbr = 1L << (l - 1);
            int64_t* nxt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * nbr) * Po);
            int64_t* det = (int64_t*)malloc(sizeof(int64_t) * (size_t)Po);
            int64_t* vplus = (int64_t*)malloc(sizeof(int64_t) * Pq);
            for (long r = 0; r < nbr; r++) {
                const int64_t* v = cur + r * Pq;
                oracle_int_level(OR_DUAL, Pq, v, nxt + r * Po, det);
                for (int k = 0; k < Pq; k++) vplus[k] = v[imod(k + 1, Pq)];
                oracle_int_level(OR_DUAL, Pq, vplus, nxt + (r + nbr) * Po, det);
            }
            free(vplus);
            free(det);
            free(cur);
            cur = nxt;
            Pq = Po;
        }
        for (long p = p_lo; p < p_hi; p++) out[(p - p_lo) * 2 + q] = band_at_i(cur, s, Pq, p);
        free(cur);
    }
}

int oracle_approx(int family, int ext, int N, int rows, const void* y, int s, int p_lo, int p_hi, void* out,
                  int nthreads) {
    if (family < 0 || family > 3 || N < 2 || (N & (N - 1)) || s < 0 || (1L << s) > N) return -1;
    if (ext != OR_PERIODIC && ext != OR_SYMMETRIC) return -1;
    if (rows < 0 || p_hi <= p_lo) return -1;
    long nb = p_hi - p_lo;
    if (nthreads <= 0) nthreads = oracle_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int r = 0; r < rows; r++) {
        if (family != OR_LEGALL53_INT)
            approx_row_float(family, ext, N, (const cplx*)y + (long)r * N, s, p_lo, p_hi, (cplx*)out + (long)r * nb);
        else
            approx_row_int(ext, N, (const int16_t*)y + (long)r * N * 2, s, p_lo, p_hi, (int64_t*)out + (long)r * nb * 2);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* The paper's orientation (eq. (20)):  */
/* the template carries the redundant tree, the received row is critically        */
/* sampled: corr^P_s[tau] = < A_s S_{-tau} x , C_s ybar >, with S_{-tau} x[n] =     */
/* x[n - tau] (the template delayed by tau), A_s its analysis approximation and    */
/* C_s ybar = branch 0 of the received tree (dual analysis).  Plain definition:     */
/* one Mallat pyramid of the delayed template per lag.  Float families only.        */
/* ------------------------------------------------------------------------ */
static void run_row_paper(int family, int J, int ext, int N, const cplx* y, int T, int n_t, const cplx* x,
                          cplx* corr, int32_t* lag, cplx* val) {
    filt_t lp;
    get_filter(family, OR_DUAL, OR_LOWPASS, &lp);
    int P[21];
    cplx* c[21];
    P[0] = (ext == OR_PERIODIC) ? N : (N == 1 ? 1 : 2 * N - 2);
    c[0] = (cplx*)malloc(sizeof(cplx) * P[0]);
    for (int n = 0; n < P[0]; n++) c[0][n] = y[ext_index(ext, N, n)];
    for (int s = 1; s <= J; s++) {                  /* branch 0: even child of branch 0 */
        P[s] = out_period(P[s - 1]);
        c[s] = (cplx*)malloc(sizeof(cplx) * P[s]);
        mallat_periodic(&lp, c[s - 1], P[s - 1], c[s]);
    }
    cplx* cs = (cplx*)calloc((size_t)n_t * (J + 1) * N, sizeof(cplx));
    cplx* xs = (cplx*)malloc(sizeof(cplx) * T);
    filt_t alp;
    get_filter(family, OR_ANALYSIS, OR_LOWPASS, &alp);
    for (int t = 0; t < n_t; t++) {
        memcpy(xs, x + (long)t * T, sizeof(cplx) * T);
        for (long tau = 0; tau < N; tau++) {
            /* analysis approximations a_s of the delayed template x[n - tau], support
               [tau, tau + T - 1] at level 0 (O3 on the shifted origin) */
            cplx* a[21];
            int alo[21], ahi[21];
            a[0] = xs; alo[0] = (int)tau; ahi[0] = (int)tau + T - 1;
            for (int s = 1; s <= J; s++) {
                int lo = alo[s - 1], hi = ahi[s - 1];
                int klo = (int)ceildiv(lo + alp.lo, 2), khi = (int)floordiv(hi + alp.hi, 2);
                a[s] = (cplx*)calloc((size_t)(khi - klo + 1), sizeof(cplx));
                for (int k = klo; k <= khi; k++) {
                    cplx acc = 0;
                    for (int m = alp.lo; m <= alp.hi; m++) {
                        long n = 2L * k - m;
                        if (n >= lo && n <= hi) acc += fget(&alp, m) * a[s - 1][n - lo];
                    }
                    a[s][k - klo] = acc;
                }
                alo[s] = klo; ahi[s] = khi;
            }
            for (int s = 0; s <= J; s++) {
                cplx acc = 0;
                for (int k = alo[s]; k <= ahi[s]; k++) acc += conj(a[s][k - alo[s]]) * c[s][imod(k, P[s])];
                cs[((long)t * (J + 1) + s) * N + tau] = acc;
            }
            for (int s = 1; s <= J; s++) free(a[s]);
        }
    }
    free(xs);
    for (int s = 0; s <= J; s++) free(c[s]);
    for (int t = 0; t < n_t; t++)
        for (int s = 0; s <= J; s++) {
            const cplx* cc = cs + ((long)t * (J + 1) + s) * N;
            if (corr) memcpy(corr + ((long)t * (J + 1) + s) * N, cc, sizeof(cplx) * N);
            long best = 0; double bv = -1.0;
            for (long tau = 0; tau < N; tau++) {
                double m = creal(cc[tau]) * creal(cc[tau]) + cimag(cc[tau]) * cimag(cc[tau]);
                if (m > bv) { bv = m; best = tau; }
            }
            if (lag) lag[t * (J + 1) + s] = (int32_t)best;
            if (val) val[t * (J + 1) + s] = cc[best];
        }
    free(cs);
}

int oracle_run_paper(int family, int J, int ext, int N, int rows, const void* y, int T, int n_t, const void* x,
                     void* corr, int32_t* lag, void* val, int nthreads) {
    if (family < 0 || family > 2 || J < 1 || J > 20 || N < 2 || (N & (N - 1)) || (1L << J) > N) return -1;
    if (T < 1 || T > N || n_t < 1 || rows < 0) return -1;
    if (ext != OR_PERIODIC && ext != OR_SYMMETRIC) return -1;
    if (nthreads <= 0) nthreads = oracle_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int r = 0; r < rows; r++)
        run_row_paper(family, J, ext, N, (const cplx*)y + (long)r * N, T, n_t, (const cplx*)x,
                      corr ? (cplx*)corr + (long)r * n_t * (J + 1) * N : NULL, lag ? lag + (long)r * n_t * (J + 1) : NULL,
                      val ? (cplx*)val + (long)r * n_t * (J + 1) : NULL);
    return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int oracle_run(int family, int J, int ext, int N, int rows, const void* y, int T, int n_t,
               const void* x, int p_lo, int p_hi, void* bands, void* corr, int32_t* lag, void* val,
               int nthreads) {
    if (family < 0 || family > 3 || J < 1 || N < 2 || (N & (N - 1)) || (1L << J) > N) return -1;
    if (T < 1 || T > N || n_t < 1 || rows < 0 || (bands && p_hi <= p_lo)) return -1;
    if (ext != OR_PERIODIC && ext != OR_SYMMETRIC) return -1;
    pyr_t* pyr = (pyr_t*)calloc(n_t, sizeof(pyr_t));
    int isint = (family == OR_LEGALL53_INT);
    for (int t = 0; t < n_t; t++) {
        const char* xt = (const char*)x + (size_t)t * T * (isint ? 2 * sizeof(int16_t) : sizeof(cplx));
        build_pyramid(family, J, T, xt, &pyr[t]);
    }
    long nb = p_hi - p_lo;
    if (nthreads <= 0) nthreads = oracle_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int r = 0; r < rows; r++) {
        if (!isint) {
            run_row_float(family, J, ext, N, (const cplx*)y + (long)r * N, T, n_t, pyr, p_lo, p_hi,
                          bands ? (cplx*)bands + (long)r * (J + 1) * nb : NULL,
                          corr ? (cplx*)corr + (long)r * n_t * (J + 1) * N : NULL,
                          lag ? lag + (long)r * n_t * (J + 1) : NULL,
                          val ? (cplx*)val + (long)r * n_t * (J + 1) : NULL);
        } else {
            run_row_int(J, ext, N, (const int16_t*)y + (long)r * N * 2, n_t, pyr, p_lo, p_hi,
                        bands ? (int64_t*)bands + (long)r * (J + 1) * nb * 2 : NULL,
                        corr ? (int32_t*)corr + (long)r * n_t * (J + 1) * N * 2 : NULL,
                        lag ? lag + (long)r * n_t * (J + 1) : NULL,
                        val ? (int32_t*)val + (long)r * n_t * (J + 1) * 2 : NULL);
        }
    }
    for (int t = 0; t < n_t; t++) pyr_free(&pyr[t]);
    free(pyr);
    return 0;
}
