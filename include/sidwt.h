/*
 * sidwt.h -- C ABI of libsidwt: SIDWT-domain multiresolution correlation of
 * complex radar range lines by lifting, B200 (sm_100a) implementation of the
 * hot path of C. Bhattacharya & P.R. Mahapatra, "A Novel Application of
 * Lifting Scheme for Multiresolution Correlation of Complex Radar Signals"
 * (arXiv cs/0607001).  Citations "PAPER.md:L" are lines of the paper text.
 *
 * What is computed (DESIGN.md section 1 gives every reading in full):
 *   Each received row y (N complex samples) is extended once (periodic, or
 *   whole-sample symmetric about 0 and N-1) and decomposed by the dual-analysis
 *   lifting program of the chosen family at EVERY fine-grid position and every
 *   level s = 1..J.  This is the paper's even/odd-shift SIDWT tree (PAPER.md:
 *   65-73, 276-282, Fig. 1/5) with branch r, coefficient k stored at
 *   tau = r + 2^s k.  It yields detail bands W_1..W_J and the approximation
 *   band U_J.  The template x (T samples, zero outside [0,T)) is decomposed
 *   critically sampled by the analysis lifting program ("stored"):
 *   b_1..b_J, a_J.  The correlation at scale s = 0..J and lag tau in [0,N) is
 *   the eq. (4) sum over the levels coarser than s:
 *       corr_J[tau] = sum_k conj(a_J[k]) U_J[tau + 2^J k]
 *       corr_s[tau] = corr_{s+1}[tau] + sum_k conj(b_{s+1}[k]) W_{s+1}[tau + 2^{s+1} k]
 *   corr_0 equals the textbook correlation sum_n conj(x[n]) ybar[n + tau];
 *   corr_s = < (scale-s approximation of x), (scale-s dual approximation of
 *   the row shifted by tau) > (eq. (5),(15),(20),(20a), PAPER.md:75-85,141-145,
 *   284-290).  Complex signals are the linear sum of real SIDWTs of Re and Im
 *   (PAPER.md:296, 322); the analytic factor 2 of eq. (19) is omitted.
 *
 * Families (lifting programs, section III):
 *   SIDWT_LEGALL53      LeGall 5/3, PAPER.md:187-213 (dual program PAPER.md:211)
 *   SIDWT_CDF97         CDF 9/7 with Table I's rational parameters (t = 5/4),
 *                       PAPER.md:215-244 (reading R-D3 of the garbled grids); any t
 *                       of the paper's family, incl. the irrational CDF 9/7, via
 *                       sidwt_plan_set_lifting_t
 *   SIDWT_DAUB4_CAUSAL  causal Daubechies-4, eq. (17)
 *                       (readings R-D1: pairs (x[2k], x[2k-1]); R-D2)
 *   SIDWT_LEGALL53_INT  reversible integer 5/3 (floor-rounded predict/update,
 *                       PAPER.md:13, 326, refs [9],[25]; reading R-INT), int16
 *                       I/Q rows, int32 coefficients, int32 wrap-around sums
 *
 * Conventions common to all calls
 *   - Device pointers are caller-owned (e.g. torch tensors' data_ptr()), 16-byte
 *     aligned.  Host pointers are caller-owned.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Every device
 *     call is stream-ordered and non-blocking; only the setup call
 *     sidwt_template_load synchronises the host (it builds the template tables).
 *     Launch failures return SIDWT_ERR_CUDA; faults inside kernels surface at
 *     the caller's next synchronisation.  No C++ exception crosses the ABI.
 *   - A plan is used by one stream at a time; it holds no global state.
 *   - Arguments are validated before any device work; on error nothing is
 *     launched and outputs are untouched.
 */
#ifndef SIDWT_H
#define SIDWT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sidwt_plan_s* sidwt_plan;

typedef enum {
    SIDWT_OK = 0,
    SIDWT_ERR_PARAM = 1,      /* bad enum, null pointer, N not a power of two >= 2   */
    SIDWT_ERR_LENGTH = 2,     /* template length T not in [1, N]       */
    SIDWT_ERR_DIMENSION = 3,  /* rows not in [1, batch], n_templates < 1             */
    SIDWT_ERR_DEPTH = 4,      /* levels < 1 or 2^levels > N, or levels > 16 */
    SIDWT_ERR_RANGE = 5,      /* size product overflows / exceeds device limits      */
    SIDWT_ERR_STATE = 6,      /* analyze/correlate before template_load              */
    SIDWT_ERR_OOM = 7,        /* device allocation failed                            */
    SIDWT_ERR_CUDA = 8        /* CUDA runtime error (launch failure, no device, ...)  */
} sidwt_status;

typedef enum {
    SIDWT_LEGALL53 = 0,
    SIDWT_CDF97 = 1,
    SIDWT_DAUB4_CAUSAL = 2,
    SIDWT_LEGALL53_INT = 3
} sidwt_filter;

typedef enum {
    SIDWT_EXT_PERIODIC = 0,   /* ybar(n) = y[n mod N]                                   */
    SIDWT_EXT_SYMMETRIC = 1   /* whole-sample symmetric about 0 and N-1 (period 2N-2)   */
} sidwt_ext;

/* Which signal carries the redundant (shift-invariant) tree (DESIGN.md R-D7):
 *  RECEIVED_TREE (default, the north star): the received row is decomposed at every shift,
 *    the template critically sampled: corr_s[tau] = < A_s x, C_s (ybar shifted by tau) >.
 *  TEMPLATE_TREE (the paper's literal orientation, eq. (20)): the
 *    template is decomposed at every shift, the received row critically sampled:
 *    corr_s[tau] = < A_s (x delayed by tau), C_s ybar >.  Equal to the default at s = 0 and
 *    at tau = 0 mod 2^s, different in between.  Float families; SIMT correlation. */
typedef enum {
    SIDWT_ORIENT_RECEIVED_TREE = 0,
    SIDWT_ORIENT_TEMPLATE_TREE = 1
} sidwt_orientation;

#define SIDWT_MAX_LEVELS 16

/* Create a plan.  filter: sidwt_filter; levels J >= 1 with 2^J <= N; N a power
 * of two >= 2; batch >= 1 is the largest `rows` any later call will pass;
 * ext: sidwt_ext.  Validation only (no device memory is touched), so it also
 * works on a machine without a GPU.  *out receives the plan. */
sidwt_status sidwt_plan_create(sidwt_plan* out, int filter, int levels, int64_t N,
                               int64_t batch, int ext);

/* Select the orientation (sidwt_orientation) before sidwt_template_load.  PARAM for an
 * unknown value or TEMPLATE_TREE with the integer family; STATE after template_load. */
sidwt_status sidwt_plan_set_orientation(sidwt_plan plan, int orientation);

/* CDF 9/7 plans: the lifting parameter t of the paper's finite-precision family
 * (PAPER.md:217-219): alpha = (1-2t)/(4(t-1)), beta = -(t-1)^2, gamma = 1/(4t(t-1)),
 * delta = t^3 - 7/4 t^2 + t, zeta = sqrt(2)/t, used by the template (analysis), the
 * received (dual) and the synthesis programs alike.  Default t = 5/4 (Table I);
 * SIDWT_CDF97_T_EXACT gives the irrational CDF 9/7 of the paper's ref. [28].  Call
 * before sidwt_template_load.  PARAM for a non-9/7 plan or t outside [0.780, 1.852]
 * (the paper's range) or |t - 1| < 1e-3 (alpha, gamma singular); STATE after
 * template_load. */
#define SIDWT_CDF97_T_EXACT 1.2301741049140007
sidwt_status sidwt_plan_set_lifting_t(sidwt_plan plan, double t);

/* Free the plan and every device buffer it owns.  NULL is accepted. */
sidwt_status sidwt_plan_destroy(sidwt_plan plan);

/* Load the template bank and build its analysis pyramid on the device.
 * host_templates: host memory, [n_templates][T] complex64 (float2: re, im) for
 * the float families, int16x2 (I, Q) for SIDWT_LEGALL53_INT.  1 <= T <= N.
 * The pyramid is computed by a device kernel in double (int64 for the integer
 * family) and stored as float2 / int2 taps; this call synchronises the device
 * once (template loading is not on the per-pulse path).  Fixes
 * sidwt_band_stride / sidwt_band_offset.  May be called again (reload). */
sidwt_status sidwt_template_load(sidwt_plan plan, const void* host_templates, int64_t T,
                                 int n_templates);
/* Errors of template_load: LENGTH / DIMENSION as above; RANGE when the plan's tiles do
 * not fit the device (the analysis lifts one shift branch per thread at the deepest
 * level, 2^(levels-1) branches in at most 512 threads, so levels <= 10 in practice;
 * shared-memory tiles of K1 / K2 over 200 KB).  All of these are detected before any
 * state changes: a rejected (re)load leaves the previously loaded template usable. */

/* Decompose rows by lifting (every level, both shift branches).
 * d_rows : device, [rows][N] complex64, or int16x2 for the integer family.
 * d_bands: device, [rows][levels+1][2][band_stride] float32 (int32 for the
 *          integer family), split-complex: plane 0 = Re, plane 1 = Im.  Band
 *          b < levels holds W_{b+1}, band `levels` holds U_J.  Fine-grid position
 *          p is stored at index p + band_offset, for p in
 *          [-band_offset, band_stride - band_offset); the whole plane is written.
 * Requires template_load (the band margins depend on the template support). */
sidwt_status sidwt_analyze(sidwt_plan plan, const void* d_rows, int64_t rows, void* d_bands,
                           void* stream);

/* Correlate bands against every loaded template at every scale and lag.
 * d_corr: device, [rows][n_templates][levels+1][N] complex64 (int32x2 for the
 *         integer family: the exact integer correlation reduced mod 2^32).
 *         Scale index s = 0 (finest, = textbook correlation) .. levels (U_J only).
 * Template banks (float families, n_templates >= 16, N a multiple of 512) form a
 * dense contraction and run on the tensor cores (tcgen05.mma): fp32 operands split
 * into bf16 hi + lo, three products (hi.hi + hi.lo + lo.hi) accumulated in fp32;
 * error ~1e-5 of the peak |corr| (the fp32 SIMT kernel: ~1e-7).  Environment
 * SIDWT_TC=0 disables this path, SIDWT_TC=1 forces it for any bank size; read at
 * template_load.  A single complex template with a long finest term (>= 128 taps; float
 * family, symmetric extension, N/64 in [16, 128] with the tiles fitting in shared memory,
 * 2^levels <= N/64) runs on the tensor
 * cores as a Toeplitz-block GEMM (the template's Toeplitz matrix against the band
 * gathered per residue class; same split precision); SIDWT_TCS=0 disables it, SIDWT_TCS=1
 * forces it for any single template that fits.  Otherwise the per-lag FP32 (INT32) SIMT
 * kernel runs. */
sidwt_status sidwt_correlate(sidwt_plan plan, const void* d_bands, int64_t rows, void* d_corr,
                             void* stream);

/* Peak search ("sample index l for maximum matching"): for every
 * (row, template, scale) the smallest lag tau in [0,N) maximising |corr|^2
 * (fp32 |.|^2 for float families; exact uint64 for the integer family).
 * d_lag: device [rows][n_templates][levels+1] int32; d_val: same shape,
 * complex64 (int32x2) value at that lag; d_val may be NULL. */
sidwt_status sidwt_peaks(sidwt_plan plan, const void* d_corr, int64_t rows, int32_t* d_lag,
                         void* d_val, void* stream);

/* Fused correlate + peaks (same outputs as sidwt_correlate followed by
 * sidwt_peaks; the peak search is folded into the correlation epilogue so
 * the correlation is not read back from HBM).  d_corr may be NULL ("peaks
 * only": nothing but lag/val is written). */
sidwt_status sidwt_correlate_peaks(sidwt_plan plan, const void* d_bands, int64_t rows,
                                   void* d_corr, int32_t* d_lag, void* d_val, void* stream);

/* The whole path on device-resident rows: sidwt_analyze then sidwt_correlate_peaks
 * (a2-a7 of the scope table), with the same outputs, bit for bit.
 * Environment SIDWT_RUN_CHUNKS=2..16 cuts the rows into chunks, the analysis of chunk
 * k+1 issued on a high-priority stream owned by the plan while the correlation + peaks
 * of chunk k run on a low-priority one (default 1 chunk: on B200 the overlap measured
 * no gain).  The call is stream-ordered on `stream` (the plan's streams are joined by
 * events before return).  d_bands: caller-owned workspace
 * as for sidwt_analyze (rows x sidwt_bands_bytes per row), overwritten; d_corr may be
 * NULL (peaks only); d_lag / d_val as for sidwt_correlate_peaks. */
sidwt_status sidwt_run(sidwt_plan plan, const void* d_rows, int64_t rows, void* d_bands, void* d_corr,
                       int32_t* d_lag, void* d_val, void* stream);

/* Fused analyze -> correlate -> peaks (single-template plans): the same outputs as
 * sidwt_analyze followed by sidwt_correlate_peaks (corr and lag/val bit-identical), but
 * the bands never leave the chip: each CTA lifts its tile of the row (plus the
 * correlation reach) in shared memory and correlates level by level.
 * d_rows as for sidwt_analyze; d_corr may be NULL (peaks only); d_lag / d_val as for
 * sidwt_correlate_peaks.  SIDWT_ERR_RANGE when the plan has no fused tiling (banks of
 * more than one template, tap tables over 1536 taps, or tiles that do not fit on chip);
 * sidwt_fused_available tells in advance. */
sidwt_status sidwt_analyze_correlate(sidwt_plan plan, const void* d_rows, int64_t rows, void* d_corr,
                                     int32_t* d_lag, void* d_val, void* stream);
/* 1 if sidwt_analyze_correlate can run for this plan, 0 if not, -1 before template_load. */
int sidwt_fused_available(sidwt_plan plan);

/* Synthesis by inverse lifting (coarse to fine, eq. (21); the
 * perfect-reconstruction property of the lifting factorisation, PAPER.md:61-63,
 * 173-179): from bands produced by sidwt_analyze, rebuild the approximation band
 * U_level (0 <= level < levels) at the fine-grid positions 0 .. N-1, using U_J and
 * W_J .. W_{level+1} and the inverse of the received (dual analysis) lifting program.
 * level 0 reconstructs the row itself (exactly, for SIDWT_LEGALL53_INT).
 * d_out: device, [rows][N] complex64, or int32x2 for the integer family.
 * Errors: DEPTH if level is outside [0, levels); STATE before template_load (the
 * band layout is fixed there; its margins include the synthesis reach). */
sidwt_status sidwt_synthesize(sidwt_plan plan, const void* d_bands, int64_t rows, int level,
                              void* d_out, void* stream);

/* End-to-end from HOST memory: copy rows host->device, analyze, correlate,
 * peaks, copy lag (and val if non-NULL) device->host, ordered on `stream`.
 * The correlation runs in its peaks-only mode (only lag / val are returned, so
 * corr is never written to HBM).  Internally pipelined over row chunks on two
 * plan-owned streams (the copy of chunk k overlaps the computation of chunk
 * k-1), joined to `stream` by events.  Uses plan-owned device buffers for
 * `batch` rows (rows, bands, lag, val), allocated on first use and reallocated
 * when a template reload grows the band stride or the bank; SIDWT_ERR_OOM if
 * they do not fit.  h_rows must be pinned for the overlap.  Returns after
 * enqueueing; synchronise `stream` before reading h_lag/h_val. */
sidwt_status sidwt_execute_host(sidwt_plan plan, const void* h_rows, int64_t rows,
                                int32_t* h_lag, void* h_val, void* stream);

/* Layout queries (valid after template_load; -1 before). */
int64_t sidwt_band_stride(sidwt_plan plan);   /* >= band_offset + N + right margin, multiple of 32 */
int64_t sidwt_band_offset(sidwt_plan plan);   /* 0 (periodic) or the left margin M_L (symmetric)    */
int64_t sidwt_bands_bytes(sidwt_plan plan, int64_t rows);
int64_t sidwt_corr_bytes(sidwt_plan plan, int64_t rows);

/* Copy the device template pyramid to host: for each template, terms
 * b_1..b_J then a_J, each `count` taps starting at coefficient index kmin
 * (kmin/count per term written to kmin[J+1], count[J+1] when non-NULL);
 * taps as float2 (int2 for the integer family), unconjugated.  host_taps may
 * be NULL to query only.  Returns the number of taps per template or -1. */
int64_t sidwt_template_taps(sidwt_plan plan, void* host_taps, int32_t* kmin, int32_t* count);

/* 1 if sidwt_correlate* of this plan run on the tensor cores as a template bank, 2 if
 * as a single-template Toeplitz-block GEMM, 0 if on the SIMT pipes, -1 before
 * template_load. */
int sidwt_uses_tensor_cores(sidwt_plan plan);

/* 1 if every tap of the loaded template bank is real (zero imaginary part, e.g. a Barker
 * code) and the SIMT correlation runs its real-template variant (2 instead of 4 FMAs per
 * complex MAC; the skipped products are exact zeros, results unchanged); 0 otherwise; -1
 * before template_load.  Environment SIDWT_REALT=0 disables the variant. */
int sidwt_template_is_real(sidwt_plan plan);

/* Number of kernel launches the last analyze / correlate / peaks / correlate_peaks
 * call enqueued (for launch accounting). */
int sidwt_last_launches(sidwt_plan plan);

const char* sidwt_status_string(sidwt_status st);

#ifdef __cplusplus
}
#endif
#endif /* SIDWT_H */
