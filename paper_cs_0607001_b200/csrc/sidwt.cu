// sidwt.cu -- host side of libsidwt: the C ABI declared in include/sidwt.h.
// Plans, validation, template loading, layout, and launches of the sm_100a
// kernels in kernels.cuh.  No computation of the path happens on the host.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/sidwt.h"
#include "kernels.cuh"
#include "corr_tc.cuh"
#include "corr_tcs.cuh"
#include "fused.cuh"
#include "corr_i8.h"

using namespace sidwt;

namespace {

#ifndef SIDWT_KRV
#define SIDWT_KRV 15
#endif
constexpr int kRV = SIDWT_KRV;     // K1 run length (odd: bank-conflict free), fused kernel and default
// run length of the analysis kernel: 13 for deep plans (J >= 5) of the four-step 9/7 program (C3
// analyze 2.14 -> 2.05 ms; C4, J = 4, is faster at 15: 0.39 vs 0.42 ms), 15 otherwise (C5: 4.59 ms
// at 15, 4.92 at 13, 5.53 at 17; A/B with -DSIDWT_KRV)
constexpr int kRV97 = SIDWT_KRV == 15 ? 13 : kRV;
inline int rv_for(int fam, int J) { return (fam == F97 && J >= 5) ? kRV97 : kRV; }
constexpr int kQ = 9;       // K2 outputs per item (odd: bank-conflict free)
constexpr int kK2NT = 256;  // K2 threads (Q = 11 with 192 threads measured slower on C2 and C5)

constexpr int kRunChunks = 16;   // sidwt_run: analysis of chunk k+1 overlaps the correlation of chunk k
constexpr int kPipeChunks = 8;   // execute_host: host->device copy of chunk k overlaps compute of chunk k-1

inline int64_t rup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace

struct sidwt_plan_s {
  int fam = 0, J = 0, ext = 0;
  int64_t N = 0, batch = 0;
  bool loaded = false;
  int T = 0, n_t = 0;
  // template terms: i < J -> b_{i+1}, i = J -> a_J
  int kmin[kMaxTerms] = {}, cnt[kMaxTerms] = {}, npad[kMaxTerms] = {}, toff[kMaxTerms] = {};
  int taps_per_t = 0;
  int ML = 0, MR = 0;
  int64_t stride = -1;
  void* d_taps = nullptr;
  // K1 configuration
  AnaParams ana{};
  int ana_threads = 0;
  int64_t ana_threads_needed = 0;  // K1 threads the deepest level needs (> 512: plan rejected, RANGE)
  size_t ana_smem = 0;
  // K2 configuration
  CorParams cor{};
  size_t cor_smem = 0;
  // workspaces
  void* d_partials = nullptr;
  size_t partials_bytes = 0;
  // execute_host workspaces and their allocated sizes (reallocated when a template reload
  // grows the band stride or the bank)
  void *w_rows = nullptr, *w_bands = nullptr, *w_lag = nullptr, *w_val = nullptr;
  size_t w_rows_bytes = 0, w_bands_bytes = 0, w_lag_bytes = 0, w_val_bytes = 0;
  // execute_host pipeline
  cudaStream_t s_copy = nullptr, s_comp = nullptr;
  cudaEvent_t ev[10] = {};
  cudaStream_t s_k1 = nullptr, s_k2 = nullptr;   // sidwt_run: analysis (high priority) / correlation streams
  cudaEvent_t rev[kRunChunks + 2] = {};
  int last_launches = 0;
  // tensor-core bank path (corr_tc.cuh)
  bool paper = false;            // orientation: template carries the redundant tree
  bool ctaps = false;            // SIMT correlation reads the taps from its kernel parameters
  bool real_taps = false;        // every template tap has a zero imaginary part
  int run_chunks = 1;            // sidwt_run default chunk count
  int ana_rv = kRV;              // K1 run length chosen at configure
  double t97 = 1.25;             // 9/7 lifting parameter t (Table I)
  // fused analyze -> correlate -> peaks (single template)
  bool fused = false;
  FusParams* fus = nullptr;      // host copy (large: carries the taps)
  size_t fus_smem = 0;
  void* d_fpartials = nullptr;
  size_t fpartials_bytes = 0;
  bool tc = false;
  int tc_sms = 148;
  TcParams tcp{};
  void* d_img = nullptr;
  size_t tc_smem = 0;
  bool tcs = false;                  // single-template tensor-core correlation (corr_tcs.cuh)
  TcsParams tcsp{};
  void* d_tcs_img = nullptr;
  size_t tcs_smem = 0;
  int tcs_total_ksteps = 0;
  bool i8 = false;                   // integer family on the int8 tensor cores (corr_i8.cu)
  I8Params i8p{};
  void* d_i8_img = nullptr;
};

static bool is_int(const sidwt_plan_s* p) { return p->fam == SIDWT_LEGALL53_INT; }
static size_t sample_bytes(const sidwt_plan_s* p) { return is_int(p) ? 4 : 8; }

// Definitions take C linkage from the extern "C" declarations in include/sidwt.h.

const char* sidwt_status_string(sidwt_status st) {
  switch (st) {
    case SIDWT_OK: return "ok";
    case SIDWT_ERR_PARAM: return "parameter error";
    case SIDWT_ERR_LENGTH: return "length error";
    case SIDWT_ERR_DIMENSION: return "dimension error";
    case SIDWT_ERR_DEPTH: return "depth error";
    case SIDWT_ERR_RANGE: return "range error";
    case SIDWT_ERR_STATE: return "state error";
    case SIDWT_ERR_OOM: return "out of device memory";
    case SIDWT_ERR_CUDA: return "CUDA error";
  }
  return "unknown status";
}

sidwt_status sidwt_plan_create(sidwt_plan* out, int filter, int levels, int64_t N, int64_t batch, int ext) {
  if (!out) return SIDWT_ERR_PARAM;
  *out = nullptr;
  if (filter < 0 || filter > 3 || (ext != SIDWT_EXT_PERIODIC && ext != SIDWT_EXT_SYMMETRIC)) return SIDWT_ERR_PARAM;
  if (N < 2 || (N & (N - 1)) != 0) return SIDWT_ERR_PARAM;
  if (N > (int64_t(1) << 24)) return SIDWT_ERR_RANGE;
  if (levels < 1 || levels > SIDWT_MAX_LEVELS || (int64_t(1) << levels) > N) return SIDWT_ERR_DEPTH;
  if (batch < 1) return SIDWT_ERR_DIMENSION;
  sidwt_plan_s* p = new (std::nothrow) sidwt_plan_s();
  if (!p) return SIDWT_ERR_OOM;
  p->fam = filter; p->J = levels; p->N = N; p->batch = batch; p->ext = ext;
  *out = p;
  return SIDWT_OK;
}

static void free_ws(sidwt_plan_s* p) {
  void** bufs[] = {&p->d_taps, &p->d_partials, &p->w_rows, &p->w_bands, &p->w_lag, &p->w_val, &p->d_img,
                   &p->d_tcs_img, &p->d_i8_img};
  for (void** b : bufs) { if (*b) cudaFree(*b); *b = nullptr; }
  p->w_rows_bytes = p->w_bands_bytes = p->w_lag_bytes = p->w_val_bytes = 0;
  for (cudaEvent_t& ev : p->ev) { if (ev) cudaEventDestroy(ev); ev = nullptr; }
  if (p->d_fpartials) { cudaFree(p->d_fpartials); p->d_fpartials = nullptr; p->fpartials_bytes = 0; }
  delete p->fus; p->fus = nullptr;
  if (p->s_copy) { cudaStreamDestroy(p->s_copy); p->s_copy = nullptr; }
  if (p->s_comp) { cudaStreamDestroy(p->s_comp); p->s_comp = nullptr; }
  if (p->s_k2) { cudaStreamDestroy(p->s_k2); p->s_k2 = nullptr; }
  if (p->s_k1) { cudaStreamDestroy(p->s_k1); p->s_k1 = nullptr; }
  for (auto& ev : p->rev)
    if (ev) { cudaEventDestroy(ev); ev = nullptr; }
  p->partials_bytes = 0;
}

sidwt_status sidwt_plan_destroy(sidwt_plan plan) {
  if (!plan) return SIDWT_OK;
  free_ws(plan);
  delete plan;
  return SIDWT_OK;
}

sidwt_status sidwt_plan_set_lifting_t(sidwt_plan p, double t) {
  if (!p || p->fam != F97) return SIDWT_ERR_PARAM;
  if (!(t >= 0.780 && t <= 1.852) || std::fabs(t - 1.0) < 1e-3) return SIDWT_ERR_PARAM;
  if (p->loaded) return SIDWT_ERR_STATE;
  p->t97 = t;
  return SIDWT_OK;
}

sidwt_status sidwt_plan_set_orientation(sidwt_plan p, int orientation) {
  if (!p || (orientation != SIDWT_ORIENT_RECEIVED_TREE && orientation != SIDWT_ORIENT_TEMPLATE_TREE)) return SIDWT_ERR_PARAM;
  if (orientation == SIDWT_ORIENT_TEMPLATE_TREE && is_int(p)) return SIDWT_ERR_PARAM;
  if (p->loaded) return SIDWT_ERR_STATE;
  p->paper = orientation == SIDWT_ORIENT_TEMPLATE_TREE;
  return SIDWT_OK;
}

int64_t sidwt_band_stride(sidwt_plan p) { return (p && p->loaded) ? p->stride : -1; }
int64_t sidwt_band_offset(sidwt_plan p) { return (p && p->loaded) ? p->ML : -1; }
int64_t sidwt_bands_bytes(sidwt_plan p, int64_t rows) {
  if (!p || !p->loaded) return -1;
  return rows * (p->J + 1) * 2 * p->stride * 4;
}
int64_t sidwt_corr_bytes(sidwt_plan p, int64_t rows) {
  if (!p || !p->loaded) return -1;
  return rows * p->n_t * (p->J + 1) * p->N * 8;
}
int sidwt_last_launches(sidwt_plan p) { return p ? p->last_launches : 0; }
int sidwt_uses_tensor_cores(sidwt_plan p) {
  return (p && p->loaded) ? (p->tc ? 1 : (p->tcs ? 2 : (p->i8 ? 3 : 0))) : -1;
}
int sidwt_template_is_real(sidwt_plan p) { return (p && p->loaded) ? (p->real_taps ? 1 : 0) : -1; }

// ---------------------------------------------------------------------------
// Template load: supports, margins, tiling, and the device pyramid (K0).
// ---------------------------------------------------------------------------
static void k2_buffers(sidwt_plan_s* p, int Q);
static void configure(sidwt_plan_s* p) {
  const int J = p->J;
  const Supp sp = analysis_support(p->fam);
  // supports of the critically sampled pyramid (zero-extended template on [0,T)); in the
  // paper's orientation the union over the template delayed by rho = 0 .. 2^{lg} - 1
  const int nres = p->paper ? (1 << J) : 1;
  int kmin[kMaxTerms], kmax[kMaxTerms];
  for (int i = 0; i <= J; ++i) { kmin[i] = INT32_MAX; kmax[i] = INT32_MIN; }
  for (int rho = 0; rho < nres; ++rho) {
    long lo = rho, hi = rho + p->T - 1;
    for (int s = 1; s <= J; ++s) {
      const long alo = cl_div2(lo + sp.lLo), ahi = fl_div2(hi + sp.lHi);
      const long blo = cl_div2(lo + sp.hLo), bhi = fl_div2(hi + sp.hHi);
      if (rho < (1 << s)) { kmin[s - 1] = std::min<int>(kmin[s - 1], (int)blo); kmax[s - 1] = std::max<int>(kmax[s - 1], (int)bhi); }
      lo = alo; hi = ahi;
    }
    kmin[J] = std::min<int>(kmin[J], (int)lo); kmax[J] = std::max<int>(kmax[J], (int)hi);
  }
  for (int i = 0; i <= J; ++i) { p->kmin[i] = kmin[i]; p->cnt[i] = kmax[i] - kmin[i] + 1; }
  int off = 0;
  for (int i = 0; i <= J; ++i) {
    p->npad[i] = (int)rup(p->cnt[i], kQ);
    p->toff[i] = off;
    const int nr = p->paper ? (1 << (i < J ? i + 1 : J)) : 1;
    off += nr * p->npad[i];
  }
  p->taps_per_t = off;
  // correlation reach -> band margins (DESIGN.md R-D6 GPU): every band value K2 reads exists.
  int ML = 0, MR = 0;
  for (int i = 0; i <= J; ++i) {
    const int g = 1 << (i < J ? i + 1 : J);
    ML = std::max(ML, -g * p->kmin[i]);
    MR = std::max(MR, g * (p->kmin[i] + p->cnt[i] - 1));
  }
  // synthesis (sidwt_synthesize): 5/3, 9/7 and integer 5/3 bands of a symmetric extension
  // are (2N-2)-periodic and whole-sample symmetric (U_s about 0, W_s about -2^{s-1};
  // SURVEY App. A.4), so out-of-range reads reflect into the stored range once it covers
  // (-2^J, 0); causal D4 bands have no symmetry and the margin holds the inverse reach.
  if (p->fam == FD4) {
    int sl = 0, sr = 0;
    inverse_reach(p->fam, sl, sr);
    const int span = (1 << (J + 1)) - 2;                         // sum_{l=1..J} 2^l
    ML = std::max(ML, sl * span);
    MR = std::max(MR, sr * span);
  } else {
    ML = std::max(ML, 1 << J);
  }
  ML = (int)rup(ML, 4);      // 16-byte aligned band segments (int8 and single-template tensor-core paths)
  if (p->ext == SIDWT_EXT_PERIODIC) { ML = 0; MR = 0; }
  p->ML = ML; p->MR = MR;
  p->stride = rup(ML + p->N + MR, 32);

  // ---- K1 tiling
  const int rv = rv_for(p->fam, J);
  p->ana_rv = rv;
  const Reach rc = dual_reach(p->fam);
  const int maxL = std::max(rc.lowL, rc.hiL);
  const int64_t halo_l = rup((int64_t)maxL * ((1LL << J) - 1), 4);
  const int64_t halo_r = std::max<int64_t>((int64_t)rc.lowR * ((1LL << J) - 1),
                                           (int64_t)rc.lowR * ((1LL << (J - 1)) - 1) + (int64_t)rc.hiR * (1LL << (J - 1)));
  int64_t lbuf_target = 6144;
  if (const char* e = std::getenv("SIDWT_K1_LBUF")) lbuf_target = std::max<int64_t>(256, atoll(e));
  int64_t ntiles = 1, tile_len = 0, lbuf = 0, threads = 0;
  for (;; ++ntiles) {
    tile_len = rup(cdiv(p->stride, ntiles), 32);
    lbuf = rup(halo_l + tile_len + halo_r, 4);
    threads = 0;
    for (int s = 1; s <= J; ++s) {
      const int64_t h = 1LL << (s - 1);
      threads = std::max(threads, h * cdiv(cdiv(lbuf, h), rv));
    }
    if ((lbuf <= lbuf_target && threads <= 512) || tile_len <= 32) break;
  }
  // more, smaller tiles while the halo stays cheap (<= 5 % of the tile, tiles >= 2048 values):
  // a larger grid hides latency better (C2: 0.179 -> 0.159 ms); long halos (C5, J = 8) keep
  // the big tile
  if (!std::getenv("SIDWT_K1_LBUF")) {
    for (int64_t nt = ntiles + 1;; ++nt) {
      const int64_t tl = rup(cdiv(p->stride, nt), 32);
      if (tl < 2048 || (halo_l + halo_r) * 20 > tl) break;
      ntiles = nt; tile_len = tl; lbuf = rup(halo_l + tile_len + halo_r, 4);
      threads = 0;
      for (int s = 1; s <= J; ++s) {
        const int64_t h = 1LL << (s - 1);
        threads = std::max(threads, h * cdiv(cdiv(lbuf, h), rv));
      }
    }
  }
  ntiles = cdiv(p->stride, tile_len);
  p->ana.lift = lift_f32(lift97_t(p->t97));
  p->ana.N = (int)p->N; p->ana.J = J; p->ana.ext = p->ext; p->ana.stride = (int)p->stride; p->ana.ML = ML;
  p->ana.tile_len = (int)tile_len; p->ana.ntiles = (int)ntiles; p->ana.halo_l = (int)halo_l; p->ana.lbuf = (int)lbuf;
  // pads absorbing the clamp-free window reads / run writes past the buffer ends (top level)
  int HL = 1, HR = 3;
  if (p->fam == F97) { HL = Dual<F97>::HL; HR = Dual<F97>::HR; }
  else if (p->fam == FD4) { HL = Dual<FD4>::HL; HR = Dual<FD4>::HR; }
  const int64_t htop = 1LL << (J - 1);
  p->ana.padl = (int)rup(HL * htop, 4);
  p->ana.padr = (int)rup((rv - 1 + HR) * htop, 4);
  p->ana_threads_needed = rup(threads, 32);
  p->ana_threads = (int)std::min<int64_t>(512, p->ana_threads_needed);
  p->ana_smem = (size_t)(p->ana.padl + 2 * (lbuf + p->ana.padr)) * 4;

  // ---- K2 tiling
  int64_t tt_target = 2048;
  if (const char* e = std::getenv("SIDWT_K2_TT")) tt_target = std::max<int64_t>(64, atoll(e));
  int64_t TT = std::min<int64_t>(p->N, std::max<int64_t>(tt_target, 1LL << J));
  CorParams& c = p->cor;
  c.N = (int)p->N; c.J = J; c.ext = p->ext; c.stride = (int)p->stride; c.ML = ML; c.n_t = p->n_t;
  c.TT = (int)TT; c.ntiles = (int)(p->N / TT); c.taps_per_t = p->taps_per_t;
  for (int i = 0; i <= J; ++i) {
    const int lg = i < J ? i + 1 : J;
    c.term[i].band = i; c.term[i].lg = lg; c.term[i].kmin = p->kmin[i];
    c.term[i].npad = p->npad[i]; c.term[i].ntap = p->cnt[i]; c.term[i].toff = p->toff[i];
  }
  k2_buffers(p, kQ);
}

// K2 band tile buffers for items of Q outputs: the tile of a term spans TT + g (ntap - 1)
// values, plus g (Q - 1) read past it by the ragged last q-block of a residue.
static void k2_buffers(sidwt_plan_s* p, int Q) {
  CorParams& c = p->cor;
  int blen_max = 0;
  for (int i = 0; i <= c.J; ++i)
    blen_max = std::max<int>(blen_max, c.TT + (1 << c.term[i].lg) * (c.term[i].ntap - 1 + Q - 1));
  c.balloc = (int)rup(blen_max + 4, 4);          // + alignment shift of the bulk copy
  // double-buffered band tiles when they fit (prefetch overlaps compute), else single
  c.nbuf = 2;
  auto smem = [&](int nb) { return 16 + rup((int64_t)p->taps_per_t * 8, 128) + (size_t)2 * nb * c.balloc * 4 + (size_t)4 * c.TT * 4; };
  if (smem(2) > 150 * 1024) c.nbuf = 1;
  p->cor_smem = smem(c.nbuf);
}

// Tensor-core bank path: float families, N a multiple of the 512-lag tile pair, a
// template bank (n_t >= 16; SIDWT_TC=0 disables, SIDWT_TC=1 forces it for any n_t).
static void configure_tc(sidwt_plan_s* p) {
  p->tc = false;
  if (p->paper) return;
  if (is_int(p) || p->N % kTcTilePair != 0) return;
  const char* env = std::getenv("SIDWT_TC");
  if (env && env[0] == '0') return;
  if (p->n_t < 16 && !(env && env[0] == '1')) return;
  TcParams& t = p->tcp;
  t = TcParams{};
  t.N = (int)p->N; t.J = p->J; t.ext = p->ext; t.stride = (int)p->stride; t.ML = p->ML; t.n_t = p->n_t;
  t.n_mt = (int)cdiv(p->n_t, kTcTemplates);
  t.ntiles = (int)(p->N / 256);
  int kofs = 0, nz_max = 0, kmax = 0, lmax = 0;
  for (int step = 0; step <= p->J; ++step) {
    const int ti = p->J - step;
    TcTerm& m = t.term[step];
    const int lg = ti < p->J ? ti + 1 : p->J;
    m.band = ti; m.g = 1 << lg; m.ge = std::min(m.g, 8); m.f = m.g / m.ge;
    m.kmin = p->kmin[ti]; m.ntap = p->cnt[ti]; m.toff = p->toff[ti];
    const int ntap_e = (m.ntap - 1) * m.f + 1;
    m.kp = (int)rup(ntap_e, 16);
    m.ksteps = 2 * m.kp / 16;
    m.kofs = kofs;
    kofs += m.ksteps;
    m.nz = (256 - 8) / m.ge + m.kp;
    nz_max = std::max(nz_max, m.nz);
    kmax = std::max(kmax, m.ksteps);
    lmax = std::max(lmax, m.ge * (m.nz - 1) + 8);
  }
  t.total_ksteps = kofs;
  t.nz_max = (int)rup(nz_max, 8);
  t.stg_len = (int)rup(lmax + 8, 8);
  t.npairs = 0;
  t.stages = 0;
  const TcSmem base = tc_smem_layout(t);                  // with 0 stages
  const int budget = 227 * 1024;
  const int fit = (budget - base.total) / kTcStageBytes;
  if (fit < 3) return;
  t.stages = std::min(kTcMaxStages, fit);
  t.a_shared = 1;                                         // second unit of a pair reuses resident K steps
  if (const char* e = std::getenv("SIDWT_TC_SHARED")) t.a_shared = atoi(e) != 0;
  if (const char* e = std::getenv("SIDWT_TC_STAGES")) t.stages = std::max(3, std::min(t.stages, atoi(e)));
  p->tc_smem = (size_t)tc_smem_layout(t).total;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p->tc_sms = sms;
  p->tc = true;
}

// Single-template tensor-core path (corr_tcs.cuh): float families, one template,
// symmetric extension, N / 64 columns in [16, 128] (multiple of 16), every residue class
// at least one 64-lag block long (2^J <= N / 64).  SIDWT_TCS=0 disables it.
static void configure_tcs(sidwt_plan_s* p) {
  p->tcs = false;
  const char* env = std::getenv("SIDWT_TCS");
  if (env && env[0] == '0') return;
  // default: complex templates with a long finest term (measured: C3 correlation 14.9 -> 9.4 ms);
  // real / short templates stay on the SIMT kernel (C2: 0.48 ms SIMT vs 1.2 ms here)
  if (!(env && env[0] == '1') && (p->real_taps || p->cnt[0] < 128)) return;
  if (p->paper || is_int(p) || p->n_t != 1 || p->ext != SIDWT_EXT_SYMMETRIC || p->tc) return;
  if (p->N % 64 != 0) return;
  const int ncols = (int)(p->N / 64);
  if (ncols < 16 || ncols > 128 || ncols % 16 != 0 || (1LL << p->J) > ncols) return;
  TcsParams& t = p->tcsp;
  t = TcsParams{};
  t.N = (int)p->N; t.J = p->J; t.stride = (int)p->stride; t.ML = p->ML; t.ncols = ncols;
  t.ncols_alloc = 32;                                             // one accumulator, double-buffered
  while (t.ncols_alloc < ncols) t.ncols_alloc *= 2;
  int kofs = 0;
  for (int step = 0; step <= p->J; ++step) {
    const int ti = p->J - step;
    TcsTerm& tm = t.term[step];
    tm.band = ti; tm.lg = ti < p->J ? ti + 1 : p->J;
    tm.kmin = p->kmin[ti]; tm.ntap = p->cnt[ti]; tm.toff = p->toff[ti];
    tm.ksteps = (int)cdiv(tm.ntap + 63, 16);
    tm.kofs = kofs; kofs += tm.ksteps;
    const int g = 1 << tm.lg;
    const int64_t a = (int64_t)p->ML + (int64_t)g * tm.kmin;   // band index of (r = 0, m = 0)
    if (a < 0) return;
    tcs_term_rows(tm, ncols);
    t.brows_max = std::max(t.brows_max, tm.kcoff[8]);
    int64_t imax = 0;                                              // last band index any buffer row reads
    for (int kc = 0; kc < 8; ++kc) {
      const int W = tm.kcoff[kc + 1] - tm.kcoff[kc];
      if (W > 0) imax = std::max<int64_t>(imax, a + (g - 1) + (int64_t)g * (64 * ((W - 1) >> tm.lg) + 8 * kc + 7));
    }
    tm.pf_a4 = (int)(a & ~3LL);
    tm.pf_len = (int)rup(std::min<int64_t>(imax + 1, p->stride) - tm.pf_a4, 4);
  }
  p->tcs_total_ksteps = kofs;
  t.stages = 6;
  if (const char* e = std::getenv("SIDWT_TCS_STAGES")) t.stages = std::max(2, std::min(8, atoi(e)));
  while (t.stages > 2 && tcs_smem_layout(t).total > 227 * 1024) --t.stages;
  if (tcs_smem_layout(t).total > 227 * 1024) return;
  p->tcs_smem = tcs_smem_layout(t).total;
  p->tcs = true;
}

// Integer family on the int8 tensor cores (corr_i8.cu): one template, symmetric extension,
// N <= 4096 (two 2048-lag tiles per row).  SIDWT_I8=0 disables it (the INT32 SIMT kernel runs).
static void configure_i8(sidwt_plan_s* p) {
  p->i8 = false;
  const char* env = std::getenv("SIDWT_I8");
  if (env && env[0] == '0') return;
  if (!is_int(p) || p->n_t != 1 || p->ext != SIDWT_EXT_SYMMETRIC || p->paper) return;
  std::vector<int2> taps((size_t)p->taps_per_t);
  if (cudaMemcpy(taps.data(), p->d_taps, taps.size() * sizeof(int2), cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  p->i8 = i8_configure(p->i8p, (int)p->N, p->J, (int)p->stride, p->ML, p->kmin, p->cnt, p->toff, taps.data());
}

// Fused path: single template, taps in the kernel parameters, and a
// tile whose on-chip bands + term results fit two CTAs per SM.
constexpr int kFusNT = 256;
static void configure_fused(sidwt_plan_s* p) {
  p->fused = false;
  if (p->n_t != 1 || !p->ctaps || p->paper) return;
  if (!p->fus) p->fus = new (std::nothrow) FusParams();
  if (!p->fus) return;
  FusParams& f = *p->fus;
  f.lift = lift_f32(lift97_t(p->t97));
  const int J = p->J;
  int fML = 0, fMR = 0;
  for (int i = 0; i <= J; ++i) {
    const int g = 1 << (i < J ? i + 1 : J);
    fML = std::max(fML, -g * p->kmin[i]);
    fMR = std::max(fMR, g * (p->kmin[i] + p->cnt[i] - 1));
  }
  const Reach rc = dual_reach(p->fam);
  const int maxL = std::max(rc.lowL, rc.hiL);
  const int64_t halo_l = rup((int64_t)maxL * ((1LL << J) - 1), 4);
  const int64_t halo_r = std::max<int64_t>((int64_t)rc.lowR * ((1LL << J) - 1),
                                           (int64_t)rc.lowR * ((1LL << (J - 1)) - 1) + (int64_t)rc.hiR * (1LL << (J - 1)));
  int HL = 1, HR = 3;
  if (p->fam == F97) { HL = Dual<F97>::HL; HR = Dual<F97>::HR; }
  else if (p->fam == FD4) { HL = Dual<FD4>::HL; HR = Dual<FD4>::HR; }
  const int64_t htop = 1LL << (J - 1);
  const int64_t padl = rup(HL * htop, 4), padr = rup((kRV - 1 + HR) * htop, 4);
  for (int64_t TT = std::min<int64_t>(p->N, 2048); TT >= 256 && TT >= (1LL << J); TT >>= 1) {
    const int64_t lbuf = rup(halo_l + fML + TT + fMR + halo_r, 4);
    int64_t threads = 0;
    for (int sl = 1; sl <= J; ++sl) {
      const int64_t h = 1LL << (sl - 1);
      threads = std::max(threads, h * cdiv(cdiv(lbuf, h), kRV));
    }
    const int64_t per = padl + 2 * (lbuf + padr);
    const size_t smem = (size_t)rup(2 * per * 4, 16) + (size_t)(J + 1) * TT * 8;
    if (threads > kFusNT || smem > 110 * 1024) continue;
    f.N = (int)p->N; f.J = J; f.ext = p->ext; f.TT = (int)TT; f.ntiles = (int)(p->N / TT);
    f.fML = fML; f.halo_l = (int)halo_l; f.lbuf = (int)lbuf; f.padl = (int)padl; f.padr = (int)padr;
    f.taps_per_t = p->taps_per_t;
    for (int i = 0; i <= J; ++i) f.term[i] = p->cor.term[i];
    memcpy(f.ctap, p->cor.ctap, sizeof(f.ctap));
    p->fus_smem = smem;
    p->fused = true;
    return;
  }
}

static sidwt_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return SIDWT_OK;
  if (e == cudaErrorMemoryAllocation) { cudaGetLastError(); return SIDWT_ERR_OOM; }
  cudaGetLastError();
  return SIDWT_ERR_CUDA;
}

sidwt_status sidwt_template_load(sidwt_plan p, const void* host_templates, int64_t T, int n_templates) {
  if (!p || !host_templates) return SIDWT_ERR_PARAM;
  if (T < 1 || T > p->N) return SIDWT_ERR_LENGTH;
  if (n_templates < 1 || n_templates > 65536) return SIDWT_ERR_DIMENSION;
  // validate the new layout before touching the loaded state: a rejected reload leaves the
  // previous template (and every buffer) usable
  {
    sidwt_plan_s* trial = new (std::nothrow) sidwt_plan_s(*p);
    if (!trial) return SIDWT_ERR_OOM;
    trial->T = (int)T; trial->n_t = n_templates;
    configure(trial);
    // K1 lifts one branch per thread at the deepest level (2^(J-1) branches): at most 512
    // threads, i.e. J <= 10 in practice; K1/K2 shared-memory tiles must fit
    const bool fits = trial->cor_smem <= 200 * 1024 && trial->ana_smem <= 200 * 1024 && trial->ana_threads_needed <= 512;
    delete trial;
    if (!fits) return SIDWT_ERR_RANGE;
  }
  if (p->d_taps) { cudaFree(p->d_taps); p->d_taps = nullptr; }
  if (p->d_partials) { cudaFree(p->d_partials); p->d_partials = nullptr; p->partials_bytes = 0; }
  if (p->d_img) { cudaFree(p->d_img); p->d_img = nullptr; }
  if (p->d_tcs_img) { cudaFree(p->d_tcs_img); p->d_tcs_img = nullptr; }
  if (p->d_i8_img) { cudaFree(p->d_i8_img); p->d_i8_img = nullptr; }
  p->loaded = false;
  p->T = (int)T; p->n_t = n_templates;
  configure(p);

  const size_t tab_bytes = (size_t)n_templates * p->taps_per_t * 8;
  const size_t x_bytes = (size_t)n_templates * T * sample_bytes(p);
  PyrParams pp{};
  pp.fam = p->fam; pp.J = p->J; pp.T = (int)T; pp.n_t = n_templates; pp.taps_per_t = p->taps_per_t;
  for (int i = 0; i <= p->J; ++i) {
    pp.klo[i] = p->kmin[i]; pp.cnt[i] = p->cnt[i]; pp.off[i] = p->toff[i]; pp.npad[i] = p->npad[i];
  }
  pp.scratch_len = (int)T + 64;
  pp.nres = p->paper ? (1 << p->J) : 1;
  pp.lift = lift97_t(p->t97);
  void* d_x = nullptr;
  double* d_scr = nullptr;
  cudaError_t e = cudaMalloc(&p->d_taps, tab_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&d_x, x_bytes);
  if (e == cudaSuccess) e = cudaMalloc((void**)&d_scr, (size_t)2 * n_templates * pp.nres * 4 * pp.scratch_len * sizeof(double));
  if (e == cudaSuccess) e = cudaMemset(p->d_taps, 0, tab_bytes);
  if (e == cudaSuccess) e = cudaMemcpy(d_x, host_templates, x_bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const int threads = 64;
    k_template_pyramid<<<(unsigned)cdiv(2 * n_templates * pp.nres, threads), threads>>>(d_x, p->d_taps, d_scr, pp);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (d_x) cudaFree(d_x);
  if (d_scr) cudaFree(d_scr);
  if (e != cudaSuccess) {
    if (p->d_taps) { cudaFree(p->d_taps); p->d_taps = nullptr; }
    return cuda_status(e);
  }
  // small tap tables travel in the SIMT correlation's kernel parameters (constant cache)
  p->ctaps = false;
  p->real_taps = false;
  if ((int64_t)n_templates * p->taps_per_t <= kCTaps && !(std::getenv("SIDWT_CTAPS") && std::getenv("SIDWT_CTAPS")[0] == '0')) {
    e = cudaMemcpy(p->cor.ctap, p->d_taps, tab_bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { cudaFree(p->d_taps); p->d_taps = nullptr; return cuda_status(e); }
    p->ctaps = true;
    // real template (imaginary bits all +-0 / integer 0): the correlation skips the t.y terms
    bool real = !(std::getenv("SIDWT_REALT") && std::getenv("SIDWT_REALT")[0] == '0');
    for (int64_t i = 0; real && i < (int64_t)n_templates * p->taps_per_t; ++i)
      real = (p->cor.ctap[i].y & 0x7fffffffu) == 0u;
    p->real_taps = real;
  }
  configure_fused(p);
  configure_tc(p);
  configure_tcs(p);
  configure_i8(p);
  if (p->i8) {
    e = cudaMalloc(&p->d_i8_img, i8_image_bytes(p->i8p));
    if (e == cudaSuccess) e = i8_build_images(p->i8p, static_cast<const int2*>(p->d_taps), p->toff,
                                              static_cast<unsigned char*>(p->d_i8_img));
    if (e != cudaSuccess) {
      if (p->d_i8_img) { cudaFree(p->d_i8_img); p->d_i8_img = nullptr; }
      cudaFree(p->d_taps); p->d_taps = nullptr;
      return cuda_status(e);
    }
  }

  if (p->tcs) {
    const size_t img_bytes = (size_t)p->tcs_total_ksteps * kTcsAStage;
    e = cudaMalloc(&p->d_tcs_img, img_bytes);
    if (e == cudaSuccess) {
      const long long items = (long long)p->tcs_total_ksteps * 4 * 128;
      k_tcs_images<<<(unsigned)cdiv(items, 256), 256>>>(static_cast<const float2*>(p->d_taps), p->tcsp,
                                                         p->tcs_total_ksteps, static_cast<unsigned char*>(p->d_tcs_img));
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      if (p->d_tcs_img) { cudaFree(p->d_tcs_img); p->d_tcs_img = nullptr; }
          cudaFree(p->d_taps); p->d_taps = nullptr;
      return cuda_status(e);
    }
  }
  if (p->tc) {
    const size_t img_bytes = (size_t)p->tcp.n_mt * p->tcp.total_ksteps * 8192;
    e = cudaMalloc(&p->d_img, img_bytes);
    if (e == cudaSuccess) {
      const long long items = (long long)p->tcp.n_mt * p->tcp.total_ksteps * 2 * kTcM;
      k_tc_images<<<(unsigned)cdiv(items, 256), 256>>>(static_cast<const float2*>(p->d_taps), p->taps_per_t, p->tcp,
                                                        static_cast<unsigned char*>(p->d_img));
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      if (p->d_img) { cudaFree(p->d_img); p->d_img = nullptr; }
      cudaFree(p->d_taps); p->d_taps = nullptr;
      return cuda_status(e);
    }
  }
  p->loaded = true;
  return SIDWT_OK;
}

int64_t sidwt_template_taps(sidwt_plan p, void* host_taps, int32_t* kmin, int32_t* count) {
  if (!p || !p->loaded) return -1;
  if (kmin) for (int i = 0; i <= p->J; ++i) kmin[i] = p->kmin[i];
  if (count) for (int i = 0; i <= p->J; ++i) count[i] = p->cnt[i];
  int64_t per_t = 0;
  for (int i = 0; i <= p->J; ++i) per_t += p->cnt[i];
  if (host_taps) {
    std::vector<uint64_t> tab((size_t)p->n_t * p->taps_per_t);
    if (cudaMemcpy(tab.data(), p->d_taps, tab.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) { cudaGetLastError(); return -1; }
    uint64_t* out = static_cast<uint64_t*>(host_taps);
    for (int t = 0; t < p->n_t; ++t)
      for (int i = 0; i <= p->J; ++i)
        for (int k = 0; k < p->cnt[i]; ++k) *out++ = tab[(size_t)t * p->taps_per_t + p->toff[i] + k];
  }
  return per_t;
}

// ---------------------------------------------------------------------------
// Device calls
// ---------------------------------------------------------------------------
template <int FAM>
static cudaError_t launch_analyze(const sidwt_plan_s* p, const void* rows, int64_t nrows, void* bands, cudaStream_t s) {
  auto kern = (FAM == F97 && p->ana_rv == kRV97) ? k_analyze<FAM, kRV97> : k_analyze<FAM, kRV>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->ana_smem);
  if (e != cudaSuccess) return e;
  AnaParams a = p->ana;
  a.rows = nrows;
  const int64_t grid = nrows * 2 * a.ntiles;
  kern<<<(unsigned)grid, p->ana_threads, p->ana_smem, s>>>(rows, bands, a);
  return cudaGetLastError();
}

sidwt_status sidwt_analyze(sidwt_plan p, const void* d_rows, int64_t rows, void* d_bands, void* stream) {
  if (!p || !d_rows || !d_bands) return SIDWT_ERR_PARAM;
  if (!p->loaded) return SIDWT_ERR_STATE;
  if (rows < 1 || rows > p->batch) return SIDWT_ERR_DIMENSION;
  if (rows * 2 * p->ana.ntiles > 0x7fffffffLL) return SIDWT_ERR_RANGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (p->fam) {
    case F53: e = launch_analyze<F53>(p, d_rows, rows, d_bands, s); break;
    case F97: e = launch_analyze<F97>(p, d_rows, rows, d_bands, s); break;
    case FD4: e = launch_analyze<FD4>(p, d_rows, rows, d_bands, s); break;
    default:  e = launch_analyze<FI53>(p, d_rows, rows, d_bands, s); break;
  }
  p->last_launches = 1;
  return cuda_status(e);
}

static sidwt_status ensure_partials(sidwt_plan_s* p) {
  const size_t rec = is_int(p) ? sizeof(PeakI) : sizeof(PeakF);
  const size_t need = (size_t)p->batch * p->n_t * (p->J + 1) * (p->tc ? 2 * p->tcp.ntiles : p->cor.ntiles) * rec;
  if (p->partials_bytes >= need) return SIDWT_OK;
  if (p->d_partials) cudaFree(p->d_partials);
  p->d_partials = nullptr;
  p->partials_bytes = 0;
  cudaError_t e = cudaMalloc(&p->d_partials, need);
  if (e != cudaSuccess) return cuda_status(e);
  p->partials_bytes = need;
  return SIDWT_OK;
}

// corr [rows][n_t][J+1][N] complex64 as a 4-D TMA tensor of 8-byte elements; box = 16 lags x
// 1 scale x 16 templates x 1 row, 128-byte swizzle (matches the epilogue staging layout).
static bool encode_corr_map(CUtensorMap* map, void* corr, int64_t rows, const sidwt_plan_s* p) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }
  const cuuint64_t dims[4] = {(cuuint64_t)p->N, (cuuint64_t)(p->J + 1), (cuuint64_t)p->n_t, (cuuint64_t)rows};
  const cuuint64_t strides[3] = {(cuuint64_t)p->N * 8, (cuuint64_t)p->N * 8 * (p->J + 1),
                                 (cuuint64_t)p->N * 8 * (p->J + 1) * p->n_t};
  const cuuint32_t box[4] = {16, 1, 16, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, corr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static sidwt_status correlate_tc(sidwt_plan_s* p, const void* d_bands, int64_t rows, void* d_corr,
                                 int32_t* d_lag, void* d_val, bool peaks, cudaStream_t s) {
  TcParams t = p->tcp;
  t.rows = rows;
  t.want_corr = d_corr != nullptr;
  t.want_peaks = peaks;
  t.npairs = rows * t.n_mt * t.ntiles / 2;
  if (t.npairs >= (1LL << 30)) return SIDWT_ERR_RANGE;
  if (d_corr && !encode_corr_map(&t.tmap, d_corr, rows, p)) return SIDWT_ERR_CUDA;
  if (const char* e = std::getenv("SIDWT_TC_PROF")) t.prof = atoi(e);
  const int64_t grid = std::min<int64_t>(t.npairs, p->tc_sms);
  cudaError_t e = cudaFuncSetAttribute(k_correlate_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->tc_smem);
  if (e == cudaSuccess) {
    k_correlate_tc<<<(unsigned)grid, kTcThreads, p->tc_smem, s>>>(static_cast<const float*>(d_bands),
                                                                  static_cast<const unsigned char*>(p->d_img),
                                                                  static_cast<float2*>(d_corr),
                                                                  static_cast<PeakF*>(p->d_partials), t);
    e = cudaGetLastError();
  }
  p->last_launches = 1;
  if (e == cudaSuccess && peaks) {
    const int64_t count = rows * p->n_t * (p->J + 1);
    k_peaks_finalize<false><<<(unsigned)cdiv(count, 8), 256, 0, s>>>(p->d_partials, 2 * t.ntiles, count, d_lag, d_val);
    e = cudaGetLastError();
    p->last_launches = 2;
  }
  return cuda_status(e);
}

static sidwt_status correlate_tcs(sidwt_plan_s* p, const void* d_bands, int64_t rows, void* d_corr,
                                  int32_t* d_lag, void* d_val, bool peaks, cudaStream_t s) {
  TcsParams t = p->tcsp;
  t.rows = rows;
  if (const char* ev = std::getenv("SIDWT_TC_PROF")) t.prof = atoi(ev);
  t.want_corr = d_corr != nullptr;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(rows, sms);
  cudaError_t e = cudaFuncSetAttribute(k_correlate_tcs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->tcs_smem);
  if (e == cudaSuccess) {
    k_correlate_tcs<<<(unsigned)grid, kTcsThreads, p->tcs_smem, s>>>(
        static_cast<const float*>(d_bands), static_cast<const unsigned char*>(p->d_tcs_img), static_cast<float2*>(d_corr),
        peaks ? d_lag : nullptr, peaks ? static_cast<float2*>(d_val) : nullptr, t);
    e = cudaGetLastError();
  }
  p->last_launches = 1;
  return cuda_status(e);
}

static sidwt_status correlate_i8(sidwt_plan_s* p, const void* d_bands, int64_t rows, void* d_corr,
                                 int32_t* d_lag, void* d_val, bool peaks, cudaStream_t s) {
  I8Params t = p->i8p;
  t.rows = rows;
  t.want_corr = d_corr != nullptr;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(rows, sms);
  cudaError_t e = i8_launch(t, static_cast<const int*>(d_bands), static_cast<const unsigned char*>(p->d_i8_img),
                            static_cast<int2*>(d_corr), peaks ? d_lag : nullptr,
                            peaks ? static_cast<int2*>(d_val) : nullptr, grid, s);
  p->last_launches = 1;
  return cuda_status(e);
}

static sidwt_status correlate_impl(sidwt_plan_s* p, const void* d_bands, int64_t rows, void* d_corr,
                                   int32_t* d_lag, void* d_val, bool peaks, cudaStream_t s) {
  if (p->tc) return correlate_tc(p, d_bands, rows, d_corr, d_lag, d_val, peaks, s);
  if (p->i8) return correlate_i8(p, d_bands, rows, d_corr, d_lag, d_val, peaks, s);
  if (p->tcs) return correlate_tcs(p, d_bands, rows, d_corr, d_lag, d_val, peaks, s);
  CorParams c = p->cor;
  c.rows = rows;
  c.want_corr = d_corr != nullptr;
  c.want_peaks = peaks;
  const int64_t grid = rows * p->n_t * c.ntiles;
  if (grid > 0x7fffffffLL) return SIDWT_ERR_RANGE;
  cudaError_t e;
  // 3 CTAs x 8 warps per SM (measured best on C2); the integer kernel's 3-multiply MAC keeps a
  // third window array and runs best at 2 CTAs/SM (C5: 17.3 vs 20.1 ms at 3)
  int minb = (is_int(p) && !p->real_taps) ? 2 : 3;
  if (const char* ev = std::getenv("SIDWT_K2_MINB")) minb = std::max(1, std::min(4, atoi(ev)));
  void (*kern)(const void*, const void*, void*, void*, const CorParams);
  const bool ct = p->ctaps;
  const bool m3 = minb >= 3;
  if (p->paper) {                                  // float families only (checked at set_orientation)
    kern = ct ? k_correlate<false, kQ, kK2NT, 3, true, true> : k_correlate<false, kQ, kK2NT, 3, false, true>;
  } else if (p->real_taps && ct) {                 // real template bank (zero imaginary taps)
    kern = is_int(p) ? k_correlate<true, kQ, kK2NT, 3, true, false, true> : k_correlate<false, kQ, kK2NT, 3, true, false, true>;
  } else if (is_int(p)) {
    if (ct) kern = m3 ? k_correlate<true, kQ, kK2NT, 3, true> : k_correlate<true, kQ, kK2NT, 2, true>;
    else kern = m3 ? k_correlate<true, kQ, kK2NT, 3, false> : k_correlate<true, kQ, kK2NT, 2, false>;
  } else {
    if (ct) kern = m3 ? k_correlate<false, kQ, kK2NT, 3, true> : k_correlate<false, kQ, kK2NT, 2, true>;
    else kern = m3 ? k_correlate<false, kQ, kK2NT, 3, false> : k_correlate<false, kQ, kK2NT, 2, false>;
  }
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->cor_smem);
  if (e == cudaSuccess) {
    kern<<<(unsigned)grid, kK2NT, p->cor_smem, s>>>(d_bands, p->d_taps, d_corr, p->d_partials, c);
    e = cudaGetLastError();
  }
  p->last_launches = 1;
  if (e == cudaSuccess && peaks) {
    const int64_t count = rows * p->n_t * (p->J + 1);
    const unsigned blocks = (unsigned)cdiv(count, 8);           // one warp per (row, template, scale)
    if (is_int(p)) k_peaks_finalize<true><<<blocks, 256, 0, s>>>(p->d_partials, c.ntiles, count, d_lag, d_val);
    else k_peaks_finalize<false><<<blocks, 256, 0, s>>>(p->d_partials, c.ntiles, count, d_lag, d_val);
    e = cudaGetLastError();
    p->last_launches = 2;
  }
  return cuda_status(e);
}

sidwt_status sidwt_correlate(sidwt_plan p, const void* d_bands, int64_t rows, void* d_corr, void* stream) {
  if (!p || !d_bands || !d_corr) return SIDWT_ERR_PARAM;
  if (!p->loaded) return SIDWT_ERR_STATE;
  if (rows < 1 || rows > p->batch) return SIDWT_ERR_DIMENSION;
  return correlate_impl(p, d_bands, rows, d_corr, nullptr, nullptr, false, static_cast<cudaStream_t>(stream));
}

sidwt_status sidwt_correlate_peaks(sidwt_plan p, const void* d_bands, int64_t rows, void* d_corr, int32_t* d_lag,
                                   void* d_val, void* stream) {
  if (!p || !d_bands || !d_lag) return SIDWT_ERR_PARAM;
  if (!p->loaded) return SIDWT_ERR_STATE;
  if (rows < 1 || rows > p->batch) return SIDWT_ERR_DIMENSION;
  sidwt_status st = ensure_partials(p);
  if (st != SIDWT_OK) return st;
  return correlate_impl(p, d_bands, rows, d_corr, d_lag, d_val, true, static_cast<cudaStream_t>(stream));
}

template <int FAM>
static cudaError_t launch_fused(sidwt_plan_s* p, const void* rows_in, int64_t rows, void* corr, bool peaks, cudaStream_t s) {
  auto kern = k_fused<FAM, kRV, kQ, kFusNT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->fus_smem);
  if (e != cudaSuccess) return e;
  FusParams& f = *p->fus;
  f.rows = rows;
  f.want_corr = corr != nullptr;
  f.want_peaks = peaks;
  kern<<<(unsigned)(rows * f.ntiles), kFusNT, p->fus_smem, s>>>(rows_in, corr, p->d_fpartials, f);
  return cudaGetLastError();
}

sidwt_status sidwt_analyze_correlate(sidwt_plan p, const void* d_rows, int64_t rows, void* d_corr, int32_t* d_lag,
                                     void* d_val, void* stream) {
  if (!p || !d_rows || !d_lag) return SIDWT_ERR_PARAM;
  if (!p->loaded) return SIDWT_ERR_STATE;
  if (rows < 1 || rows > p->batch) return SIDWT_ERR_DIMENSION;
  if (!p->fused) return SIDWT_ERR_RANGE;
  if (rows * p->fus->ntiles > 0x7fffffffLL) return SIDWT_ERR_RANGE;
  const size_t rec = is_int(p) ? sizeof(PeakI) : sizeof(PeakF);
  const size_t need = (size_t)p->batch * (p->J + 1) * p->fus->ntiles * rec;
  if (p->fpartials_bytes < need) {
    if (p->d_fpartials) cudaFree(p->d_fpartials);
    p->d_fpartials = nullptr;
    p->fpartials_bytes = 0;
    cudaError_t e = cudaMalloc(&p->d_fpartials, need);
    if (e != cudaSuccess) return cuda_status(e);
    p->fpartials_bytes = need;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (p->fam) {
    case F53: e = launch_fused<F53>(p, d_rows, rows, d_corr, true, s); break;
    case F97: e = launch_fused<F97>(p, d_rows, rows, d_corr, true, s); break;
    case FD4: e = launch_fused<FD4>(p, d_rows, rows, d_corr, true, s); break;
    default:  e = launch_fused<FI53>(p, d_rows, rows, d_corr, true, s); break;
  }
  if (e == cudaSuccess) {
    const int64_t count = rows * (p->J + 1);
    const unsigned blocks = (unsigned)cdiv(count, 8);
    if (is_int(p)) k_peaks_finalize<true><<<blocks, 256, 0, s>>>(p->d_fpartials, p->fus->ntiles, count, d_lag, d_val);
    else k_peaks_finalize<false><<<blocks, 256, 0, s>>>(p->d_fpartials, p->fus->ntiles, count, d_lag, d_val);
    e = cudaGetLastError();
  }
  p->last_launches = 2;
  return cuda_status(e);
}

int sidwt_fused_available(sidwt_plan p) { return (p && p->loaded) ? (p->fused ? 1 : 0) : -1; }

sidwt_status sidwt_peaks(sidwt_plan p, const void* d_corr, int64_t rows, int32_t* d_lag, void* d_val, void* stream) {
  if (!p || !d_corr || !d_lag) return SIDWT_ERR_PARAM;
  if (!p->loaded) return SIDWT_ERR_STATE;
  if (rows < 1 || rows > p->batch) return SIDWT_ERR_DIMENSION;
  const int64_t count = rows * p->n_t * (p->J + 1);
  if (count > 0x7fffffffLL) return SIDWT_ERR_RANGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (is_int(p)) k_peaks<true><<<(unsigned)count, 256, 0, s>>>(d_corr, (int)p->N, d_lag, d_val);
  else k_peaks<false><<<(unsigned)count, 256, 0, s>>>(d_corr, (int)p->N, d_lag, d_val);
  p->last_launches = 1;
  return cuda_status(cudaGetLastError());
}

template <int FAM>
static cudaError_t launch_synthesize(const sidwt_plan_s* p, const void* bands, int64_t rows, int level, void* out,
                                     cudaStream_t s) {
  int sl = 0, sr = 0;
  inverse_reach(p->fam, sl, sr);
  SynParams q{};
  q.lift = lift_f32(lift97_t(p->t97));
  q.N = (int)p->N; q.J = p->J; q.ext = p->ext; q.stride = (int)p->stride; q.ML = p->ML; q.level = level;
  q.TL = (int)std::min<int64_t>(p->N, 2048);
  q.ntiles = (int)cdiv(p->N, q.TL);
  const int span = (1 << (p->J + 1)) - (1 << (level + 1));
  q.halo_l = sl * span; q.halo_r = sr * span;
  q.lbuf = (int)rup(q.halo_l + q.TL + q.halo_r, 4);
  q.rows = rows;
  const size_t smem = (size_t)3 * q.lbuf * 4;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  auto kern = k_synthesize<FAM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)(rows * 2 * q.ntiles), 256, smem, s>>>(bands, out, q);
  return cudaGetLastError();
}

sidwt_status sidwt_synthesize(sidwt_plan p, const void* d_bands, int64_t rows, int level, void* d_out, void* stream) {
  if (!p || !d_bands || !d_out) return SIDWT_ERR_PARAM;
  if (!p->loaded) return SIDWT_ERR_STATE;
  if (rows < 1 || rows > p->batch) return SIDWT_ERR_DIMENSION;
  if (level < 0 || level >= p->J) return SIDWT_ERR_DEPTH;
  if (rows * 2 * cdiv(p->N, 2048) > 0x7fffffffLL) return SIDWT_ERR_RANGE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (p->fam) {
    case F53: e = launch_synthesize<F53>(p, d_bands, rows, level, d_out, s); break;
    case F97: e = launch_synthesize<F97>(p, d_bands, rows, level, d_out, s); break;
    case FD4: e = launch_synthesize<FD4>(p, d_bands, rows, level, d_out, s); break;
    default:  e = launch_synthesize<FI53>(p, d_bands, rows, level, d_out, s); break;
  }
  p->last_launches = 1;
  if (e == cudaErrorInvalidValue) { cudaGetLastError(); return SIDWT_ERR_RANGE; }
  return cuda_status(e);
}

// End to end from host buffers, pipelined: the rows are cut into chunks; chunk k's
// host->device copy (copy stream) overlaps the analyze + correlate + peaks of chunk k-1
// (compute stream); both streams are ordered after, and the caller's stream after them,
// by events, so the call is still stream-ordered on `stream`.
sidwt_status sidwt_execute_host(sidwt_plan p, const void* h_rows, int64_t rows, int32_t* h_lag, void* h_val,
                                void* stream) {
  if (!p || !h_rows || !h_lag) return SIDWT_ERR_PARAM;
  if (!p->loaded) return SIDWT_ERR_STATE;
  if (rows < 1 || rows > p->batch) return SIDWT_ERR_DIMENSION;
  cudaError_t e = cudaSuccess;
  // plan-owned workspaces for `batch` rows, sized from the current layout (a template reload
  // may grow the band stride or the bank: reallocate then)
  const size_t cnt = (size_t)p->batch * p->n_t * (p->J + 1);
  auto ensure = [&](void*& buf, size_t& have, size_t need) {
    if (e != cudaSuccess || have >= need) return;
    if (buf) cudaFree(buf);
    buf = nullptr;
    have = 0;
    e = cudaMalloc(&buf, need);
    if (e == cudaSuccess) have = need;
  };
  ensure(p->w_rows, p->w_rows_bytes, (size_t)p->batch * p->N * sample_bytes(p));
  ensure(p->w_bands, p->w_bands_bytes, (size_t)sidwt_bands_bytes(p, p->batch));
  ensure(p->w_lag, p->w_lag_bytes, cnt * 4);
  ensure(p->w_val, p->w_val_bytes, cnt * 8);
  if (e == cudaSuccess && !p->s_copy) e = cudaStreamCreateWithFlags(&p->s_copy, cudaStreamNonBlocking);
  if (e == cudaSuccess && !p->s_comp) e = cudaStreamCreateWithFlags(&p->s_comp, cudaStreamNonBlocking);
  for (int k = 0; e == cudaSuccess && k < kPipeChunks + 2; ++k)
    if (!p->ev[k]) e = cudaEventCreateWithFlags(&p->ev[k], cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_status(e);
  sidwt_status st = ensure_partials(p);
  if (st != SIDWT_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaEvent_t ev_start = p->ev[kPipeChunks], ev_done = p->ev[kPipeChunks + 1];
  e = cudaEventRecord(ev_start, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_copy, ev_start, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_comp, ev_start, 0);
  if (e != cudaSuccess) return cuda_status(e);
  const int nch = (int)std::min<int64_t>(kPipeChunks, rows);
  const int64_t per = cdiv(rows, nch);
  const size_t sb = sample_bytes(p);
  const size_t per_row_out = (size_t)p->n_t * (p->J + 1);
  int launches = 0;
  for (int k = 0; k < nch; ++k) {
    const int64_t r0 = k * per, nr = std::min<int64_t>(per, rows - r0);
    if (nr <= 0) break;
    char* drows = static_cast<char*>(p->w_rows) + (size_t)r0 * p->N * sb;
    e = cudaMemcpyAsync(drows, static_cast<const char*>(h_rows) + (size_t)r0 * p->N * sb, (size_t)nr * p->N * sb,
                        cudaMemcpyHostToDevice, p->s_copy);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev[k], p->s_copy);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_comp, p->ev[k], 0);
    if (e != cudaSuccess) return cuda_status(e);
    char* dbands = static_cast<char*>(p->w_bands) + (size_t)sidwt_bands_bytes(p, r0);
    int32_t* dlag = static_cast<int32_t*>(p->w_lag) + r0 * per_row_out;
    char* dval = static_cast<char*>(p->w_val) + (size_t)r0 * per_row_out * 8;
    st = sidwt_analyze(p, drows, nr, dbands, p->s_comp);
    if (st != SIDWT_OK) return st;
    launches += p->last_launches;
    // peaks only: the call returns lag / val, so the correlation is not written to HBM
    st = sidwt_correlate_peaks(p, dbands, nr, nullptr, dlag, dval, p->s_comp);
    if (st != SIDWT_OK) return st;
    launches += p->last_launches;
    e = cudaMemcpyAsync(h_lag + r0 * per_row_out, dlag, (size_t)nr * per_row_out * 4, cudaMemcpyDeviceToHost, p->s_comp);
    if (e == cudaSuccess && h_val)
      e = cudaMemcpyAsync(static_cast<char*>(h_val) + (size_t)r0 * per_row_out * 8, dval, (size_t)nr * per_row_out * 8,
                          cudaMemcpyDeviceToHost, p->s_comp);
    if (e != cudaSuccess) return cuda_status(e);
  }
  e = cudaEventRecord(ev_done, p->s_comp);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev_done, 0);
  p->last_launches = launches;
  return cuda_status(e);
}

// Whole path on device-resident rows (analyze -> correlate -> peaks).  Optionally
// (SIDWT_RUN_CHUNKS > 1) the rows are cut into chunks: the analysis (HBM-bound) of
// chunk k+1 runs on a high-priority stream while the correlation (issue-bound) of chunk
// k runs on a low-priority one.  Measured on B200 (C2, C3, C5): no overlap materialises
// (the correlation's CTAs hold the SMs' shared memory), so 1 chunk is the default.
// Same outputs as sidwt_analyze + sidwt_correlate_peaks.
sidwt_status sidwt_run(sidwt_plan p, const void* d_rows, int64_t rows, void* d_bands, void* d_corr, int32_t* d_lag,
                       void* d_val, void* stream) {
  if (!p || !d_rows || !d_bands || !d_lag) return SIDWT_ERR_PARAM;
  if (!p->loaded) return SIDWT_ERR_STATE;
  if (rows < 1 || rows > p->batch) return SIDWT_ERR_DIMENSION;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int nch = p->run_chunks;
  if (const char* ev = std::getenv("SIDWT_RUN_CHUNKS")) nch = std::max(1, std::min(kRunChunks, atoi(ev)));
  nch = (int)std::min<int64_t>(nch, rows);
  sidwt_status st = ensure_partials(p);
  if (st != SIDWT_OK) return st;
  if (nch <= 1) {
    st = sidwt_analyze(p, d_rows, rows, d_bands, stream);
    if (st != SIDWT_OK) return st;
    const int l1 = p->last_launches;
    st = correlate_impl(p, d_bands, rows, d_corr, d_lag, d_val, true, s);
    p->last_launches += l1;
    return st;
  }
  cudaError_t e = cudaSuccess;
  if (!p->s_k1) {
    int lo = 0, hi = 0;
    e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&p->s_k1, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&p->s_k2, cudaStreamNonBlocking, lo);
  }
  for (int k = 0; e == cudaSuccess && k < kRunChunks + 2; ++k)
    if (!p->rev[k]) e = cudaEventCreateWithFlags(&p->rev[k], cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_status(e);
  cudaEvent_t ev_start = p->rev[kRunChunks], ev_done = p->rev[kRunChunks + 1];
  e = cudaEventRecord(ev_start, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_k1, ev_start, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_k2, ev_start, 0);
  if (e != cudaSuccess) return cuda_status(e);
  const int64_t per = cdiv(rows, nch);
  const size_t sb = sample_bytes(p);
  const size_t per_row_out = (size_t)p->n_t * (p->J + 1);
  int launches = 0;
  for (int k = 0; k < nch; ++k) {
    const int64_t r0 = k * per, nr = std::min<int64_t>(per, rows - r0);
    if (nr <= 0) break;
    char* dbands = static_cast<char*>(d_bands) + (size_t)sidwt_bands_bytes(p, r0);
    st = sidwt_analyze(p, static_cast<const char*>(d_rows) + (size_t)r0 * p->N * sb, nr, dbands, p->s_k1);
    if (st != SIDWT_OK) return st;
    launches += p->last_launches;
    e = cudaEventRecord(p->rev[k], p->s_k1);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_k2, p->rev[k], 0);
    if (e != cudaSuccess) return cuda_status(e);
    // chunks are serialised on s_k2, so they can share the peak partials buffer
    char* dcorr = d_corr ? static_cast<char*>(d_corr) + (size_t)sidwt_corr_bytes(p, r0) : nullptr;
    char* dval = d_val ? static_cast<char*>(d_val) + (size_t)r0 * per_row_out * 8 : nullptr;
    st = correlate_impl(p, dbands, nr, dcorr, d_lag + r0 * per_row_out, dval, true, p->s_k2);
    if (st != SIDWT_OK) return st;
    launches += p->last_launches;
  }
  e = cudaEventRecord(ev_done, p->s_k2);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev_done, 0);
  p->last_launches = launches;
  return cuda_status(e);
}
