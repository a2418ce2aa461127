// corr_i8.h -- integer-family correlation on the 5th-generation tensor cores (tcgen05.mma
// kind::i8), sm_100a: parameters and host entry points (kernels in corr_i8.cu, a separate
// translation unit).  Reversible integer 5/3 (reading R-INT): the bands
// are exact int32 and the correlation must be the exact integer reduced mod 2^32, so the
// contraction is carried out on byte digits with int32 accumulation -- exact -- and the
// digit products are recombined with shifts in the epilogue.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace sidwt {

constexpr int kI8MaxTerms = 17;

struct I8Term {
  int band, lg, kmin, ntap;
  int strided;      // g >= 16: one tap per 16-byte K half, the two halves of a K step g bytes apart
  int ksteps;       // K steps (32 bytes of K) per data component
  int kadv;         // A start advance per K step (bytes): 32 (dense) or 2 g (strided)
  int lbo;          // A leading byte offset (K-half stride): 16 (dense) or g (strided)
  int sh;           // dense: g kmin - P0, the stream offset of tap 0 at shift 0; strided: 0
  int P0;           // fine-grid position of stream byte 0
  int seg_a4;       // band index (P0 + ML) of the staged segment, multiple of 4
  int seg_len;      // int32 values staged per component (multiple of 4)
  int dig;          // data digits the static bound of the band needs (2..4)
  int img_ofs;      // byte offset of the term's B images: [ksteps][2 data components][ncol x 32 B]
};

struct I8Params {
  CUtensorMap cmap;                   // corr as [rows (J+1) N / 16 lag blocks][2 halves][8 lags] of 8-byte elements
  int N, J, stride, ML, ntiles, tn, ncol, dmax;
  int nband, nstream, nimg;           // ring depths: staged band segments, digit streams, B images
  int seg_alloc, plane, img_alloc;    // int32 per component per band stage; bytes per digit plane; bytes per image stage
  int want_corr;
  int tma_store;                      // corr_s written by TMA tensor stores (N a multiple of 512), else st.global
  long long rows;
  I8Term term[kI8MaxTerms];           // by processing step (0 = coarsest, a_J)
};

// Configure the path for one loaded integer template (host).  kmin / cnt / toff: the plan's
// term supports (term i < J: b_{i+1}, i = J: a_J) and table offsets; taps: host copy of the
// template's table ([taps_per_t] int2, unconjugated).  Returns false when the path does not
// apply (then the SIMT kernel runs).
bool i8_configure(I8Params& p, int N, int J, int stride, int ML, const int* kmin, const int* cnt, const int* toff,
                  const int2* taps);
size_t i8_image_bytes(const I8Params& p);
size_t i8_smem_bytes(const I8Params& p);
// B operand images (the template's Toeplitz digit matrices) from the device tap table.
cudaError_t i8_build_images(const I8Params& p, const int2* d_taps, const int* toff, unsigned char* d_img);
// corr: [rows][J+1][N] int2 or NULL (peaks only); lag / val: [rows][J+1] or NULL.
cudaError_t i8_launch(const I8Params& p, const int* bands, const unsigned char* img, int2* corr, int32_t* lag,
                      int2* val, int grid, cudaStream_t s);

}  // namespace sidwt
