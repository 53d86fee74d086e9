/* kk_cufft_cmp.h -- cuFFT-based COMPARISON pipeline for S1-S4 of the KK receiver
 * (libkkrx_cufft.so).  Not the product path: the north star asks for cuFFT "reported
 * only as a comparison" and SURVEY.md 8(d) lists a "cuFFT-based variant: same numbers,
 * comparison only".  The product is libkkrx.so (kk_rx.h), whose fused chain kernel
 * computes the same x2 without materialising anything in HBM.
 *
 * What it computes (the same operations as kk_rx's S1-S4, "a pair of 100%
 * overlap-save 1024-point FFTs ... another pair of FFTs" for the static EQ, l.53):
 *   S1  v = max(code + d, v_min), a = sqrt(v), l = 0.5 ln v
 *   S2  phi = IFFT(+i sgn(k) FFT(l)) blockwise: block j keeps [512 j, 512 j + 512) of the
 *       1024-point window starting at 512 j - 256, sgn(0) = sgn(512) = 0; blocks 2p and
 *       2p + 1 packed as one complex transform                        (reading R1, S2)
 *   S3  E_s[n] = (a e^{i phi} - A_hat) e^{i theta_n},
 *       theta_n = 2 pi ((tone_bin n) mod N) / N                        (S3, reading R7)
 *   S4  x2[m] = sum_{i=-101}^{101} h_i E_s[2m - i] by overlap-save: 1024-point FFT of the
 *       E_s window starting at 768 q - 128, times DFT(h placed circularly), spectral fold
 *       Z_k = (Y_k + Y_{k+512}) / 2, 512-point IFFT, keep outputs [64, 448) (S4)
 * as a multi-kernel pipeline: pack kernel -> cuFFT C2C -> mask kernel -> cuFFT C2C ->
 * S3 kernel (E_s materialised in HBM) -> cuFFT C2C over overlapping windows (advanced
 * layout, idist = 768) -> multiply-fold kernel -> cuFFT C2C 512 -> extract kernel.
 *
 * Conventions: all pointers to the data are DEVICE pointers; positions are buffer-local
 * (n = 0 is the buffer's first sample).  Status codes are kk_rx.h's (0 = OK, -1 bad
 * argument, -2 out of memory, -3 CUDA/cuFFT failure).
 */
#ifndef KK_CUFFT_CMP_H
#define KK_CUFFT_CMP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kk_cmp kk_cmp_t;

/* Create a pipeline for up to max_batch buffers of buffer_len samples (a multiple of 1024).
 * fir: 2*203 floats (re, im), tap i = t - 101 (as kk_rx_params.fir); copied.
 * a_hat: the carrier amplitude A_hat = sqrt(d c / (1 + c)) (reading R6) the caller uses.
 * Allocates the work arrays (~ 45 B per sample of the batch) and the cuFFT plans. */
int kk_cmp_create(kk_cmp_t **out, int64_t buffer_len, int max_batch, float dc_offset, float a_hat, float v_min,
                  int64_t tone_bin, const float *fir, int fir_len);

/* Left and right halo (samples) the pipeline reads around every buffer. */
int kk_cmp_halo(const kk_cmp_t *h, int64_t *left, int64_t *right);

/* x2 of nbuf <= max_batch buffers.  codes: device int16, buffer b starts at
 * codes + b * buffer_len, with the halo readable on both sides (a contiguous stream).
 * x2: device complex64 (re, im interleaved), nbuf * buffer_len / 2 entries, x2 index m of
 * buffer b at b * buffer_len / 2 + m.  Enqueued on stream (cudaStream_t; NULL = legacy
 * default stream); returns without synchronising. */
int kk_cmp_x2(kk_cmp_t *h, const int16_t *codes, int nbuf, float *x2, void *stream);

/* Number of kernel launches (own kernels + cuFFT executions) one kk_cmp_x2 call enqueues. */
int kk_cmp_launches(const kk_cmp_t *h, int nbuf);

/* Frees everything; NULL is a no-op. */
int kk_cmp_destroy(kk_cmp_t *h);

#ifdef __cplusplus
}
#endif
#endif
