/*
 * kk_rx.h -- C ABI of the B200-native Kramers-Kronig receiver hot path.
 *
 * One call processes raw 12-bit ADC buffers (int16 codes) into symbol decisions,
 * demapped labels and error counts, following the real-time DSP chain of
 * arXiv 2108.07004, Sec. 2:
 *
 *   S1 fixed->float, + DC offset, sqrt, log          PAPER l.47 ("first kernel")
 *   S2 blockwise 1024-pt Hilbert (keep centre 512)    PAPER l.47 ("step 3")
 *   S3 a*e^{i phi}, carrier removal, downconversion
 *   S4 203-tap static EQ + 4->2 sps resampling
 *   S5 4-tap widely-linear LMS (update pass + apply)
 *   S6 minimum-Euclidean-distance decision
 *   S7 demap to labels ("bits to RAM") + counting
 *
 * Readings of the paper where it is silent are listed in DESIGN.md (R1..R17).
 * All functions are thread-compatible: one handle per host thread.
 *
 * Errors: every function returns kk_status.  KK_EINVAL for bad arguments,
 * KK_ENOMEM for allocation failure, KK_ECUDA for a CUDA runtime error (sticky:
 * the handle must be destroyed), KK_ESTATE for calls in the wrong order,
 * KK_EUNSUPPORTED for unsupported configurations.  kk_rx_last_error() returns
 * a human-readable message for the last failure on the calling thread.
 * Data-domain problems are never errors: code + d < v_min is clamped and
 * counted (clipped_samples); a diverging adaptive equaliser sets a flag bit.
 */
#ifndef KK_RX_H
#define KK_RX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KK_RX_ABI_VERSION 2

typedef struct kk_rx kk_rx_t; /* opaque: owns device scratch, tables, streams */

typedef enum {
  KK_OK = 0,
  KK_EINVAL = -1,
  KK_ENOMEM = -2,
  KK_ECUDA = -3,
  KK_ESTATE = -4,
  KK_EUNSUPPORTED = -5
} kk_status;

/* Modulation formats.  GS8 / GS128 / CUSTOM need `points` and
 * `labels` in kk_rx_params (the paper uploads them, l.53); the conventional
 * formats are built in (Gray square QAM, 4x2 rectangular 8-QAM, cross 32/128;
 * reading R12) unless `points` overrides them. */
typedef enum {
  KK_QAM4 = 0, KK_QAM8 = 1, KK_QAM16 = 2, KK_QAM32 = 3, KK_QAM64 = 4, KK_QAM128 = 5,
  KK_GS8 = 6, KK_GS128 = 7, KK_CUSTOM = 8
} kk_format;

/* Reference of the adaptive-equaliser update (reading R10).
 * DD_SOFT: decision-directed with the soft gate gamma = min(1,(D2-D1)/tau) (default)
 * PILOT  : the known pattern symbol (the paper's training mode)
 * DD_HARD: textbook decision-directed (gamma = 1). */
typedef enum { KK_UPD_DD_SOFT = 0, KK_UPD_PILOT = 1, KK_UPD_DD_HARD = 2 } kk_update_mode;

#define KK_DUMP_ES 1u /* keep E_s (after S3) of the last call for kk_rx_debug_es() */
#define KK_DUMP_X2 2u /* materialise x2 (after S4) of the whole last batch for kk_rx_debug_x2()
                       * (by default only the update-pass tails are materialised) */

typedef struct {
  float dc_offset;          /* d, ADC-code units, added before sqrt/log */
  int64_t tone_bin;         /* tone frequency = tone_bin * fs / buffer_len; default 541065 */
  const float *fir;         /* REQUIRED: 2*fir_len floats (re,im interleaved), tap i = index-101, 4 sps */
  int32_t fir_len;          /* must be 203 */
  const float *w_init;      /* 16 floats: w[0..3] then g[0..3], complex interleaved; NULL = w=(0,1,0,0), g=0 */
  float mu;                 /* LMS step, default 1e-3 */
  int32_t k_update;         /* K: LMS steps per sub-block update pass, default 4096 */
  int32_t sub_block;        /* L: symbols per fixed-tap sub-block; 0 = buffer_len/sps (default) */
  float gate_tau;           /* tau of the soft gate; < 0 => d_min^2/4 (default); 0 => hard */
  int32_t update_mode;      /* kk_update_mode */
  const float *points;      /* 2*m floats (re,im), or NULL for the built-in table of `fmt` */
  const uint8_t *labels;    /* m bit labels, a permutation of 0..m-1 */
  int32_t m;                /* number of points (4..128, power of two) */
  const uint8_t *ref_pattern; /* error-count / PILOT reference: point INDICES, length ref_len; NULL = no counting */
  int32_t ref_len;          /* P, pattern period in symbols (2^20 in the paper) */
  int64_t ref_offset;       /* pattern index of symbol 0 of stream buffer 0 */
  float v_min;              /* clamp floor of code + d, default 1.0 (one LSB) */
  int32_t device;           /* CUDA device ordinal, -1 = current */
  void *cuda_stream;        /* cudaStream_t to launch on, NULL = handle-owned stream */
  uint32_t debug_dump;      /* bitmask of KK_DUMP_* */
  int32_t max_batch;        /* buffers per internal batch (device scratch sizing), default 16 */
  /* ABI 2: pre-KK intensity equaliser: real taps g_k,
   * k = -h..h, h = (pre_fir_len-1)/2 <= 8, applied before sqrt/log:
   * v' = sum_k g_k (code[n-k] + d).  NULL = off. */
  const float *pre_fir;
  int32_t pre_fir_len;
} kk_rx_params;

/* Per-buffer (or aggregate) counters, "Error counting". */
typedef struct {
  uint64_t bit_errors;      /* sum popcount(label[d_n] ^ label[ref_n]) */
  uint64_t sym_errors;      /* #(d_n != ref_n) */
  uint64_t bits;            /* symbols * log2(m) (0 when no ref_pattern) */
  uint64_t symbols;         /* buffer_len / sps per buffer */
  uint64_t clipped_samples; /* samples with code + d < v_min (clamped) */
  uint64_t gated_updates;   /* LMS steps whose soft gate was < 1 */
  uint32_t flags;           /* bit 0: adaptive equaliser diverged (mean |e|^2 > 1 or non-finite taps) */
  uint32_t reserved;
} kk_rx_counts;

/* Fill *p with defaults (tone_bin 541065, mu 1e-3, K 4096, L 0, tau -1,
 * DD_SOFT, v_min 1, device -1, max_batch 16; pointers NULL).  Host only. */
void kk_rx_params_default(kk_rx_params *p);

/* Create a receiver.  fmt: kk_format; sps must be 4 (4 -> 2);
 * buffer_len: samples per buffer (2^22 in the paper), multiple of 512,
 * >= 4*k_update + 3200, <= 2^30; cspr_db: carrier-to-signal power ratio used
 * for carrier removal A_hat = sqrt(d c/(1+c)) (reading R6).
 * Copies every table it needs from *p (the caller may free them after).
 * Allocates device memory on p->device.  Errors: KK_EINVAL (bad params),
 * KK_ENOMEM, KK_ECUDA (no device). */
kk_status kk_rx_create(kk_rx_t **out, int fmt, int sps, int64_t buffer_len, float cspr_db,
                       const kk_rx_params *p);

/* Samples that must be readable before the first and after the last sample of
 * the buffers passed to kk_rx_process*.  Outputs of buffer b depend only on
 * raw samples [b*N - left, (b+1)*N + right). */
kk_status kk_rx_halo(const kk_rx_t *h, int64_t *left, int64_t *right);

/* Same, without a handle (host only; for sizing and tests). */
kk_status kk_rx_halo_for(int64_t buffer_len, int32_t k_update, int64_t *left, int64_t *right);

/* Process one buffer.  `buffer` points at its first sample inside a contiguous
 * caller-owned stream (device or host memory; halos readable).  out_symbols:
 * buffer_len/4 bytes (device or host), each the bit label of the decided point
 * ("demapped into bits").  out_errors: host struct, may be NULL.
 * Returns when the outputs are valid.  Advances the stream position by one
 * buffer (pattern offset for error counting). */
kk_status kk_rx_process(kk_rx_t *h, const int16_t *buffer, uint8_t *out_symbols, kk_rx_counts *out_errors);

/* Process nbuf consecutive buffers starting at `first` (contiguous stream).
 * out_symbols: nbuf*buffer_len/4 bytes or NULL; out_per_buf: nbuf host structs
 * or NULL.  Internally batched (max_batch) and pipelined: with host input the
 * copy of batch j+1 overlaps the compute of batch j. */
kk_status kk_rx_process_batch(kk_rx_t *h, const int16_t *first, int64_t nbuf, uint8_t *out_symbols,
                              kk_rx_counts *out_per_buf);

/* Asynchronous submission (the streaming receiver).
 * Enqueues nbuf consecutive buffers starting at `first` (contiguous stream, halos
 * readable; device memory, or host memory staged through the handle's copy stream)
 * and returns without waiting.  The library keeps two batches in flight: the LMS
 * update pass of batch j (one SM) runs concurrently with the fused chain of batch
 * j-1, and that chain launch also computes batch j's update-pass x2 tails.  The
 * chain of the newest batch is launched by the next submit or by kk_rx_sync.
 * Results equal kk_rx_process_batch on the same buffers bit for bit.
 * Memory: the first submission (and any larger nbuf later) allocates the device staging
 * of every pipeline slot at once (tails, taps, counters, labels, and for host or packed
 * input a copy of the batch + halos), so steady-state submits never allocate.
 * Host input: page-locked memory (cudaHostAlloc / cudaHostRegister / torch pin_memory) is
 * copied by DMA straight from the caller's buffer; PAGEABLE host memory is first copied by
 * host threads into a pinned staging buffer of the pipeline slot (allocated once, then
 * reused) and DMA'd from there, so it keeps the copy/compute overlap at the cost of one host
 * memcpy (the submit call returns after that memcpy).  kk_rx_pageable_staged counts them.
 * `first` (and the halos) must stay valid and unmodified until kk_rx_sync returns;
 * input written by the caller on the handle's cuda_stream before the call is
 * honoured (stream order).  out_symbols: nbuf*buffer_len/4 bytes (device or host)
 * or NULL; valid after kk_rx_sync.  Advances the stream position by nbuf.
 * Errors: KK_EUNSUPPORTED with sub_block < buffer_len/4 or debug dumps; KK_EINVAL
 * for bad arguments or nbuf > 4096. */
kk_status kk_rx_submit_batch(kk_rx_t *h, const int16_t *first, int64_t nbuf, uint8_t *out_symbols);

/* Same as kk_rx_submit_batch for the packed 12-bit ADC format: two two's-complement
 * 12-bit codes per 3 bytes, little-endian (b0 = c0[7:0], b1 = c0[11:8] | c1[3:0] << 4,
 * b2 = c1[11:4]); `first` points at the byte of the first buffer's first sample (its
 * sample index must be even), the halos are readable in the same format.  Host or device
 * memory; the handle copies 1.5 bytes per sample (host input: over PCIe on its copy stream)
 * and unpacks on the GPU.  Results are bit-identical to the int16 path on the same codes.
 * Errors as kk_rx_submit_batch; KK_EUNSUPPORTED if the halos or buffer_len are not
 * multiples of 8 samples. */
kk_status kk_rx_submit_batch_packed12(kk_rx_t *h, const uint8_t *first, int64_t nbuf, uint8_t *out_symbols);

/* Finish every submitted batch and return their per-buffer counters in submission
 * order: up to max_out structs to out_per_buf (may be NULL), the total count to
 * *n_out (may be NULL).  Blocks until all outputs are valid. */
kk_status kk_rx_sync(kk_rx_t *h, kk_rx_counts *out_per_buf, int64_t max_out, int64_t *n_out);

/* Change the DC offset d (the offset lost by the AC-coupled ADC, swept offline)
 * for subsequent submissions and calls; A_hat = sqrt(d c/(1+c)) follows (reading R6).
 * Batches already submitted keep the offset they were submitted with.  KK_EINVAL if d <= 0. */
kk_status kk_rx_set_dc_offset(kk_rx_t *h, float dc_offset);

/* DC-offset sweep, the paper's measurement procedure (every measurement is
 * repeated with different DC offsets, the best Q kept): the nbuf buffers at `first` (as in
 * kk_rx_submit_batch) are processed once per offset dc_values[0..nd-1] (each a full S1-S7
 * pass, back to back through the streaming pipeline; labels are not returned).
 * out_per_dc: nd host structs (counters summed over the buffers) or NULL; *best: index of
 * the lowest bit-error ratio (first on ties).  KK_ESTATE while submitted batches are not
 * yet synced (kk_rx_sync first: their counters are the caller's).  The hypothesis passes
 * do not count as traffic: kk_rx_totals is unchanged by the call.  Restores the handle's DC
 * offset and advances the stream position by nbuf.  KK_EINVAL for bad arguments or
 * non-positive offsets. */
kk_status kk_rx_dc_sweep(kk_rx_t *h, const int16_t *first, int64_t nbuf, const float *dc_values, int nd,
                         kk_rx_counts *out_per_dc, int *best);

/* Generalised sweep ("batched DC-offset (and CSPR-hypothesis)
 * sweep"): hypothesis k uses DC offset dc_values[k] and, when cspr_db_values != NULL,
 * CSPR cspr_db_values[k] (A_hat = sqrt(d c/(1+c)), c = 10^(CSPR/10), reading R6); NULL
 * keeps the handle's CSPR (= kk_rx_dc_sweep).  Same outputs and conventions as
 * kk_rx_dc_sweep; the handle's offset and CSPR are restored afterwards.
 * KK_EINVAL: dc <= 0, |CSPR| >= 60 dB, nd <= 0, nbuf <= 0. */
kk_status kk_rx_sweep(kk_rx_t *h, const int16_t *first, int64_t nbuf, const float *dc_values,
                      const float *cspr_db_values, int nd, kk_rx_counts *out_per_hyp, int *best);

/* Set the CSPR hypothesis (dB) of the handle: A_hat = sqrt(d c/(1+c)) with the current DC
 * offset.  Takes effect for batches submitted afterwards.  KK_EINVAL if |CSPR| >= 60 dB. */
kk_status kk_rx_set_cspr(kk_rx_t *h, float cspr_db);

/* Frame synchronisation (the first init-time step; PAPER l.53,
 * l.64: the 2^20-symbol PCG64 pattern is known).  Computes E_s of one buffer (same
 * conventions as kk_rx_process) and correlates its symbol-instant samples
 * y_n = E_s[4 (n0 + n)], n < n_corr, with the pattern points over every cyclic lag k:
 *   c(k) = sum_n y_n conj(points[pattern[(n0 + n + k) mod P]]);
 * *n_off = argmax_k |c(k)| (lowest k on ties): the symbol sent at buffer index n is
 * pattern[(n + n_off) mod P] -- pass it as ref_offset / to kk_rx_train_fir's symbols.
 * peak (2 floats, or NULL): c(n_off); peak_to_mean (or NULL): |c(n_off)|^2 / mean_k |c(k)|^2.
 * Needs ref_pattern; 16 <= n_corr <= 8192; 4*(n0+n_corr-1) < buffer_len.  KK_ESTATE while
 * the streaming pipeline holds batches. */
kk_status kk_rx_frame_sync(kk_rx_t *h, const int16_t *buffer, int64_t n0, int32_t n_corr, int64_t *n_off,
                           float *peak, double *peak_to_mean);

/* Init-time training (the static equaliser "is optimized offline using a
 * training sequence every time that the data acquisition is initialized"; the adaptive
 * equaliser converges "using a training sequence").  All three need an idle streaming
 * pipeline (KK_ESTATE otherwise).
 *
 * kk_rx_train_fir: least-squares 203-tap static equaliser (reading R4) on ONE buffer
 * (`buffer` as for kk_rx_process, device or host, halos readable) whose transmitted
 * symbols [n_first, n_first + n_count) are known: symbols = 2*n_count floats (re, im).
 * min_h sum_n |sum_t h_t E_s[4n + 101 - t] - s_n|^2 + ridge tr(R)/203 |h|^2, E_s from the
 * GPU's S1-S3, normal equations and Cholesky solve in fp64 on the GPU.  Needs
 * 4*n_first >= 101 and 4*(n_first+n_count-1)+101 < buffer_len.  out_fir: 2*203 floats
 * (the layout of kk_rx_params.fir); not applied (see kk_rx_set_fir).
 *
 * kk_rx_set_fir: replace the static equaliser (2*203 floats; the EQ spectrum is recomputed
 * in fp64 as at create).
 *
 * kk_rx_train_taps: the widely-linear taps after k_steps LMS steps in PILOT mode (known
 * ref_pattern, from the handle's W_init and mu) over symbols [0, k_steps) of one buffer at
 * the handle's stream position; out_w: 16 floats in the layout of kk_rx_params.w_init.
 * KK_EINVAL without ref_pattern.  kk_rx_set_w_init installs such taps as W_init. */
kk_status kk_rx_train_fir(kk_rx_t *h, const int16_t *buffer, const float *symbols, int64_t n_first, int64_t n_count,
                          double ridge, float *out_fir);
kk_status kk_rx_set_fir(kk_rx_t *h, const float *fir);
kk_status kk_rx_train_taps(kk_rx_t *h, const int16_t *buffer, int32_t k_steps, float *out_w);
kk_status kk_rx_set_w_init(kk_rx_t *h, const float *w);

/* GMI of constellations in complex AWGN (the GS optimiser's objective;
 * SURVEY 8(f) NEXT-4), on the current CUDA device: standard BICM GMI (bits per symbol),
 * Es = 1, N0 = 10^(-snr_db/10), expectation by 2-D Gauss-Hermite quadrature of `order`
 * nodes per dimension.  points: n_cand * 2*m floats (re, im; candidate c at c*2*m),
 * labels: n_cand * m bit labels (permutations of 0..m-1), m a power of two <= 256.
 * out_gmi: n_cand doubles.  Blocking.  KK_EINVAL for bad arguments, KK_ECUDA. */
kk_status kk_gmi_awgn(const float *points, const uint8_t *labels, int m, int n_cand, double snr_db, int order,
                      double *out_gmi);

/* Host only: Gauss-Hermite nodes and weights (weight e^{-t^2}, ascending nodes), Golub-Welsch.
 * Returns order (1..64) or -1. */
int kk_hermgauss(int order, double *nodes, double *weights);

/* Kernel launches issued by submit/sync since the previous call of this function. */
int64_t kk_rx_async_launches(kk_rx_t *h);

/* Number of kk_rx_submit_batch calls whose PAGEABLE host input was staged through a pipeline
 * slot's pinned buffer (see kk_rx_submit_batch); host-only read, never fails for a valid handle.
 * KK_EINVAL: NULL handle or n. */
kk_status kk_rx_pageable_staged(const kk_rx_t *h, int64_t *n);

/* Set the stream index of the next buffer (pattern offset = ref_offset +
 * index*buffer_len/4 mod ref_len).  Default after create: 0. */
kk_status kk_rx_seek(kk_rx_t *h, int64_t buffer_index);

/* Adaptive taps used for buffer `buf` (0-based) of the LAST internal batch of
 * the last call: 16 floats (w[4], g[4] complex) per sub-block, all sub-blocks. */
kk_status kk_rx_get_taps(kk_rx_t *h, int64_t buf, float *out);

/* Running totals since create / kk_rx_reset_totals. */
kk_status kk_rx_totals(const kk_rx_t *h, kk_rx_counts *out);
kk_status kk_rx_reset_totals(kk_rx_t *h);

/* Debug (parity tests): x2 (S4 output, 2 sps) of the last internal batch,
 * x2 index relative to that batch's first buffer (x2 index m <-> 4-sps position
 * 2m); valid range [-(2*k_update+2), nbuf*buffer_len/2) with KK_DUMP_X2 (or
 * sub_block < buffer_len/4); otherwise only the update-pass tails
 * [b*N/2 - 2*k_update - 2, b*N/2) are defined.  2*count floats. */
kk_status kk_rx_debug_x2(kk_rx_t *h, int64_t first, int64_t count, float *out);

/* Debug: E_s (S3 output, 4 sps) of the last internal batch (needs
 * KK_DUMP_ES at create), positions [0, nbuf*buffer_len). 2*count floats. */
kk_status kk_rx_debug_es(kk_rx_t *h, int64_t first, int64_t count, float *out);

/* Built-in constellation table (host only): 2*m floats, m labels. Returns m or <0. */
int kk_rx_constellation(int fmt, float *points_out, uint8_t *labels_out);

/* Host-only (tests): the two exact decision look-up tables the kernels use, built
 * for `points` (2*m floats, re/im) and soft-gate `tau` (0 = hard / PILOT).
 * lms_cells: 2*G*G floats (G = return value, 128): per cell (row-major, cell
 * (cx,cy) at cy*G+cx) either the coordinates of the unique point that is nearest
 * everywhere in the cell with every other point >= tau farther (FAST), or
 * (NaN, bits of a word of 4 ascending 8-bit candidate indices, 128 = none;
 * 0xffffffff = brute force) (SLOW).  Cell of y: floor(clamp(y*linv + lc, 0, G-1)),
 * lms_geom = (lcx, lcy, linv).  dec_cells: g*g words of the fused chain's decision
 * table (4 ascending 7-bit candidates, bit 31 = brute force), g <= 128;
 * dec_geom = (x0, y0, inv, g), g = 0 when m <= 8 (brute force only).  Any output
 * may be NULL.  Returns G, or -1 (bad arguments). */
int kk_rx_decision_tables(const float *points, int m, float tau, float *lms_cells, float *lms_geom,
                          uint32_t *dec_cells, float *dec_geom);

/* Number of kernel launches issued by the last process call (for the bench). */
int64_t kk_rx_last_launches(const kk_rx_t *h);

/* Per-kernel device timing (CUDA events recorded on the launch stream around
 * each kernel of every internal batch).  kk_rx_set_timing(h, 1) enables and
 * resets; kk_rx_kernel_times returns accumulated milliseconds and launch
 * counts of 3 slots: [0] S1-S4 x2 pass (update-pass tails, or the whole batch
 * when sub_block < buffer), [1] the LMS update pass, [2] the fused
 * S1-S7 chain kernel (or the apply kernel when sub_block < buffer). */
kk_status kk_rx_set_timing(kk_rx_t *h, int on);
kk_status kk_rx_kernel_times(const kk_rx_t *h, double *ms_out, int64_t *n_out);

/* Message for the last failure on this thread (never NULL). */
const char *kk_rx_last_error(const kk_rx_t *h);

/* Free everything; NULL is a no-op. */
kk_status kk_rx_destroy(kk_rx_t *h);

int kk_rx_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KK_RX_H */
