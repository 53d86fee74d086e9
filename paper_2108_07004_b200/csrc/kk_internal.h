// kk_internal.h -- launch-argument structs shared by the host API and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace kk {

// Geometry of the fused chain kernel.
//   Hilbert chunk grid: 512 samples, window 1024 centred (reading R2)
//   EQ grid           : overlap-save NF = 1024, keep 768 (margin 128 >= 101 FIR
//                       reach), blocks start at owner position -128 + 768 j
//   one CTA step      : 3072 samples = 3 Hilbert FFT pairs + 4 EQ blocks
//                       (+ 768 symbols of WL apply / decision in APPLY mode)
constexpr int STEP = 3072;
constexpr int EQ_KEEP = 768;
constexpr int EBUF = STEP + 256;    // D = E_tf - A_hat window of one step: [3072 i - 256, 3072 i + 3072)
constexpr int STG = STEP + 512;     // codes of one step: [3072 i - 256, 3072 i + 3328)
constexpr int WARM = 1536;          // warm-up codes: [3072 i - 1280, 3072 i + 256)
constexpr int PKH = 8;              // extra codes staged per side (pre-KK equaliser reach, <= 8)
constexpr int STG2 = STG + 2 * PKH;   // staged codes of one step: [3072 i - 256 - PKH, ...)
constexpr int WARM2 = WARM + 2 * PKH; // staged warm-up codes
constexpr int XS = 1848;            // x2 window of one step (APPLY, 1538 used): positions 3072 i - 132 + 2 j;
                                    // pre-KK: the step's 112 padded v' rows (112 x 33 floats) in phase H
constexpr int NWARPS = 4;          // warps per group
#ifndef KK_NGROUP
#define KK_NGROUP 4
#endif
constexpr int NGROUP = KK_NGROUP;  // independent groups per CTA (one CTA per SM)
constexpr int TILE = 32 * 33;       // per-warp transpose tile (floats)
constexpr int SYM_PER_STEP = 768;
constexpr int MAX_SEG = 4;

enum SegMode { SEG_APPLY = 0, SEG_X2_TAIL = 1, SEG_X2_FULL = 2 };

// exact decision look-up table (built on the host):
// cell word = 4 ascending 7-bit point indices (bits 7c .. 7c+6; short lists are
// padded with their first index) | bit 31 = brute force (crowded cell)
struct DecLut {
  const uint32_t* cell;            // [g*g]
  float x0, y0, inv;               // cell (cx, cy) covers [x0 + cx/inv, ...); -x0*inv, -y0*inv are half-integers
  int g;                           // grid size (0 = no LUT: always brute force), 64 or 128
  float cxm, cym;                  // -x0*inv - 1/2 + 2^23 (exact): y*inv + cxm rounds to floor(cell) + 2^23
  int lg;                          // log2(g)
};

// A segment of the step list: owners o = owner_first + k (k in [0, n_own)),
// steps [i_begin, i_end) of each.  Owner o's codes start at codes + o*N.
struct Seg {
  int32_t owner_first, n_own, i_begin, i_end;
  int32_t mode;            // SegMode
  int32_t count_clip;      // count clipped samples of positions [0, N) (APPLY / FULL)
  int32_t ref;             // FULL: owner whose position 0 is x2dst[0]; TAIL/APPLY: index base
  int32_t pad;
  float2* x2dst;           // TAIL: [k][X2H] tails; FULL: x2 index 0 of owner `ref`
  uint8_t* out;            // APPLY: labels of owner owner_first
  unsigned long long* counts;  // [k][8]
  const float2* taps;      // APPLY: [k][8]
  int64_t n_off;           // APPLY: pattern index of symbol 0 of owner owner_first
  const int16_t* codes;    // owner o's samples start at codes + o*N (halos readable)
  float dc, a_hat;         // DC offset d and carrier amplitude A_hat of this segment's batch
  float prek_dsum;         // d * sum(pre-KK taps) (pre-KK equaliser only)
};

// LMS update-pass look-up table (built on the host):
// G x G cells (G a power of two) over the constellation's bounding box (+2 d_min).
// Entry of cell (cx, cy) = float2:
//   (px, py)          FAST: one point k is the nearest everywhere in the cell AND
//                     every other point is >= tau farther (soft gate = 1): ref = p_k
//   (NaN, bits(word)) SLOW: word = 4 ascending 8-bit point indices (128 = none)
//                     holding every point that can be nearest or within tau of the
//                     nearest anywhere in the cell; word = ~0u: brute force
// The outermost ring of cells is always SLOW/brute (y is clamped into the grid).
constexpr int LMS_LUT_G = 128;
constexpr int GRAM_SPLIT = 16;  // train_fir: training symbols split over grid.z (partial R/b planes, fixed-order sum)
constexpr uint32_t LMS_BRUTE = 0xffffffffu;


struct LmsArgs {
  const float2* lut;       // [G*G] entries
  float lcx, lcy, linv;    // cell coordinate = y * linv + lc (clamped to [0, G-1])
  const float2* x2_b0;     // x2 index 0 (position 0) of chain buffer 0
  int64_t x2_stride;       // x2 samples between consecutive buffers' position 0
  int64_t n_sym;           // symbols per buffer
  int64_t L;               // sub-block
  int32_t nsub;            // n_sym / L
  int32_t nchains;         // nbuf * nsub
  int32_t K;
  float mu, inv_tau;
  int32_t mode;
  int32_t m;
  const float2* pts;       // [m]
  const uint8_t* pattern;  // [P] or nullptr
  int64_t P;
  int64_t n_off0;          // pattern offset of buffer 0
  const float2* w_init;    // [8]
  float2* taps;            // [nchains][8]
  unsigned long long* counts;  // [nbuf][8]
  const unsigned long long* wait_ctr;  // lane kernel: spin until *wait_ctr >= wait_target (x2 tails ready)
  unsigned long long wait_target;
};

struct ChainArgs {
  int64_t N;               // buffer_len
  int32_t nseg;
  Seg seg[MAX_SEG];
  int64_t total_steps;
  int64_t x2h;             // tail length (x2 samples) = 2K + 64
  float dc, vmin, a_hat, invN;
  uint32_t tb_mod, s32;    // tone_bin mod N, (tb*32) mod N
  float2 rot[16];          // e^{2 pi i ((tb 32 r) mod N) / N}, r = 0..15 (EQ output downconversion)
  const float2* tw1024;    // [32*32] e^{-2 pi i r l / 1024}
  const float2* tw512;     // [16*32] e^{-2 pi i r l / 512}
  const float2* Hs;        // [1024] DFT of the tone-shifted h, / 1024 (reading R5 + downconversion)
  float2* es_dump;         // debug: E_s of owners >= 0 of FULL segments, [owner*N + p], or nullptr
  int aligned16;
  int64_t n_sym;
  int32_t m;
  const float2* pts;       // [m]
  const uint8_t* labels;   // [m]
  const uint8_t* pattern;  // [P] or nullptr
  int64_t P;
  int32_t pat_tma;         // pattern staged by bulk copies (P % 16 == 0)
  DecLut lut;
  // work distribution: work_ctr == nullptr -> static contiguous ranges per group; else
  // dynamic grabs from *work_ctr (zeroed before the launch): whole owners of a leading
  // SEG_X2_TAIL segment first, then guided chunks
  unsigned long long* work_ctr;
  unsigned long long* tail_ctr;  // if set: += 1 (release) after every finished SEG_X2_TAIL step
  // the LMS update pass of the next batch as extra CTAs of this launch (the last lms_ctas
  // blocks; lane-per-chain body, waits on tail_ctr for the tails this launch computes)
  int32_t lms_ctas, lms_mode;
  int32_t lms_warp;  // extra CTAs run the warp-per-chain update pass (one chain each) instead of lanes
  LmsArgs lms;
  // pre-KK intensity equaliser: v' = sum_{k=-h..h} prek[k+h] code[n-k] + dsum,
  // dsum = d * sum(prek) per segment (Seg.prek_dsum); prek_h < 0: off (the plain kernel)
  int32_t prek_h;
  float prek[2 * PKH + 1];
  // diagnostics (KKRX_PHASE_TIMING): per-group clock64 sums [0] staging, [1] phase H,
  // [2] phase E, [3] phase A + step tail, [4] steps, [5] H task busy (3 warps), [6] E task busy (4 warps)
  unsigned long long* dbg;
};

struct ApplyArgs {
  const float2* x2;        // x2 index 0 of buffer 0 (full layout, stride N/2)
  int64_t n_sym, L;
  int32_t nsub;
  int64_t total;           // nbuf * n_sym
  int32_t m;
  const float2* pts;
  const uint8_t* labels;
  const uint8_t* pattern;
  int64_t P, n_off0;
  const float2* taps;
  uint8_t* out;
  unsigned long long* counts;
  DecLut lut;
};

// counter slots
enum { C_BITERR = 0, C_SYMERR = 1, C_BITS = 2, C_SYMS = 3, C_CLIP = 4, C_GATED = 5, C_FLAGS = 6, C_ESUM = 7 };

size_t chain_smem_bytes();
cudaError_t chain_setup(int device, int* grid_out);
cudaError_t lms_setup();
cudaError_t launch_chain(const ChainArgs& a, int grid, cudaStream_t s);
cudaError_t launch_lms(const LmsArgs& a, cudaStream_t s);
cudaError_t launch_lms_lanes(const LmsArgs& a, cudaStream_t s);
int lms_lanes_ctas(int nchains);
cudaError_t launch_apply(const ApplyArgs& a, cudaStream_t s);
cudaError_t launch_frame_sync(const float2* es, int64_t es_first, int L, const uint8_t* pattern, int64_t P, int64_t n0,
                              const float2* pts, int m, unsigned long long* best, double* sum2, float2* cval,
                              cudaStream_t s);
cudaError_t launch_train_fir(const float2* es, int64_t pos_first, const float2* sym, int n_count, int ntap, double ridge,
                             double2* R, double2* b, float* out, cudaStream_t s);
cudaError_t launch_gmi(const float2* pts, const uint8_t* labs, int m, int nb, const double2* nodes, const double* wts,
                       int nq, double n0, int n_cand, double* out, cudaStream_t s);
cudaError_t launch_unpack12(const uint8_t* src, int16_t* dst, int64_t n_samples, cudaStream_t s);

}  // namespace kk
