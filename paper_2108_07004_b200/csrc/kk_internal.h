// kk_internal.h -- launch-argument structs shared by the host API and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace kk {

// Geometry of the fused S1-S4 kernel.
//   Hilbert chunk grid: 512 samples, window 1024 centred (reading R2)
//   EQ grid           : overlap-save NF = 1024, keep 768 (margin 128 >= 101 FIR
//                       reach), blocks start at owner position -128 + 768 j
//   one CTA step      : 3072 samples = 3 Hilbert FFT pairs + 4 EQ blocks
constexpr int STEP = 3072;
constexpr int EQ_KEEP = 768;
constexpr int EBUF = STEP + 256;    // E_s window of one step: [3072 i - 256, 3072 i + 3072)
constexpr int STG = STEP + 512;     // codes of one step: [3072 i - 256, 3072 i + 3328)
constexpr int X2_WARPS = 4;
constexpr int TILE = 32 * 33;       // per-warp transpose tile (float2)

struct X2Args {
  const int16_t* codes;    // sample 0 of batch buffer 0 (halos readable)
  int64_t N;               // buffer_len
  int32_t steps_per_buf;   // S_N
  int32_t pre_first_step;  // i0 of the halo pre-pass (owner -1)
  int32_t pre_steps;       // S_N - i0, or 0
  int32_t nbuf;
  int64_t total_steps;
  float dc, vmin, a_hat, invN;
  uint32_t tb_mod, s32, s512;  // tone_bin mod N, (tb*32) mod N, (tb*512) mod N
  float2* x2;              // x2 index 0 (= position 0 of batch buffer 0); valid down to x2_lo
  int64_t x2_lo;
  const float2* tw1024;    // [32*32] e^{-2 pi i r l / 1024}
  const float2* tw512;     // [16*32] e^{-2 pi i r l / 512}
  const float2* H;         // [1024] DFT of circularly placed h, / 1024
  unsigned long long* counts;  // [nbuf][8]
  float2* es_dump;         // debug: E_s at batch positions [0, nbuf*N) or nullptr
  int aligned16;
};

struct LmsArgs {
  const float2* x2;        // x2 index 0
  int64_t n_sym;           // symbols per buffer
  int64_t L;               // sub-block
  int32_t nsub;            // n_sym / L
  int32_t nchains;         // nbuf * nsub
  int32_t K;
  float mu, tau;
  int32_t mode;
  int32_t m;
  const float2* pts;       // [m]
  const uint8_t* pattern;  // [P] or nullptr
  int64_t P;
  int64_t n_off0;          // pattern offset of batch buffer 0
  const float2* w_init;    // [8]
  float2* taps;            // [nchains][8]
  unsigned long long* counts;  // [nbuf][8]
};

struct ApplyArgs {
  const float2* x2;
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
};

// counter slots
enum { C_BITERR = 0, C_SYMERR = 1, C_BITS = 2, C_SYMS = 3, C_CLIP = 4, C_GATED = 5, C_FLAGS = 6, C_ESUM = 7 };

size_t x2_smem_bytes();
cudaError_t launch_x2(const X2Args& a, int grid, cudaStream_t s);
cudaError_t launch_lms(const LmsArgs& a, cudaStream_t s);
cudaError_t launch_apply(const ApplyArgs& a, cudaStream_t s);
int x2_occupancy_grid(int device);

}  // namespace kk
