// kk_kernels.cu -- sm_100a kernels of the KK receiver hot path.
//
//   kk_chain_kernel<PREKK>   the whole per-sample chain, fused, one 512-thread CTA per SM
//       (4 groups x 4 warps): S1 front end, S2 blockwise Hilbert, S3 reconstruction +
//       carrier removal, S4 static EQ with 4->2 fold and downconversion, S5' fixed-tap WL
//       apply, S6 decision, S7 demap + count.  Reads int16 codes, writes uint8 labels;
//       E_s and x2 never leave shared memory.  Segment modes: APPLY (labels), X2_TAIL (the
//       x2 tails the next batch's LMS pass reads), X2_FULL (debug / sub_block < N/4).
//       PREKK = the optional pre-KK intensity FIR fused into the S1/S3 code reads.  The
//       last CTAs of a streaming launch run the next batch's S5 update pass
//       (lms_lanes_body: lane per chain, or lms_warp_cta: warp per chain for few chains)
//       and then join the chain work.
//   kk_lms_kernel    S5 update pass: one warp per sub-block chain of K steps
//                    (sequential, "significant time", few resources)
//   kk_lms_lanes_kernel  the same pass with one lane per chain (one SM for a batch)
//   kk_apply_kernel  S5'-S7 from materialised x2 (sub_block < buffer only)
//   kk_unpack12_kernel   packed 12-bit ADC bytes -> int16 codes (host-input path)
//   kk_gram_kernel / kk_chol_solve_kernel   init-time LS fit of the static EQ (fp64)
//   kk_fsync_kernel  init-time frame synchronisation against the PCG64 pattern
//   kk_gmi_kernel    batched AWGN GMI of constellations (GS optimiser workload)
//
// No tensor cores: nothing here is a dense contraction.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kk_fft.cuh"
#include "kk_internal.h"

#ifndef KK_GUIDE_DIV
#define KK_GUIDE_DIV 4   // guided chunks: remaining steps / (KK_GUIDE_DIV x groups), at most KK_GUIDE_MAX
                         // (measured: 2 / 256 costs the plain chain 11 %, gains the pre-KK one 2.4 %)
#endif
#ifndef KK_GUIDE_MAX
#define KK_GUIDE_MAX 64
#endif
#ifndef KK_A_ROUNDS
#define KK_A_ROUNDS 3  // phase A: each thread's 6 symbols in this many rounds (3: -3 % vs 1, code size)
#endif
#ifndef KK_S3_UNROLL
#define KK_S3_UNROLL 2  // S3 output loop unroll (code size vs exposed code-load latency)
#endif
#ifndef KK_PHASE_TIMING
#define KK_PHASE_TIMING 0
#endif

namespace kk {

constexpr int S3_UNROLL = KK_S3_UNROLL;
template <int V>
struct IntC {
  static constexpr int value = V;
};

// compile-time phase tag of unrolled loop bodies
template <int Q>
struct Phase {
  static constexpr int value = Q;
};

// one CTA per SM = NGROUP independent 4-warp groups (each the former 128-thread CTA,
// synchronised by its own named barrier) sharing one copy of the read-only tables
constexpr size_t SMEM_TW = 1024 * sizeof(float2);     // 1024-pt twiddles
constexpr size_t SMEM_H = 1024 * sizeof(float2);      // static-EQ spectrum Hs
constexpr size_t SMEM_TW512 = 512 * sizeof(float2);   // 512-pt twiddles
constexpr size_t SMEM_LUT = 64 * 64 * sizeof(uint32_t);  // decision table (g <= 64)
#if KK_TMEM_TABLES
constexpr size_t SMEM_SHARED = SMEM_LUT;  // the per-lane twiddle / EQ tables live in TMEM (kk_fft.cuh)
#else
constexpr size_t SMEM_SHARED = SMEM_TW + SMEM_H + SMEM_TW512 + SMEM_LUT;
#endif
constexpr size_t SMEM_EBUF = EBUF * sizeof(float2);
constexpr size_t SMEM_STG = STG2 * sizeof(int16_t);
static_assert(SMEM_STG % 16 == 0 && (PKH * 2) % 16 == 0, "bulk copies of the staged codes stay 16-B aligned");
constexpr size_t SMEM_XS = XS * sizeof(float2);  // also holds the warm-up codes (WARM int16)
constexpr size_t SMEM_PAT = 832;                 // pattern bytes of one step (768 + alignment)
constexpr size_t SMEM_GROUP0 = SMEM_EBUF + SMEM_STG + SMEM_XS + SMEM_PAT + 64 + 16;  // + factored WL taps + mbarriers
// + the row-31 pads of the FFT transpose tiles (kk_fft.cuh fft1024): 48 float2 per warp role,
// the pad placed at the bank offset its tile needs; group regions 128-B aligned
constexpr size_t SMEM_PADS = NWARPS * 48 * sizeof(float2);
constexpr size_t SMEM_GROUP = ((SMEM_GROUP0 + 127) / 128) * 128 + SMEM_PADS;
constexpr size_t SMEM_LMS_NEED = LMS_LUT_G * LMS_LUT_G * 8 + (2 * 5632 + 16) * 8 + 130 * 8 + 8;
constexpr size_t CHAIN_SMEM0 = SMEM_SHARED + NGROUP * SMEM_GROUP;
constexpr size_t CHAIN_SMEM = CHAIN_SMEM0 > SMEM_LMS_NEED ? CHAIN_SMEM0 : SMEM_LMS_NEED;  // the LMS CTAs reuse it
static_assert(SMEM_GROUP % 128 == 0 && SMEM_SHARED % 128 == 0, "128-B aligned regions");
static_assert((SMEM_EBUF + SMEM_STG) % 16 == 0, "x2 window 16-B aligned (phase A reads it with 128-bit loads)");
static_assert(LMS_LUT_G * LMS_LUT_G * 8 + 129 * 8 <= CHAIN_SMEM, "LMS CTAs fit the chain smem");
static_assert(SMEM_LMS_NEED <= CHAIN_SMEM,
              "warp-per-chain LMS CTAs (table + x2 window + points + mbarrier) fit the chain smem");
static_assert(WARM2 * sizeof(int16_t) + 1023 * sizeof(float2) <= SMEM_XS, "warm-up codes + its 31 x 33 float2 tile fit the x2 window");
static_assert((WARM2 * sizeof(int16_t)) % 8 == 0, "warm-up tile float2-aligned");
constexpr int WOFF = WARM2 * (int)sizeof(int16_t) / (int)sizeof(float2);  // float2 offset of the warm-up tile in xs
static_assert(TILE * sizeof(float) <= EQ_KEEP * sizeof(float2), "transpose tile must fit an EQ stride of ebuf");
static_assert(XS >= 1024 && 3 * 1024 <= STEP, "E-phase 64-bit transpose tiles: three in ebuf[0, STEP), one in xs");
static_assert((STEP + 512) / 32 * 33 * sizeof(float) <= SMEM_XS, "pre-KK v' rows of a step fit the x2 window");

size_t chain_smem_bytes() { return CHAIN_SMEM; }

__device__ __forceinline__ uint32_t add_mod(uint32_t q, uint32_t s, uint32_t n) {
  const uint32_t r = q + s;
  return (r >= n) ? r - n : r;
}

__device__ __forceinline__ uint32_t tone_index(const ChainArgs& a, int64_t pos) {
  // (tone_bin * pos) mod N, exact (reading R7); pos may be negative (halo)
  int64_t r = ((int64_t)a.tb_mod * pos) % a.N;
  if (r < 0) r += a.N;
  return (uint32_t)r;
}

// MUFU forms without the denormal fix-ups of the CUDA math wrappers (arguments here are
// >= v_min > 0, far from the denormal range)
__device__ __forceinline__ float lg2_ftz(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrt_ftz(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// sin/cos of an angle that needs no range reduction (|x| of a few pi: the hardware
// works in turns, so only the fp32 precision of x / 2 pi matters)
__device__ __forceinline__ void sincos_small(float x, float* s, float* c) {
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(*s) : "f"(x));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(*c) : "f"(x));
}

__device__ __forceinline__ void cis_turns(float t, float* s, float* c) {
  // e^{2 pi i t} for any t, with exact reduction to [-1/2, 1/2] before __sincosf
  t -= rintf(t);
  sincos_small(t * 6.2831853071795865f, s, c);
}

// Exact minimum-distance decision (ties -> lowest index, reading R11): the LUT
// cell lists (ascending) every point that can be nearest anywhere in the
// (slightly enlarged) cell; brute force outside the grid or for crowded cells.
constexpr uint32_t LUT_BRUTE = 1u << 31;

// table in shared memory (s_cells, g <= 64) or global (L.cell)
__device__ __forceinline__ uint32_t lut_word(float2 y, const DecLut& L, const uint32_t* s_cells, bool in_smem) {
  if (L.g > 0) {
    const float fx = (y.x - L.x0) * L.inv, fy = (y.y - L.y0) * L.inv;
    if (fx >= 0.f && fy >= 0.f && fx < (float)L.g && fy < (float)L.g) {
      const int c = (int)fy * L.g + (int)fx;
      return in_smem ? s_cells[c] : __ldg(L.cell + c);
    }
  }
  return LUT_BRUTE;
}

__device__ __noinline__ int decide_brute(float2 y, const float2* __restrict__ sp, int m) {
  float best = __int_as_float(0x7f800000);
  int kb = 0;
  for (int k = 0; k < m; ++k) {
    const float dx = y.x - sp[k].x, dy = y.y - sp[k].y;
    const float d = fmaf(dx, dx, dy * dy);
    if (d < best) {
      best = d;
      kb = k;
    }
  }
  return kb;
}

// 4 candidates, branch-free (ascending order + strict < = lowest index on ties;
// padded duplicates never replace); crowded / off-grid -> brute force (rare)
__device__ __forceinline__ int decide_word(float2 y, uint32_t w, const float2* __restrict__ sp, int m) {
  if (w & LUT_BRUTE) return decide_brute(y, sp, m);
  int kb = (int)(w & 127u);
  float dx = y.x - sp[kb].x, dy = y.y - sp[kb].y;
  float best = fmaf(dx, dx, dy * dy);
#pragma unroll
  for (int c = 1; c < 4; ++c) {
    const int k = (int)((w >> (7 * c)) & 127u);
    dx = y.x - sp[k].x;
    dy = y.y - sp[k].y;
    const float d = fmaf(dx, dx, dy * dy);
    const bool better = d < best;
    best = better ? d : best;
    kb = better ? k : kb;
  }
  return kb;
}

// branch-free cell of y (clamped into the grid; the outer ring of cells is brute force).
// float->int by the 2^23 magic number folded into the FFMA (exact half-integer origin)
__device__ __forceinline__ int lut_cell(float2 y, const DecLut& L) {
  const float lo = 8388608.0f, hi = 8388608.0f + (float)(L.g - 1);
  const float fx = fminf(fmaxf(fmaf(y.x, L.inv, L.cxm), lo), hi), fy = fminf(fmaxf(fmaf(y.y, L.inv, L.cym), lo), hi);
  const int m = L.g - 1;
  return ((int)(__float_as_uint(fy) & m) << L.lg) | (int)(__float_as_uint(fx) & m);
}

// argmin over the 4 ascending candidates of a table word: pairwise tournament, strict <
// keeps the lower index on ties (pad entries repeat the first candidate)
__device__ __forceinline__ int decide4(float2 y, uint32_t w, const float2* __restrict__ sp) {
  int k[4];
  float d[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    k[c] = (int)((w >> (7 * c)) & 127u);
    const float2 p = sp[k[c]];
    const float dx = y.x - p.x, dy = y.y - p.y;
    d[c] = fmaf(dx, dx, dy * dy);
  }
  const bool b01 = d[1] < d[0], b23 = d[3] < d[2];
  const float m01 = b01 ? d[1] : d[0], m23 = b23 ? d[3] : d[2];
  const int k01 = b01 ? k[1] : k[0], k23 = b23 ? k[3] : k[2];
  return (m23 < m01) ? k23 : k01;
}

__device__ __forceinline__ int decide(float2 y, const DecLut& L, const float2* __restrict__ sp, int m) {
  const uint32_t w = (L.g > 0) ? __ldg(L.cell + lut_cell(y, L)) : LUT_BRUTE;
  return (w & LUT_BRUTE) ? decide_brute(y, sp, m) : decide4(y, w, sp);
}

__device__ __forceinline__ float2 wl_out(const float2 (&w)[4], const float2 (&g)[4], float2 u0, float2 u1, float2 u2,
                                         float2 u3) {
  // y = w^T u + g^T u*  (SPEC.md l.388 convention), u = (x2[2n+1], x2[2n], x2[2n-1], x2[2n-2])
  const float2 uu[4] = {u0, u1, u2, u3};
  float2 y = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    y.x += w[k].x * uu[k].x - w[k].y * uu[k].y + g[k].x * uu[k].x + g[k].y * uu[k].y;
    y.y += w[k].x * uu[k].y + w[k].y * uu[k].x + g[k].y * uu[k].x - g[k].x * uu[k].y;
  }
  return y;
}

__device__ __forceinline__ unsigned warp_sum(unsigned v) { return __reduce_add_sync(0xffffffffu, v); }

__device__ __forceinline__ int opaque_i(int x) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

// named barrier of one 4-warp group (ids 1..NGROUP; 0 is __syncthreads)
// KK_JITTER (race hunting, tools/gpu/race_jitter.sh): every warp sleeps a pseudo-random
// 0..4 us before each group barrier, so warps and groups reach the shared-memory hand-offs
// in scrambled orders; results must stay bit-identical to the plain build
#ifndef KK_JITTER
#define KK_JITTER 0
#endif
__device__ __forceinline__ void jitter() {
#if KK_JITTER
  unsigned x = (unsigned)clock64() * 2654435761u ^ (threadIdx.x >> 5) * 40503u ^ blockIdx.x * 9973u;
  x ^= x >> 13;
  x *= 0x5bd1e995u;
  x ^= x >> 15;
  if ((x & 3u) == 0u) __nanosleep(x % 4000u);
#endif
}
__device__ __forceinline__ void group_sync(int gi) {
  jitter();
  asm volatile("bar.sync %0, %1;" ::"r"(gi + 1), "r"(NWARPS * 32) : "memory");
}

// --- TMA bulk copy + mbarrier helpers (sm_90+)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "KK_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra KK_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// v = code + d at staged index q, or with the pre-KK intensity equaliser (SURVEY 8(f)
// NEXT-3) v' = sum_{k=-h..h} g_k code[q - k] + d sum(g) (taps as kernel-parameter operands)
// int16 -> float without I2F (a quarter-rate XU instruction; the FIR does ~37 per
// sample): 2^23 + 2^22 + c is exact in fp32 for |c| < 2^22, so one IADD and one exact
// FADD give (float)c bit for bit
__device__ __forceinline__ float i16f(int16_t c) { return __int_as_float((int)c + 0x4B400000) - 12582912.0f; }
// int16 code -> float in S1/S3: the exact IADD + FADD form (ALU + FMA pipes) instead of I2F (the
// quarter-rate XU pipe that also carries the LG2 / SQRT / SIN / COS of S1 and S3); bit-identical
#ifndef KK_I2F_MAGIC
#define KK_I2F_MAGIC 1
#endif
#if KK_I2F_MAGIC
#define CODEF(c) i16f(c)
#else
#define CODEF(c) ((float)(c))
#endif

template <bool PREKK>
__device__ __forceinline__ float prek_v(const ChainArgs& a, const int16_t* src, int q, const Seg& sg) {
  if (!PREKK) return (float)src[q] + sg.dc;
  float v = sg.prek_dsum;
  // rolled: this is the warm-step path only; its unrolled form was ~2.4 k instructions of
  // cold code beside the hot loops (instruction fetch), the producer prek_rows is the hot one
#pragma unroll 1
  for (int k = -a.prek_h; k <= a.prek_h; ++k) v = fmaf(a.prek[k + PKH], i16f(src[q - k]), v);
  return v;
}

// two pre-KK FIR outputs of one lane at staged indices q and q + 32 (S1's samples j and
// j + 1), both halves through one FFMA2 per tap: per tap two loads, two exact int16->float
// IADDs and one FADD2 (the magic number off both halves) -- bit for bit prek_v<true> twice
__device__ __forceinline__ float2 prek_pair(const ChainArgs& a, const int16_t* src, int q, const Seg& sg) {
  float2 acc = make_float2(sg.prek_dsum, sg.prek_dsum);
#pragma unroll 1
  for (int k = -a.prek_h; k <= a.prek_h; ++k) {  // rolled: warm steps only (see prek_v)
    const float2 m = make_float2(__int_as_float((int)src[q - k] + 0x4B400000),
                                 __int_as_float((int)src[q + 32 - k] + 0x4B400000));
#if KK_F32X2
    const float2 c = add2(m, make_float2(-12582912.0f, -12582912.0f));
    acc = fma2(make_float2(a.prek[k + PKH], a.prek[k + PKH]), c, acc);
#else
    acc.x = fmaf(a.prek[k + PKH], m.x - 12582912.0f, acc.x);
    acc.y = fmaf(a.prek[k + PKH], m.y - 12582912.0f, acc.y);
#endif
  }
  return acc;
}

// Pre-KK FIR of a whole step, once per sample: v'[p] for the step's
// staged positions p in [0, VROWS*32) (position p = owner position sbase + p), row r = 32
// consecutive positions, one row per lane (rows 28 w .. 28 w + 27 of warp role w), kept in a
// register sliding window: 48 codes in, 32 outputs, the taps applied in prek_v's order
// (k ascending from dsum) so each v' is bit for bit prek_v<true>.  Stored padded (row r at
// vst + 33 r: conflict-free stores; the readers' position lane + 32 j maps to lane + 33 j).
constexpr int VROWS = (STEP + 512) / 32;  // 112 rows = positions [3072 i - 256, 3072 i + 3328)
__device__ __forceinline__ void prek_rows(const ChainArgs& a, const int16_t* __restrict__ stg, float* __restrict__ vst,
                                          int warp, int lane, const Seg& sg) {
  constexpr int RPW = VROWS / NWARPS;  // 28 rows per warp role
  static_assert(RPW * NWARPS == VROWS && RPW <= 32, "pre-KK rows per warp");
  if (lane >= RPW) return;
  const int r = RPW * warp + lane;
  float cf[32 + 2 * PKH];
  // codes of positions 32 r - PKH .. 32 r + 31 + PKH: stg index PKH + p - PKH = 32 r + m
  const uint4* s4 = reinterpret_cast<const uint4*>(stg + 32 * r);
#pragma unroll
  for (int m = 0; m < (32 + 2 * PKH) / 8; ++m) {
    const uint4 w = s4[m];
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      cf[8 * m + 2 * e] = i16f((int16_t)(ww[e] & 0xffffu));
      cf[8 * m + 2 * e + 1] = i16f((int16_t)(ww[e] >> 16));
    }
  }
  float acc[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = sg.prek_dsum;
#pragma unroll
  for (int k = -PKH; k <= PKH; ++k)
    if (k >= -a.prek_h && k <= a.prek_h) {
      const float g = a.prek[k + PKH];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = fmaf(g, cf[PKH + j - k], acc[j]);
    }
  float* dst = vst + 33 * r;
#pragma unroll
  for (int j = 0; j < 32; ++j) dst[j] = acc[j];
}

struct StepPos {
  int s, o;
  int64_t i;
};

__device__ __forceinline__ int64_t seg_steps_dev(const Seg& s) { return (int64_t)s.n_own * (s.i_end - s.i_begin); }

// the step after p in the step list (segments of owners x steps), without divisions
__device__ __forceinline__ StepPos next_step(const ChainArgs& a, StepPos p) {
  const Seg& sg = a.seg[p.s];
  if (p.i + 1 < sg.i_end) return StepPos{p.s, p.o, p.i + 1};
  if (p.o + 1 < sg.owner_first + sg.n_own) return StepPos{p.s, p.o + 1, (int64_t)sg.i_begin};
  if (p.s + 1 < a.nseg) return StepPos{p.s + 1, a.seg[p.s + 1].owner_first, (int64_t)a.seg[p.s + 1].i_begin};
  return StepPos{-1, 0, 0};
}

__device__ __forceinline__ StepPos decode_step(const ChainArgs& a, int64_t g) {
  StepPos r{0, 0, 0};
#pragma unroll 1
  for (int s = 0; s < a.nseg; ++s) {
    const int64_t per = a.seg[s].i_end - a.seg[s].i_begin;
    const int64_t cnt = per * a.seg[s].n_own;
    if (g < cnt || s == a.nseg - 1) {
      const int64_t k = g / per;
      r.s = s;
      r.o = a.seg[s].owner_first + (int)k;
      r.i = a.seg[s].i_begin + (g - k * per);
      return r;
    }
    g -= cnt;
  }
  return r;
}

constexpr size_t LMS_LUT_BYTES = (size_t)LMS_LUT_G * LMS_LUT_G * sizeof(float2);
constexpr int LMS_CHUNK = 5632;  // update steps per shared-memory window of x2 (kk_lms_kernel / lms_warp_body)

// ---------------------------------------------------------------------------
// Kernel 2b: LMS update pass with one LANE per chain (up to 512 chains per CTA,
// all sharing one copy of the LMS table).  Same arithmetic and step order as
// kk_lms_kernel; a warp's instruction stream serves 32 chains, so the whole
// update pass of a batch occupies a single SM and runs concurrently with the
// fused chain kernel of the previous batch (kk_rx_submit_batch pipeline).  The
// x2 samples stream from L2 through a 16-register ring per lane, prefetched five
// steps ahead.  Optionally spins until the chain kernel has published the x2
// tails it reads (wait_ctr).
// ---------------------------------------------------------------------------
constexpr int LMSL_MAXW = 16;

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// body shared by the standalone kernel (compile-time MODE) and the LMS CTAs of a
// fused chain launch (kk_chain_kernel, runtime mode); smem: [LUT 128 KB][s_pts 129]
// MODE: 0 DD soft gate, 1 PILOT (known pattern), 2 DD hard (gamma = 1)
__device__ __forceinline__ void lms_lanes_body(const LmsArgs& a, unsigned char* lmsl_smem, int blk, const int MODE) {
  float2* s_pts = reinterpret_cast<float2*>(lmsl_smem + LMS_LUT_BYTES);
  const float2* s_lut = reinterpret_cast<const float2*>(lmsl_smem);
  const float INF = __int_as_float(0x7f800000);
  if (MODE != 1) {
    const float4* src = reinterpret_cast<const float4*>(a.lut);
    float4* dst = reinterpret_cast<float4*>(lmsl_smem);
    for (int i = threadIdx.x; i < LMS_LUT_G * LMS_LUT_G / 2; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  for (int i = threadIdx.x; i < 129; i += blockDim.x) s_pts[i] = (i < a.m) ? a.pts[i] : make_float2(INF, INF);
  __syncthreads();
  // chains spread over the warps (chain blk*blockDim + lane*W + warp): with fewer chains
  // than threads every warp gets a few lanes, so the rare slow table path of one lane
  // (divergence) and the per-lane x2 loads cost a warp less; idle lanes replay lane 0's
  // chain of their warp (same control flow, results dropped); chainless warps leave
  const int W = (int)(blockDim.x >> 5), wid = (int)(threadIdx.x >> 5), lid = (int)(threadIdx.x & 31);
  const int c = blk * (int)blockDim.x + lid * W + wid;
  const int c0 = blk * (int)blockDim.x + wid;
  if (c0 >= a.nchains) return;
  if (a.wait_ctr) {
    if (lid == 0)
      while (ld_acquire_u64(a.wait_ctr) < a.wait_target) __nanosleep(200);
    __syncwarp();
  }
  const bool valid = c < a.nchains;
  const int cc = valid ? c : c0;
  const int b = cc / a.nsub, sblk = cc - b * a.nsub;
  const int64_t n0l = (int64_t)sblk * a.L - a.K;
  const int64_t n0 = (int64_t)b * a.n_sym + n0l;
  const float2* xw = a.x2_b0 + (int64_t)b * a.x2_stride + 2 * n0l - 4;  // W[i] = xw[i] (= x2[2 n0l - 4 + i])
  float A[4], B[4], C[4], D[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 w = a.w_init[k], g = a.w_init[4 + k];
    A[k] = w.x + g.x;
    B[k] = g.y - w.y;
    C[k] = w.y + g.y;
    D[k] = w.x - g.x;
  }
  const float mu2 = 2.0f * a.mu;
  const float MAG = 8388608.0f;
  const float lcx = a.lcx - 0.5f + MAG, lcy = a.lcy - 0.5f + MAG;
  const float glo = MAG, ghi = MAG + (float)(LMS_LUT_G - 1);
  unsigned gated = 0;
  float esum = 0.f;
  int64_t pidx = 0;
  if (MODE == 1) {
    pidx = (a.n_off0 + n0) % a.P;
    if (pidx < 0) pidx += a.P;
  }
  auto filt = [&](float2 u0, float2 u1, float2 u2, float2 u3) {
    const float2 uu[4] = {u0, u1, u2, u3};
    float x0 = 0.f, x1 = 0.f, y0 = 0.f, y1 = 0.f;
#pragma unroll
    for (int k = 0; k < 4; k += 2) {
      x0 = fmaf(A[k], uu[k].x, fmaf(B[k], uu[k].y, x0));
      x1 = fmaf(A[k + 1], uu[k + 1].x, fmaf(B[k + 1], uu[k + 1].y, x1));
      y0 = fmaf(C[k], uu[k].x, fmaf(D[k], uu[k].y, y0));
      y1 = fmaf(C[k + 1], uu[k + 1].x, fmaf(D[k + 1], uu[k + 1].y, y1));
    }
    return make_float2(x0 + x1, y0 + y1);
  };
  auto dot2 = [](float2 u, float2 v) { return fmaf(u.x, v.x, u.y * v.y); };
  // ring: R[i & 15] = W[i]; step j reads W[2j .. 2j+7] and refills W[2j+16], W[2j+17]
  float2 R[16];
  {
    const float4* q = reinterpret_cast<const float4*>(xw);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 t = __ldcg(q + i);
      R[2 * i] = make_float2(t.x, t.y);
      R[2 * i + 1] = make_float2(t.z, t.w);
    }
  }
  float qa = dot2(R[3], R[5]), qb = dot2(R[2], R[4]);
  float2 y = filt(R[5], R[4], R[3], R[2]), ep = make_float2(0.f, 0.f);
  auto step = [&](auto qc, int j) {
    constexpr int q = decltype(qc)::value;  // j & 7
    (void)MODE;
    const float2 u0 = R[(2 * q + 5) & 15], u1 = R[(2 * q + 4) & 15], u2 = R[(2 * q + 3) & 15],
                 u3 = R[(2 * q + 2) & 15];
    const float2 v0 = R[(2 * q + 7) & 15], v1 = R[(2 * q + 6) & 15], w2 = R[(2 * q + 1) & 15], w3 = R[(2 * q) & 15];
    const float4 nx = __ldcg(reinterpret_cast<const float4*>(xw + 2 * j + 16));
    float2 ent = make_float2(0.f, 0.f);
    bool out = false;
    int pk = 0;
    if (MODE == 1) {
      pk = a.pattern[pidx];
      pidx = (pidx + 1 == a.P) ? 0 : pidx + 1;
    } else {
      const float fx = fmaf(y.x, a.linv, lcx), fy = fmaf(y.y, a.linv, lcy);
      const uint32_t cell = ((__float_as_uint(fy) << 10) | (__float_as_uint(fx) << 3)) & ((LMS_LUT_G * LMS_LUT_G - 1) << 3);
      ent = *reinterpret_cast<const float2*>(reinterpret_cast<const unsigned char*>(s_lut) + cell);
      out = (fx < glo) | (fx > ghi) | (fy < glo) | (fy > ghi) | (fx != fx) | (fy != fy);
    }
    {
      const float2 pp[4] = {u2, u3, w2, w3};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        A[k] = fmaf(ep.x, pp[k].x, A[k]);
        B[k] = fmaf(ep.x, pp[k].y, B[k]);
        C[k] = fmaf(ep.y, pp[k].x, C[k]);
        D[k] = fmaf(ep.y, pp[k].y, D[k]);
      }
    }
    const float2 yh = filt(v0, v1, u0, u1);
    const float q5 = dot2(u0, v0), q4 = dot2(u1, v1);
    const float r = mu2 * (((q5 + q4) + qa) + qb);
    float2 e, yn;
    if (MODE == 1) {
      const float2 ref = s_pts[pk];
      e = make_float2(ref.x - y.x, ref.y - y.y);
      yn = make_float2(fmaf(r, e.x, yh.x), fmaf(r, e.y, yh.y));
    } else {
      e = make_float2(ent.x - y.x, ent.y - y.y);
      yn = make_float2(fmaf(r, e.x, yh.x), fmaf(r, e.y, yh.y));
      if (out | isnan(yn.x)) {
        const uint32_t w = out ? LMS_BRUTE : __float_as_uint(ent.y);
        float d1 = INF, d2 = INF;
        int k1 = 0;
        if (w == LMS_BRUTE) {
          for (int k = 0; k < a.m; ++k) {
            const float dx = y.x - s_pts[k].x, dy = y.y - s_pts[k].y;
            const float d = fmaf(dx, dx, dy * dy);
            const bool bt = d < d1;
            d2 = bt ? d1 : fminf(d2, d);
            k1 = bt ? k : k1;
            d1 = bt ? d : d1;
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int k = (int)((w >> (8 * jj)) & 0xffu);
            const float dx = y.x - s_pts[k].x, dy = y.y - s_pts[k].y;
            const float d = fmaf(dx, dx, dy * dy);
            const bool bt = d < d1;
            d2 = bt ? d1 : fminf(d2, d);
            k1 = bt ? k : k1;
            d1 = bt ? d : d1;
          }
        }
        const float2 ref = s_pts[k1];
        float gamma = 1.0f;
        if (MODE == 0) gamma = fminf(1.0f, fmaxf(d2 - d1, 0.f) * a.inv_tau);
        gated += (gamma < 1.0f) ? 1u : 0u;
        e = make_float2(gamma * (ref.x - y.x), gamma * (ref.y - y.y));
        yn = make_float2(fmaf(r, e.x, yh.x), fmaf(r, e.y, yh.y));
      }
    }
    esum = fmaf(e.x, e.x, fmaf(e.y, e.y, esum));
    y = yn;
    ep = make_float2(mu2 * e.x, mu2 * e.y);
    qa = q5;
    qb = q4;
    R[(2 * q) & 15] = make_float2(nx.x, nx.y);
    R[(2 * q + 1) & 15] = make_float2(nx.z, nx.w);
  };
  const int K8 = a.K & ~7;
#pragma unroll 1
  for (int j = 0; j < K8; j += 8) {
    step(Phase<0>{}, j);
    step(Phase<1>{}, j + 1);
    step(Phase<2>{}, j + 2);
    step(Phase<3>{}, j + 3);
    step(Phase<4>{}, j + 4);
    step(Phase<5>{}, j + 5);
    step(Phase<6>{}, j + 6);
    step(Phase<7>{}, j + 7);
  }
  const int rem = a.K - K8;
  if (rem > 0) step(Phase<0>{}, K8);
  if (rem > 1) step(Phase<1>{}, K8 + 1);
  if (rem > 2) step(Phase<2>{}, K8 + 2);
  if (rem > 3) step(Phase<3>{}, K8 + 3);
  if (rem > 4) step(Phase<4>{}, K8 + 4);
  if (rem > 5) step(Phase<5>{}, K8 + 5);
  if (rem > 6) step(Phase<6>{}, K8 + 6);
  // the update of the last step: u_{K-1} = (W[2K+3], W[2K+2], W[2K+1], W[2K])
  {
    const float2 lastu[4] = {__ldcg(xw + 2 * a.K + 3), __ldcg(xw + 2 * a.K + 2), __ldcg(xw + 2 * a.K + 1),
                             __ldcg(xw + 2 * a.K)};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      A[k] = fmaf(ep.x, lastu[k].x, A[k]);
      B[k] = fmaf(ep.x, lastu[k].y, B[k]);
      C[k] = fmaf(ep.y, lastu[k].x, C[k]);
      D[k] = fmaf(ep.y, lastu[k].y, D[k]);
    }
  }
  if (valid) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a.taps[(int64_t)c * 8 + k] = make_float2(0.5f * (A[k] + D[k]), 0.5f * (C[k] - B[k]));
      a.taps[(int64_t)c * 8 + 4 + k] = make_float2(0.5f * (A[k] - D[k]), 0.5f * (C[k] + B[k]));
    }
    if (gated) atomicAdd(&a.counts[b * 8 + C_GATED], (unsigned long long)gated);
    bool bad = !(esum / (float)a.K <= 1.0f);
#pragma unroll
    for (int k = 0; k < 4; ++k) bad |= !isfinite(A[k] + B[k] + C[k] + D[k]);
    if (bad) atomicOr(&a.counts[b * 8 + C_FLAGS], 1ull);
  }
}

template <int MODE>
__global__ void __launch_bounds__(LMSL_MAXW * 32) kk_lms_lanes_kernel(LmsArgs a) {
  extern __shared__ __align__(128) unsigned char lmsl_smem[];
  lms_lanes_body(a, lmsl_smem, blockIdx.x, MODE);
}

// ---------------------------------------------------------------------------
// Kernel 1: the fused chain.  A persistent grid; each CTA walks a contiguous
// range of the step list (segments of owners x steps).  Per 3072-sample step:
//   stage codes (TMA bulk copy prefetched during the previous step)
//   phase H: 3 Hilbert FFT pairs (warps 0-2) + the warm-up pair (warp 3) when
//            the CTA starts a new owner: S1, S2, S3 -> D = E_tf - A_hat in smem
//   phase E: 4 static-EQ blocks (one per warp): S4 -> x2 (smem or HBM)
//   phase A: 768 symbols of S5' + S6 + S7 (APPLY segments)
// ---------------------------------------------------------------------------
template <int MODE>
__device__ __forceinline__ void lms_warp_body(const LmsArgs& a, unsigned char* lms_smem, float2* s_pts,
                                              uint64_t* s_barp, int c, int lane);

// S5' + S6 + S7 for NS symbols of one step: symbol sidx_k = s0 + sstride k (step-relative,
// buffer symbol nbase + sidx_k), x2 window xs, factored taps in smem, exact table decision,
// label store, error counts.  refp: the step's pattern bytes in smem (TMA path) or nullptr
// (pattern[(pb + sidx) mod P]).
template <int NS>
__device__ __forceinline__ void apply_symbols(const ChainArgs& a, int s0, int sstride, int nbase, const float2* xs,
                                              const float2* s_taps, const uint32_t* s_lut, bool lut_smem,
                                              const float2* s_pts, const uint8_t* s_lab, uint8_t* outp, bool count_ref,
                                              const uint8_t* refp, int64_t pb, unsigned& acc_se, unsigned& acc_be) {
  int refv[NS];
  if (count_ref) {
    if (refp) {
#pragma unroll
      for (int k = 0; k < NS; ++k) refv[k] = refp[s0 + sstride * k];
    } else {
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        int64_t pi = pb + s0 + sstride * k;
        while (pi >= a.P) pi -= a.P;
        refv[k] = a.pattern[pi];
      }
    }
  }
  float2 yv[NS];
  uint32_t cw[NS];
  {
    float2 ta[4], tc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ta[q] = s_taps[q];
      tc[q] = s_taps[4 + q];
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int sidx = s0 + sstride * k;
      const float4 lo = reinterpret_cast<const float4*>(xs)[sidx];
      const float4 hi = reinterpret_cast<const float4*>(xs)[sidx + 1];
      const float2 u[4] = {make_float2(hi.z, hi.w), make_float2(hi.x, hi.y), make_float2(lo.z, lo.w),
                           make_float2(lo.x, lo.y)};
#if KK_F32X2
      float2 acc0 = mul2(ta[0], make_float2(u[0].x, u[0].x)), acc1 = mul2(ta[1], make_float2(u[1].x, u[1].x));
      acc0 = fma2(tc[0], make_float2(u[0].y, u[0].y), acc0);
      acc1 = fma2(tc[1], make_float2(u[1].y, u[1].y), acc1);
      acc0 = fma2(ta[2], make_float2(u[2].x, u[2].x), acc0);
      acc1 = fma2(ta[3], make_float2(u[3].x, u[3].x), acc1);
      acc0 = fma2(tc[2], make_float2(u[2].y, u[2].y), acc0);
      acc1 = fma2(tc[3], make_float2(u[3].y, u[3].y), acc1);
      yv[k] = add2(acc0, acc1);
#else
      float x0 = 0.f, x1 = 0.f, y0 = 0.f, y1 = 0.f;
#pragma unroll
      for (int t = 0; t < 4; t += 2) {
        x0 = fmaf(ta[t].x, u[t].x, fmaf(ta[t].y, u[t].y, x0));
        x1 = fmaf(ta[t + 1].x, u[t + 1].x, fmaf(ta[t + 1].y, u[t + 1].y, x1));
        y0 = fmaf(tc[t].x, u[t].x, fmaf(tc[t].y, u[t].y, y0));
        y1 = fmaf(tc[t + 1].x, u[t + 1].x, fmaf(tc[t + 1].y, u[t + 1].y, y1));
      }
      yv[k] = make_float2(x0 + x1, y0 + y1);
#endif
    }
  }
  if (lut_smem) {
#pragma unroll
    for (int k = 0; k < NS; ++k) cw[k] = s_lut[lut_cell(yv[k], a.lut)];
  } else {
#pragma unroll
    for (int k = 0; k < NS; ++k) cw[k] = (a.lut.g > 0) ? __ldg(a.lut.cell + lut_cell(yv[k], a.lut)) : LUT_BRUTE;
  }
  int dk[NS];
  bool anyb = false;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    dk[k] = decide4(yv[k], cw[k], s_pts);
    anyb |= (cw[k] & LUT_BRUTE) != 0;
  }
  if (__any_sync(0xffffffffu, anyb)) {
#pragma unroll
    for (int k = 0; k < NS; ++k)
      if (cw[k] & LUT_BRUTE) dk[k] = decide_brute(yv[k], s_pts, a.m);
  }
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    const int sidx = s0 + sstride * k;
    const int n = nbase + sidx;
    if (n >= 0 && n < (int)a.n_sym) {
      const int d = dk[k];
      const uint8_t ld = s_lab[d];
      outp[n] = ld;
      if (count_ref) {
        acc_se += (refv[k] != d) ? 1u : 0u;
        acc_be += __popc((unsigned)(ld ^ s_lab[refv[k]]));
      }
    }
  }
}

// few chains (ChainArgs.lms_warp): one chain per extra CTA, warp 0 runs the
// warp-per-chain update pass (x2 window in shared memory) after the tails are published
__device__ __forceinline__ void lms_warp_cta(const LmsArgs& a, unsigned char* smem, int c, int mode) {
  float2* sp = reinterpret_cast<float2*>(smem + LMS_LUT_BYTES + (2 * LMS_CHUNK + 16) * sizeof(float2));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sp + 130);
  const int lane = (int)threadIdx.x;
  if (a.wait_ctr) {
    if (lane == 0)
      while (ld_acquire_u64(a.wait_ctr) < a.wait_target) __nanosleep(200);
    __syncwarp();
  }
  if (mode == 1)
    lms_warp_body<1>(a, smem, sp, bar, c, lane);
  else if (mode == 2)
    lms_warp_body<2>(a, smem, sp, bar, c, lane);
  else
    lms_warp_body<0>(a, smem, sp, bar, c, lane);
  __syncwarp();
  if (lane == 0) mbar_inval(bar);  // the memory becomes chain-kernel shared memory next
}

template <bool PREKK>
__global__ void __launch_bounds__(NGROUP * NWARPS * 32, 1) kk_chain_kernel(ChainArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (a.lms_ctas > 0 && (int)blockIdx.x >= (int)gridDim.x - a.lms_ctas) {
    // the next batch's LMS update pass: these CTAs come last in the launch order and wait
    // only for tail steps of this launch, which the chain CTAs never wait for.  Afterwards
    // they join the chain work (dynamic schedule only) with the shared memory rebuilt
    const int lblk = (int)blockIdx.x - ((int)gridDim.x - a.lms_ctas);
    if (a.lms_warp) {
      if (threadIdx.x < 32 && lblk < a.lms.nchains) lms_warp_cta(a.lms, smem_raw, lblk, a.lms_mode);
    } else {
      lms_lanes_body(a.lms, smem_raw, lblk, a.lms_mode);
    }
    if (a.work_ctr == nullptr) return;
    __syncthreads();
  }
#if KK_TMEM_TABLES
  const float2* s_tw = nullptr;     // the per-lane tables are in TMEM (below)
  const float2* s_tw512 = nullptr;
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem_raw);
#else
  float2* s_tw = reinterpret_cast<float2*>(smem_raw);
  float2* s_H = reinterpret_cast<float2*>(smem_raw + SMEM_TW);
  float2* s_tw512 = reinterpret_cast<float2*>(smem_raw + SMEM_TW + SMEM_H);
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem_raw + SMEM_TW + SMEM_H + SMEM_TW512);
#endif
  static_assert(SMEM_SHARED - SMEM_LUT == (KK_TMEM_TABLES ? 0 : SMEM_TW + SMEM_H + SMEM_TW512), "shared table layout");
  // opaque copies: ptxas would otherwise rematerialise these (and the group's smem
  // pointers) from S2R SR_TID.X at every use under register pressure
  const int gi = opaque_i(threadIdx.x / (NWARPS * 32));   // group of this thread
  const int tid = opaque_i(threadIdx.x % (NWARPS * 32));  // thread index inside the group
  unsigned char* gbase = smem_raw + SMEM_SHARED + (size_t)gi * SMEM_GROUP;
  float2* ebuf = reinterpret_cast<float2*>(gbase);
  int16_t* stg = reinterpret_cast<int16_t*>(gbase + SMEM_EBUF);
  float2* xs = reinterpret_cast<float2*>(gbase + SMEM_EBUF + SMEM_STG);
  uint8_t* spat = gbase + SMEM_EBUF + SMEM_STG + SMEM_XS;
  int16_t* wstg = reinterpret_cast<int16_t*>(xs);  // warm-up codes (H phase only)
  float* wscr = reinterpret_cast<float*>(xs + WOFF);  // warm-up task's transpose tile
  float2* s_taps = reinterpret_cast<float2*>(gbase + SMEM_EBUF + SMEM_STG + SMEM_XS + SMEM_PAT);  // ta[4], tc[4]
  uint64_t* bar = reinterpret_cast<uint64_t*>(gbase + SMEM_EBUF + SMEM_STG + SMEM_XS + SMEM_PAT + 64);
  uint64_t* pbar = bar + 1;
  float2* pads = reinterpret_cast<float2*>(gbase + ((SMEM_GROUP0 + 127) / 128) * 128);  // transpose-tile row-31 pads
  __shared__ float2 s_pts[128];
  __shared__ uint8_t s_lab[128];

#if !KK_TMEM_TABLES
  for (int k = threadIdx.x; k < 1024; k += blockDim.x) {
    s_tw[k] = a.tw1024[k];
    s_H[k] = a.Hs[k];
  }
  for (int k = threadIdx.x; k < 512; k += blockDim.x) s_tw512[k] = a.tw512[k];
#endif
  const bool lut_smem = a.lut.g > 0 && a.lut.g <= 64;
  if (lut_smem)
    for (int k = threadIdx.x; k < a.lut.g * a.lut.g; k += blockDim.x) s_lut[k] = a.lut.cell[k];
  for (int k = threadIdx.x; k < a.m; k += blockDim.x) {
    s_pts[k] = a.pts[k];
    s_lab[k] = a.labels[k];
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(pbar, 1);
    mbar_fence_init();
  }
#if KK_TMEM_TABLES
  // per-lane tables in TMEM (kk_fft.cuh): warp 0 allocates; warps 0-3 fill their lane quarter
  // (every quarter holds the same 32-lane tables, so any warp reads quarter warp % 4)
  __shared__ uint32_t s_tmem;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "n"(TM_ALLOC)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem + ((uint32_t)(32 * ((threadIdx.x >> 5) & 3)) << 16);
  if (threadIdx.x < 128) {
    const int l = threadIdx.x & 31;
#pragma unroll 1
    for (int r = 1; r < 32; ++r) tm_st2(tmem + TM_TW1024 + 2 * (r - 1), a.tw1024[r * 32 + l]);
    tm_st2(tmem + TM_TW1024 + 62, make_float2(0.f, 0.f));
#pragma unroll 1
    for (int r = 1; r < 16; ++r) tm_st2(tmem + TM_TW512 + 2 * (r - 1), a.tw512[r * 32 + l]);
    tm_st2(tmem + TM_TW512 + 30, make_float2(0.f, 0.f));
#pragma unroll 1
    for (int k = 0; k < 32; ++k) tm_st2(tmem + TM_H + 2 * k, a.Hs[l + 32 * k]);
    tm_wait_st();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#else
  const uint32_t tmem = 0;
  __syncthreads();
#endif

  // task role of this warp inside its group, rotated by the group index: warp w of the
  // CTA issues on sub-partition w % 4 and phase H leaves one role idle, so without the
  // rotation all four idle warps would share one sub-partition
  const int warp = ((tid >> 5) + gi) & (NWARPS - 1), lane = tid & 31;
  const uint32_t n32 = (uint32_t)a.N;
  const int64_t ngroups = (int64_t)(gridDim.x - a.lms_ctas) * NGROUP, grp = (int64_t)blockIdx.x * NGROUP + gi;
  const int64_t T = a.total_steps;
  const bool dyn = a.work_ctr != nullptr;
  int64_t g0 = dyn ? 0 : grp * T / ngroups;
  int64_t g1 = dyn ? 0 : (grp + 1) * T / ngroups;
  __shared__ long long s_grab[NGROUP][2];
  __shared__ long long s_pb[NGROUP];  // pattern index of this step's first symbol (thread 0 -> phase A)
  unsigned long long seen = 0;  // (tid 0) last observed work counter
#if KK_PHASE_TIMING
  long long tdbg[7] = {0, 0, 0, 0, 0, 0, 0};  // diagnostics (a.dbg; build with -DKK_PHASE_TIMING=1)
  long long tmark = 0;
#define KK_DBG(stmt) \
  if (a.dbg) {       \
    stmt;            \
  }
#else
#define KK_DBG(stmt)
#endif
  unsigned pphase = 0;
  int prev_s = -1, prev_o = -1000000;
  int64_t prev_i = -1000000;
  unsigned acc_clip = 0, acc_se = 0, acc_be = 0;
  unsigned phase_bit = 0;
  bool prefetched = false;

  auto flush = [&](int s, int o) {
    if (s < 0) return;
    const unsigned c = warp_sum(acc_clip), se = warp_sum(acc_se), be = warp_sum(acc_be);
    unsigned long long* cnt = a.seg[s].counts;
    if (lane == 0 && cnt) {
      const int64_t k = (int64_t)(o - a.seg[s].owner_first) * 8;
      if (c) atomicAdd(&cnt[k + C_CLIP], (unsigned long long)c);
      if (se) atomicAdd(&cnt[k + C_SYMERR], (unsigned long long)se);
      if (be) atomicAdd(&cnt[k + C_BITERR], (unsigned long long)be);
    }
    acc_clip = acc_se = acc_be = 0;
  };

  // tone phase indices (tb * P) mod N of the EQ outputs: P = sbase + 768 q + 2 (r1 + 256 h) + 32 r2
  const uint32_t s3072 = tone_index(a, STEP);
  // this warp's EQ block q = warp and lane offset 2 (r1 + 256 h), folded into one constant
  const uint32_t q_lane = tone_index(a, (int64_t)EQ_KEEP * warp + 2 * ((lane >> 1) + 256 * (lane & 1)));
  uint32_t q_step = 0;

#pragma unroll 1
  for (;;) {
  if (dyn) {
    // grab the next chunk: one owner's steps while inside a leading tail segment (so
    // the x2 tails a concurrent LMS pass waits for are finished first), then guided
    // chunks shrinking with the remaining work
    if (tid == 0) {
      unsigned long long c;
      const int64_t tail_steps = (a.seg[0].mode == SEG_X2_TAIL) ? seg_steps_dev(a.seg[0]) : 0;
      if ((int64_t)seen < tail_steps) {
        c = (unsigned long long)(a.seg[0].i_end - a.seg[0].i_begin);
      } else {
        const int64_t rem = T - (int64_t)seen;
        // pre-KK: larger chunks (a warm step -- a chunk start -- evaluates its pre-KK FIR on the fly)
        constexpr int64_t GDIV = PREKK ? KK_GUIDE_DIV / 2 : KK_GUIDE_DIV, GMAX = PREKK ? 4 * KK_GUIDE_MAX : KK_GUIDE_MAX;
        int64_t cc = rem / (GDIV * ngroups);
        c = (unsigned long long)(cc < 1 ? 1 : (cc > GMAX ? GMAX : cc));
      }
      const unsigned long long st = atomicAdd(a.work_ctr, c);
      seen = st + c;
      s_grab[gi][0] = (long long)st;
      s_grab[gi][1] = (long long)c;
    }
    group_sync(gi);
    g0 = s_grab[gi][0];
    g1 = g0 + s_grab[gi][1];
    if (g1 > T) g1 = T;
  }
  if (g0 >= g1) break;
  StepPos cur = decode_step(a, g0);
  for (int64_t g = g0; g < g1; ++g) {
    const int s = cur.s, owner = cur.o;
    const int64_t i = cur.i;
    const Seg& sg = a.seg[s];
    const int mode = sg.mode;
    const bool warm = !(s == prev_s && owner == prev_o && i == prev_i + 1);
    StepPos nxt = (g + 1 < g1) ? next_step(a, cur) : StepPos{-1, 0, 0};
    const bool next_cont = (g + 1 < g1) && nxt.s == s && nxt.o == owner && nxt.i == i + 1;
    if (s != prev_s || owner != prev_o) {
      flush(prev_s, prev_o);
      if (mode == SEG_APPLY && tid < 4) {
        // WL taps of the new owner, factored: y.x = sum ta.x u.x + ta.y u.y, y.y = sum tc.x u.x + tc.y u.y
        // (kept in shared memory: only phase A reads them)
        const float2* tp = sg.taps + (int64_t)(owner - sg.owner_first) * 8;
        const float2 w = tp[tid], gg = tp[4 + tid];
#if KK_F32X2
        // paired: (y.x, y.y) = sum_q P[q] u.x + Q[q] u.y, P = (ta.x, tc.x), Q = (ta.y, tc.y)
        s_taps[tid] = make_float2(w.x + gg.x, w.y + gg.y);
        s_taps[4 + tid] = make_float2(gg.y - w.y, w.x - gg.x);
#else
        s_taps[tid] = make_float2(w.x + gg.x, gg.y - w.y);
        s_taps[4 + tid] = make_float2(w.y + gg.y, w.x - gg.x);
#endif
      }
    }
    const int16_t* obase = sg.codes + (int64_t)owner * a.N;
    const int64_t sbase = (int64_t)STEP * i - 256;   // owner position of stg[0] and ebuf[0]
    const float invd = 1.0f / sg.dc;
    const float dc_invd = sg.dc * invd, vmin_invd = a.vmin * invd;
    q_step = warm ? tone_index(a, sbase) : add_mod(q_step, s3072, n32);
    const int64_t wbase = (int64_t)STEP * i - 1280;  // owner position of wstg[0]

    KK_DBG(tmark = clock64())
    // ---- codes of this step
    if (prefetched) {
      mbar_wait(bar, phase_bit);
      phase_bit ^= 1u;
    } else if (a.aligned16) {
      const uint4* s4 = reinterpret_cast<const uint4*>(obase + sbase - PKH);
      uint4* d4 = reinterpret_cast<uint4*>(stg);
      for (int k = tid; k < STG2 / 8; k += NWARPS * 32) d4[k] = __ldg(s4 + k);
    } else {
      for (int k = tid; k < STG2; k += NWARPS * 32) stg[k] = obase[sbase - PKH + k];
    }
    if (warm) {
      if (a.aligned16) {
        const uint4* s4 = reinterpret_cast<const uint4*>(obase + wbase - PKH);
        uint4* d4 = reinterpret_cast<uint4*>(wstg);
        for (int k = tid; k < WARM2 / 8; k += NWARPS * 32) d4[k] = __ldg(s4 + k);
      } else {
        for (int k = tid; k < WARM2; k += NWARPS * 32) wstg[k] = obase[wbase - PKH + k];
      }
    }
    // pattern bytes of this step's symbols (APPLY with counting): bulk copy, waited for in phase A
    const bool count_ref = (mode == SEG_APPLY) && a.pattern != nullptr;
    if (count_ref && tid == 0) {
      // pattern index of symbol 768 i - 32: + 768 (mod P) along a run (the previous step's
      // value is still in s_pb), one division otherwise; kept in smem, not in a register
      int64_t pb_run;
      if (!warm) {
        pb_run = s_pb[gi] + SYM_PER_STEP;
        while (pb_run >= a.P) pb_run -= a.P;
      } else {
        pb_run = (sg.n_off + (int64_t)(owner - sg.owner_first) * a.n_sym + (int64_t)SYM_PER_STEP * i - 32) % a.P;
        if (pb_run < 0) pb_run += a.P;
      }
      s_pb[gi] = pb_run;
    }
    if (count_ref && a.pat_tma) {
      if (tid == 0) {
        const int64_t pb = s_pb[gi];
        const int64_t pa = pb & ~(int64_t)15;
        const unsigned len = (unsigned)(((pb - pa) + SYM_PER_STEP + 15) & ~15);
        const unsigned len1 = (pa + len <= a.P) ? len : (unsigned)(a.P - pa);
        fence_proxy_async();
        mbar_expect_tx(pbar, len);
        bulk_copy(spat, a.pattern + pa, len1, pbar);
        if (len1 < len) bulk_copy(spat + len1, a.pattern, len - len1, pbar);
        mbar_arrive(pbar);
      }
    }
    group_sync(gi);
    // pre-KK FIR once per sample for the whole step (x2 window = v' rows, free until phase E)
    float* vst = (PREKK && !warm) ? reinterpret_cast<float*>(xs) : nullptr;
    if (PREKK && !warm) {
      prek_rows(a, stg, vst, warp, lane, sg);
      group_sync(gi);
    }

    KK_DBG(const long long t = clock64(); tdbg[0] += t - tmark; tmark = t)
    // ---- phase 0: Hilbert pairs (warps 0-2, warp 3 = warm-up pair); phase 1: EQ blocks
#pragma unroll 1
    for (int phase = 0; phase < 2; ++phase) {
      const bool isH = phase == 0;
#if KK_PHASE_TIMING
      const long long tph = a.dbg ? clock64() : 0;
#endif
      if (!isH) {
        // stg is free now: prefetch the next step's codes (async proxy) behind phases E and A
        prefetched = next_cont && a.aligned16;
        if (prefetched && tid == 0) {
          fence_proxy_async();
          bulk_load(stg, obase + sbase + STEP - PKH, STG2 * sizeof(int16_t), bar);
        }
      }
      const bool active = !isH || warp < 3 || warm;
      if (active) {
        float2 v[32];
        int64_t c0 = 0;
        const bool wt = isH && warp >= 3;  // warm-up task
        const int16_t* src = wt ? wstg : stg;
        const int64_t base = wt ? wbase : sbase;
        if (isH) {
          // S1: l = 0.5 ln(v/d) (the constant 0.5 ln d is in the DC bin, zeroed by the mask)
          c0 = wt ? 6 * i - 2 : 6 * i + 2 * warp;
          const int re0 = (int)(512 * c0 - 256 - base);
          // pre-KK FIR: v' from the step's rows (non-warm steps: window position 1024 w + lane + 32 j
          // -> padded 1056 w + lane + 33 j), or evaluated here (warm steps, the warm-up task)
          const float* vrow = (vst && !wt) ? vst + 1056 * warp + lane : nullptr;
          // one unrolled loop per input mode (0 codes, 1 staged v' rows, 2 v' evaluated here), the
          // mode chosen once per task: no per-sample branch, no FIR code inside the hot loop
          auto s1_loop = [&](auto mode_tag) {
            constexpr int MODE = decltype(mode_tag)::value;
            float2 cvp = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 48; ++j) {
              const int q = PKH + re0 + lane + 32 * j;
              // l = lg2(max(code + d, v_min) / d), as max(code/d + 1, v_min/d): one FFMA
              float lv;
              if (MODE == 0) {
                lv = fmaxf(fmaf(CODEF(src[q]), invd, dc_invd), vmin_invd);
              } else {
                float cvj;
                if (MODE == 1) {
                  cvj = vrow[33 * j];
                } else {
                  if ((j & 1) == 0) cvp = prek_pair(a, src, q, sg);  // samples j and j + 1
                  cvj = (j & 1) ? cvp.y : cvp.x;
                }
                lv = fmaxf(cvj, a.vmin) * invd;
              }
              // 0.5 ln 2 / 1024 (the 1/1024 of the inverse FFT folded in): applied here, or
              // (KK_F32X2) by the Hilbert mask multiply, the transform being linear
#if KK_F32X2
              const float l = lg2_ftz(lv);
#else
              const float l = lg2_ftz(lv) * (0.34657359027997264f / 1024.0f);
#endif
              if (j < 32) v[brev(j, 5)].x = l;        // FFT input registers are bit-reversed
              if (j >= 16) v[brev(j - 16, 5)].y = l;
            }
          };
          if (!PREKK)
            s1_loop(IntC<0>{});
          else if (vrow)
            s1_loop(IntC<1>{});
          else
            s1_loop(IntC<2>{});
        } else {
#pragma unroll
          for (int r = 0; r < 32; ++r) v[brev(r, 5)] = ebuf[EQ_KEEP * warp + lane + 32 * r];
        }
        // transpose tile: H tasks use their own (not yet written) output slice of ebuf,
        // the warm-up task a slice of xs; E tasks reuse ebuf once every window is loaded.
        // E tasks: full 32 x 32 float2 tiles (64-bit transposes): warps 0-2 in ebuf[0, 3072)
        // (the kept tail [3072, 3328) untouched), warp 3 in the x2 window xs, which nothing
        // reads during phase E and which the epilogue writes only after a group barrier
        float* scr = wt ? wscr
                        : reinterpret_cast<float*>(isH ? ebuf + 256 + 1024 * warp : (warp < 3 ? ebuf + 1024 * warp : xs));
        if (!isH) group_sync(gi);  // all E windows are in registers before ebuf becomes scratch
        // this warp's row-31 pad at the bank offset of its tile (tile base - 1 mod 16 float2)
        float2* padp = pads + 48 * warp + ((((smem_u32(scr) >> 3) & 15u) + 15u) & 15u);
        const int nfft = isH ? 2 : 1;
#pragma unroll 1
        for (int f = 0; f < nfft; ++f) {
          // H tasks: 64-bit transposes through their own 1024-sample output slice
          fft1024(v, lane, scr, s_tw, tmem, padp);
          if (isH && f == 0) {
            // S2: phi = -H{l} <-> +i sgn(k) L_k (reading R1; the /1024 is in S1), conjugated so the
            // next forward FFT computes the inverse: IFFT(Y) = conj(FFT(conj(Y)))
            float2 nv[32];
#pragma unroll
            for (int k2 = 0; k2 < 32; ++k2) {
              const float2 y = v[k2];
#if KK_F32X2
              // one FMUL2 per element: swapped halves times -+K, K = 0.5 ln 2 / 1024 (S1 scale)
              constexpr float KS = 0.34657359027997264f / 1024.0f;
              float2 r = mul2(make_float2(y.y, y.x), (k2 < 16) ? make_float2(-KS, -KS) : make_float2(KS, KS));
#else
              float2 r = (k2 < 16) ? make_float2(-y.y, -y.x) : make_float2(y.y, y.x);
#endif
              if ((k2 == 0 || k2 == 16) && lane == 0) r = make_float2(0.f, 0.f);
              nv[brev(k2, 5)] = r;  // bit-reversed input of the next transform
            }
#pragma unroll
            for (int k2 = 0; k2 < 32; ++k2) v[k2] = nv[k2];
          }
        }
        if (isH) {
          // S3 (tone frame): D = sqrt(v) e^{i phi} - A_hat; phi_re = v.x, phi_im = -v.y.
          // Window index m = lane + 32 n2 (n2 in [8, 24)); chunk c0 at m - 256, chunk c0+1 at m + 256.
          const int s_off = (int)(512 * c0 - 256 - base);
          const int e_off = (int)(512 * c0 - 256 - sbase);
          // warm-up task: all 1024 outputs to a slice of xs (its tile is dead), then its last 256 to ebuf[0, 256)
          float2* dst = wt ? (xs + WOFF - 256) : (ebuf + e_off);
          const bool cnt = !wt && sg.count_clip && (mode == SEG_APPLY || owner >= sg.ref);
          const int lim = (int)((a.N - sbase < (int64_t)(1 << 30)) ? a.N - sbase : (int64_t)(1 << 30)) - e_off;
          unsigned clip = 0;
          float cmin = __int_as_float(0x7f800000);
          // both phases of window position m (chunk c0: v.x; chunk c0 + 1: -v.y) as one float2
          // in output slot m (the same lane writes and later reads it; 64-bit, conflict-free),
          // then one rolled loop over the 32 outputs (keeps the kernel's code small)
#pragma unroll
          for (int n2 = 8; n2 < 24; ++n2) dst[lane + 32 * n2] = v[n2];
          // outputs mm = lane + 256 + 32 t (chunk c0) and mm + 512 (chunk c0 + 1), t = 0..15
          const int16_t* sp0 = src + PKH + s_off + lane + 256;
          float2* dp0 = dst + lane + 256;
          const bool allin = lim >= 1280;  // every output position of this task is < N
          // S3 per input mode (0 codes, 1 staged v' rows, 2 v' evaluated here), chosen once per task
          auto s3_loop = [&](auto mode_tag) {
            constexpr int MODE = decltype(mode_tag)::value;
            // the inputs of output t + 1 (its two codes / v' values and its phase pair) are loaded
            // during output t, so the shared-memory latency is off the S3 dependency chain
            auto load_cv = [&](int tt, int hh) -> float {
              return MODE == 0 ? CODEF(sp0[32 * tt + 512 * hh]) + sg.dc
                               : MODE == 1 ? vst[1056 * warp + 264 + lane + 33 * tt + 528 * hh]
                                           : prek_v<true>(a, sp0, 32 * tt + 512 * hh, sg);
            };
            float2 ph_n = dp0[0];
            float cv_n0 = MODE < 2 ? load_cv(0, 0) : 0.f, cv_n1 = MODE < 2 ? load_cv(0, 1) : 0.f;
#pragma unroll S3_UNROLL
            for (int t = 0; t < 16; ++t) {
              const float2 ph = ph_n;  // read before output slot m is overwritten below
              const float cvt[2] = {cv_n0, cv_n1};
              if (MODE < 2) {
                const int tn = t < 15 ? t + 1 : 15;
                ph_n = dp0[32 * tn];
                cv_n0 = load_cv(tn, 0);
                cv_n1 = load_cv(tn, 1);
              } else if (t < 15) {
                ph_n = dp0[32 * (t + 1)];
              }
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int o = 32 * t + 512 * hh;
                const float phi = hh ? -ph.y : ph.x;
                const float cv = MODE < 2 ? cvt[hh] : load_cv(t, hh);
                const float vv = fmaxf(cv, a.vmin);
                const float amp = sqrt_ftz(vv);
                float sp, cp;
                sincos_small(phi, &sp, &cp);  // |phi| of a few rad at most (KK phase)
#if KK_F32X2
                dp0[o] = fma2(make_float2(amp, amp), make_float2(cp, sp), make_float2(-sg.a_hat, 0.f));
#else
                dp0[o] = make_float2(fmaf(amp, cp, -sg.a_hat), amp * sp);
#endif
                cmin = fminf(cmin, cv);
              }
            }
          };
          if (!PREKK)
            s3_loop(IntC<0>{});
          else if (!warm)
            s3_loop(IntC<1>{});
          else
            s3_loop(IntC<2>{});
          if (cnt && cmin < a.vmin) {
            // rare: some input of this task was clamped -- count exactly (positions < N)
#pragma unroll 1
            for (int t = 0; t < 16; ++t)
              for (int hh = 0; hh < 2; ++hh) {
                const int o = 32 * t + 512 * hh;
                const float cv = !PREKK ? CODEF(sp0[o]) + sg.dc
                                 : (!warm ? vst[1056 * warp + 264 + lane + 33 * t + 528 * hh]
                                          : prek_v<true>(a, sp0, o, sg));
                clip += (cv < a.vmin && (allin || lane + 256 + o < lim)) ? 1u : 0u;
              }
          }
          if (cnt) acc_clip += clip;
          if (wt) {
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 8; ++k) ebuf[lane + 32 * k] = dst[1024 + lane + 32 * k];
          }
          if (a.es_dump && !wt && mode == SEG_X2_FULL && owner >= sg.ref) {
            // debug only: E_s = D e^{i theta_p} at owned positions
            __syncwarp();
#pragma unroll 1
            for (int k = lane; k < 1024; k += 32) {
              const int ei = e_off + 256 + k;
              const int64_t pp = sbase + ei;
              if (pp >= 0 && pp < a.N) {
                const float2 d = ebuf[ei];
                float st, ct;
                cis_turns((float)tone_index(a, pp) * a.invN, &st, &ct);
                a.es_dump[(int64_t)(owner - sg.ref) * a.N + pp] =
                    make_float2(d.x * ct - d.y * st, d.x * st + d.y * ct);
              }
            }
          }
        } else {
          // S4: x2 = e^{i theta_P} * IDFT512(fold(DFT1024(D) * Hs))  (downconversion moved
          // behind the LTI filter: Hs is the DFT of h_i e^{-2 pi i tb i / N}, reading R5)
          const int q = warp;
          float2 z[16];
#if KK_TMEM_TABLES
          // H[lane + 32 k2] and H[lane + 32 (k2 + 16)] from this lane's TMEM table, 4 at a time
          float2 hlo[4], hhi[4];
#endif
#pragma unroll
          for (int k2 = 0; k2 < 16; ++k2) {
#if KK_TMEM_TABLES
            if ((k2 & 3) == 0) {
              tm_ld4(tmem + TM_H + 2 * k2, hlo);
              tm_ld4(tmem + TM_H + 2 * (k2 + 16), hhi);
              tm_wait(hhi);
              asm volatile("" : "+f"(hlo[0].x), "+f"(hlo[0].y), "+f"(hlo[1].x), "+f"(hlo[1].y), "+f"(hlo[2].x),
                           "+f"(hlo[2].y), "+f"(hlo[3].x), "+f"(hlo[3].y) : "f"(hhi[0].x));
            }
            const float2 s0 = c_mul(v[k2], hlo[k2 & 3]);
            const float2 s1 = c_mul(v[k2 + 16], hhi[k2 & 3]);
#else
            const float2 s0 = c_mul(v[k2], s_H[lane + 32 * k2]);
            const float2 s1 = c_mul(v[k2 + 16], s_H[lane + 32 * (k2 + 16)]);
#endif
#if KK_F32X2
            z[brev(k2, 4)] = add2(make_float2(s0.x, -s0.y), make_float2(s1.x, -s1.y));  // conj -> forward DFT = inverse
#else
            z[brev(k2, 4)] = make_float2(s0.x + s1.x, -(s0.y + s1.y));  // conj -> forward DFT = inverse
#endif
          }
          fft512_pairs(z, lane, scr, s_tw512, tmem);
          group_sync(gi);  // every tile (warp 3's lies in xs) is done before xs is written
          const int h = lane & 1, r1 = lane >> 1;
          // lane holds window outputs rr = r1 + 16 r2 + 256 h, i.e. positions P = P0 + 2 rr: a
          // stride-16 run in x2 index; keep rr in [rlo, 448) and (X2 modes) the owned positions
          const int rlo = (mode == SEG_APPLY && q == 0) ? 62 : 64;
          const int rbase = r1 + 256 * h;
          int lo2 = (rlo - rbase + 15) >> 4, hi2 = (448 - rbase + 15) >> 4;  // r2 range of kept outputs
          lo2 = lo2 < 0 ? 0 : lo2;
          hi2 = hi2 > 16 ? 16 : hi2;
          const int64_t P0 = sbase + EQ_KEEP * q + 2 * rbase;  // position of r2 = 0
          float2* dptr = nullptr;
          if (mode == SEG_APPLY) {
            dptr = xs + (384 * q + rbase - 62);
          } else {
            // owned window [own_lo, N) in position; x2 index = P / 2 relative to the destination base
            const int64_t tail_lo = a.N - 2 * a.x2h;
            int64_t own_lo, dbase;
            if (mode == SEG_X2_TAIL) {
              own_lo = tail_lo;
              dbase = (int64_t)(owner - sg.owner_first) * a.x2h - (tail_lo >> 1);
            } else {
              own_lo = (owner < sg.ref) ? tail_lo : 0;
              dbase = (int64_t)(owner - sg.ref) * (a.N >> 1);
            }
            // r2 with own_lo <= P0 + 32 r2 < N
            const int64_t l2 = (own_lo - P0 + 31) >> 5, h2 = (a.N - P0 + 31) >> 5;
            lo2 = (int)(l2 > lo2 ? (l2 < 16 ? l2 : 16) : lo2);
            hi2 = (int)(h2 < hi2 ? (h2 > 0 ? h2 : 0) : hi2);
            dptr = sg.x2dst + dbase + (P0 >> 1);
          }
          // e^{i theta_P} at P = P0 + 32 r2: one sincos for the lane's base, times the
          // constant e^{i theta(32 r2)} (host fp64, rounded once; kernel-parameter operands)
          float sb, cb;
          cis_turns((float)add_mod(q_step, q_lane, n32) * a.invN, &sb, &cb);  // (tb * P0) mod N
#pragma unroll
          for (int r2 = 0; r2 < 16; ++r2) {
            if (r2 >= lo2 && r2 < hi2) {
              const float2 rr = a.rot[r2];
              const float2 o = z[r2];
#if KK_F32X2
              // e = e^{i theta_P} = (cb, sb) rr;  conj(o) e = o.x (ct, st) + o.y (st, -ct)
              const float2 e = c_mul(make_float2(cb, sb), rr);
              dptr[16 * r2] = fma2(make_float2(e.y, -e.x), make_float2(o.y, o.y), mul2(e, make_float2(o.x, o.x)));
#else
              const float ct = fmaf(cb, rr.x, -sb * rr.y), st = fmaf(cb, rr.y, sb * rr.x);
              dptr[16 * r2] = make_float2(o.x * ct + o.y * st, o.x * st - o.y * ct);  // conj(o) e^{i theta}
#endif
            }
          }
        }
        KK_DBG(tdbg[isH ? 5 : 6] += clock64() - tph)
      }
      group_sync(gi);
      KK_DBG(const long long t = clock64(); tdbg[isH ? 1 : 2] += t - tmark; tmark = t)
    }

    if (mode == SEG_APPLY) {
      // ---- S5' + S6 + S7 on symbols [768 i - 32, 768 i + 736) of this owner: each thread's
      // symbols in KK_A_ROUNDS rounds (code size of the unrolled body vs in-flight symbols)
      const int nbase = SYM_PER_STEP * (int)i - 32;
      const int64_t ko = owner - sg.owner_first;
      uint8_t* outp = sg.out + ko * a.n_sym;
      const uint8_t* refp = nullptr;
      const int64_t pb = s_pb[gi];
      if (count_ref && a.pat_tma) {
        mbar_wait(pbar, pphase);
        pphase ^= 1u;
        refp = spat + (int)(pb & 15);
      }
      constexpr int SPT_R = SYM_PER_STEP / (NWARPS * 32) / KK_A_ROUNDS;
#pragma unroll 1
      for (int rd = 0; rd < KK_A_ROUNDS; ++rd)
        apply_symbols<SPT_R>(a, tid + NWARPS * 32 * SPT_R * rd, NWARPS * 32, nbase, xs, s_taps, s_lut, lut_smem, s_pts,
                             s_lab, outp, count_ref, refp, pb, acc_se, acc_be);
    }
    // keep the last 256 D samples for the next step's first EQ window
    for (int k = tid; k < 256; k += NWARPS * 32) ebuf[k] = ebuf[STEP + k];
    const bool pub = mode == SEG_X2_TAIL && a.tail_ctr != nullptr;
    if (pub) __threadfence();  // this step's x2 tail stores, before the release below
    group_sync(gi);
    if (pub && tid == 0) {
      __threadfence();
      atomicAdd(a.tail_ctr, 1ull);
    }
    KK_DBG(tdbg[3] += clock64() - tmark; tdbg[4] += 1)
    prev_s = s;
    prev_o = owner;
    prev_i = i;
    cur = nxt;
  }
  if (!dyn) break;
  }
  flush(prev_s, prev_o);
#if KK_TMEM_TABLES
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();  // every group is done with the TMEM tables
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "n"(TM_ALLOC) : "memory");
#endif
#if KK_PHASE_TIMING
  if (a.dbg) {
    // group totals from the group's thread 0 (wall-clock phases), busy times from every lane 0
    if (tid == 0)
      for (int k = 0; k < 5; ++k) atomicAdd(a.dbg + k, (unsigned long long)tdbg[k]);
    if (lane == 0) {
      atomicAdd(a.dbg + 5, (unsigned long long)tdbg[5]);
      atomicAdd(a.dbg + 6, (unsigned long long)tdbg[6]);
    }
  }
#endif
#undef KK_DBG
}

cudaError_t chain_setup(int device, int* grid_out) {
  int sms = 0, occ = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaFuncSetAttribute(kk_chain_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CHAIN_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kk_chain_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CHAIN_SMEM);
  if (e != cudaSuccess) return e;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kk_chain_kernel<false>, NGROUP * NWARPS * 32, CHAIN_SMEM);
  if (occ < 1) occ = 1;
  *grid_out = sms * occ;
  return cudaGetLastError();
}

cudaError_t launch_chain(const ChainArgs& a, int grid, cudaStream_t s) {
  if (a.total_steps <= 0) return cudaSuccess;
  if (grid > a.total_steps) grid = (int)a.total_steps;
  if (a.prek_h >= 0)
    kk_chain_kernel<true><<<grid, NGROUP * NWARPS * 32, CHAIN_SMEM, s>>>(a);
  else
    kk_chain_kernel<false><<<grid, NGROUP * NWARPS * 32, CHAIN_SMEM, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Kernel 2: LMS update pass, one warp per sub-block chain (reading R10), 4 chains
// per CTA sharing one LMS look-up table in shared memory.  The chain is
// inherently sequential, so the kernel minimises the per-step
// latency: the critical path is y_n -> decision -> e_n -> y_{n+1}.
//  * the widely-linear filter y = w^T u + g^T u* is the real 2x2 matrix filter
//      [y.x; y.y] = sum_k [[A_k, B_k], [C_k, D_k]] [u_k.x; u_k.y],
//    A = w.x + g.x, B = g.y - w.y, C = w.y + g.y, D = w.x - g.x, and the LMS update
//    w += mu e u*, g += mu e u is exactly  [dA dB; dC dD] = 2 mu [e.x; e.y] [u.x u.y]
//    (16 FFMA per step instead of 32); w, g are recovered at the end;
//  * lookahead: y_{n+1} = yhat_{n+1} + 2 mu (sum_k u_{n,k} . u_{n+1,k}) e_n, with
//    yhat computed from the pre-update matrix off the critical path;
//  * decision: one shared-memory load of the cell entry of y.  FAST cells (one
//    point nearest everywhere in the cell and every other point >= tau farther)
//    give ref = p_k and gamma = 1 directly; SLOW cells list the <= 4 points that
//    can be nearest or within tau of it (ascending, so strict < keeps the lowest
//    index on ties), from which k1, D1 and D2 (second-smallest distance) follow
//    exactly as in the oracle; cells with longer lists fall back to brute force.
// ---------------------------------------------------------------------------
constexpr size_t LMS_SMEM_MAX = 220 * 1024;  // + static smem <= 227 KB
static_assert(LMS_LUT_BYTES + (2 * LMS_CHUNK + 16) * sizeof(float2) <= LMS_SMEM_MAX, "LMS smem budget");


// one warp per chain; shared memory = [LUT (not in PILOT mode)] [x2 window of <= LMS_CHUNK steps].
// The body runs in kk_lms_kernel (one 32-thread CTA per chain) and in warp 0 of extra CTAs
// of a chain launch (streaming pipeline with few chains: ChainArgs.lms_warp).
template <int MODE>  // 0: DD soft gate, 1: PILOT (known pattern), 2: DD hard (gamma = 1)
__device__ __forceinline__ void lms_warp_body(const LmsArgs& a, unsigned char* lms_smem, float2* s_pts,
                                              uint64_t* s_barp, int c, int lane) {
  uint64_t& s_bar = *s_barp;
  constexpr size_t LUTB = (MODE == 1) ? 0 : LMS_LUT_BYTES;
  const float2* s_lut = reinterpret_cast<const float2*>(lms_smem);
  float2* s_win = reinterpret_cast<float2*>(lms_smem + LUTB);
  const float INF = __int_as_float(0x7f800000);
  for (int i = lane; i < 129; i += 32) s_pts[i] = (i < a.m) ? a.pts[i] : make_float2(INF, INF);
  const int b = c / a.nsub, sblk = c - b * a.nsub;
  const int64_t n0l = (int64_t)sblk * a.L - a.K;       // first update symbol, buffer-relative
  const int64_t n0 = (int64_t)b * a.n_sym + n0l;       // ... relative to buffer 0 (pattern index)
  const float2* xp = a.x2_b0 + (int64_t)b * a.x2_stride + 2 * n0l - 2;  // step s uses xp[2s .. 2s+5]
  if (lane == 0) {
    mbar_init(&s_bar, 1);
    mbar_fence_init();
  }
  __syncwarp();
  unsigned phase = 0;
  // copy x2[2 sa - 1 (16-B alignment) .. 2 sb + 6) of steps [sa, sb) (+ the LUT with the first chunk)
  auto load_window = [&](int sa, int sb, bool with_lut) -> const float2* {
    const float2* src = xp + 2 * sa - 2;  // W[0] = x of step sa - 1 (its u for the deferred update)
    const int mis = (int)(((uintptr_t)src >> 3) & 1);  // float2 elements before a 16-B boundary
    const float2* srca = src - mis;
    const unsigned n = (unsigned)(2 * (sb - sa) + 8 + mis + 1) & ~1u;
    if (lane == 0) {
      if (with_lut) {
        mbar_expect_tx(&s_bar, (unsigned)LUTB);
        bulk_copy(lms_smem, a.lut, (unsigned)LUTB, &s_bar);
      }
      mbar_expect_tx(&s_bar, n * (unsigned)sizeof(float2));
      bulk_copy(s_win, srca, n * (unsigned)sizeof(float2), &s_bar);
      mbar_arrive(&s_bar);
    }
    mbar_wait(&s_bar, phase);
    phase ^= 1u;
    return s_win + mis;
  };
  float A[4], B[4], C[4], D[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 w = a.w_init[k], g = a.w_init[4 + k];
    A[k] = w.x + g.x;
    B[k] = g.y - w.y;
    C[k] = w.y + g.y;
    D[k] = w.x - g.x;
  }
  const float mu2 = 2.0f * a.mu;
  // cell coordinate with the float->int conversion folded into the FFMA: lc is a
  // half-integer (host), so lc - 1/2 + 2^23 is exact and the single rounding of fmaf
  // leaves floor(y*linv + lc) (up to round-half-even at exact integers, absorbed by
  // the 1e-3 cell enlargement of the table) in the low mantissa bits; clamping in the
  // float domain maps y outside the grid to the brute-force outer ring.
  const float MAG = 8388608.0f;
  const float lcx = a.lcx - 0.5f + MAG, lcy = a.lcy - 0.5f + MAG;
  const float glo = MAG, ghi = MAG + (float)(LMS_LUT_G - 1);
  unsigned gated = 0;
  float esum = 0.f;
  int64_t pidx = 0;
  if (MODE == 1) {
    pidx = (a.n_off0 + n0) % a.P;
    if (pidx < 0) pidx += a.P;
  }
  auto filt = [&](float2 u0, float2 u1, float2 u2, float2 u3) {
    const float2 uu[4] = {u0, u1, u2, u3};
    float x0 = 0.f, x1 = 0.f, y0 = 0.f, y1 = 0.f;
#pragma unroll
    for (int k = 0; k < 4; k += 2) {
      x0 = fmaf(A[k], uu[k].x, fmaf(B[k], uu[k].y, x0));
      x1 = fmaf(A[k + 1], uu[k + 1].x, fmaf(B[k + 1], uu[k + 1].y, x1));
      y0 = fmaf(C[k], uu[k].x, fmaf(D[k], uu[k].y, y0));
      y1 = fmaf(C[k + 1], uu[k + 1].x, fmaf(D[k + 1], uu[k + 1].y, y1));
    }
    return make_float2(x0 + x1, y0 + y1);
  };
  // One LMS step n (chunk-local j = n - sa).  The x2 window W (W[i] = xp[2 sa - 2 + i])
  // lives in an 8-register circular buffer R[i & 7]; step j reads W[2j .. 2j+7]:
  //   u_n = (W[2j+5], W[2j+4], W[2j+3], W[2j+2]),  u_{n+1} = (W[2j+7], W[2j+6], u0, u1),
  //   u_{n-1} = (W[2j+3], W[2j+2], W[2j+1], W[2j])
  // and refills the two dead slots with W[2j+8], W[2j+9]; the phase j & 3 is a
  // compile-time constant of the 4-step unrolled body, so no register is copied.
  // State on entry: y = y_n, ep = mu2 e_{n-1} (not yet applied to the matrix),
  // qa = W[2j+3].W[2j+5], qb = W[2j+2].W[2j+4].  In program order: start the cell
  // lookup of y_n (critical path); independent of it, and filling its latency, apply
  // the update of e_{n-1} to the matrix and form yhat_{n+1} = M u_{n+1} and r_n; then
  // resolve the decision, e_n, and y_{n+1} = yhat_{n+1} + r_n e_n.
  float2 y = make_float2(0.f, 0.f), ep = make_float2(0.f, 0.f);
  float2 R[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) R[i] = y;
  float qa = 0.f, qb = 0.f;
  auto dot2 = [](float2 u, float2 v) { return fmaf(u.x, v.x, u.y * v.y); };
  auto step = [&](auto qc, const float2* W, int j) {
    constexpr int q = decltype(qc)::value;
    const float2 u0 = R[(2 * q + 5) & 7], u1 = R[(2 * q + 4) & 7], u2 = R[(2 * q + 3) & 7], u3 = R[(2 * q + 2) & 7];
    const float2 v0 = R[(2 * q + 7) & 7], v1 = R[(2 * q + 6) & 7], w2 = R[(2 * q + 1) & 7], w3 = R[(2 * q) & 7];
    const float4 nx = *reinterpret_cast<const float4*>(W + 2 * j + 8);
    float2 ent = make_float2(0.f, 0.f);
    bool out = false;
    int pk = 0;
    if (MODE == 1) {
      pk = a.pattern[pidx];
      pidx = (pidx + 1 == a.P) ? 0 : pidx + 1;
    } else {
      // masked index (always inside the table, loaded unconditionally); y outside the
      // grid -> brute force
      const float fx = fmaf(y.x, a.linv, lcx), fy = fmaf(y.y, a.linv, lcy);
      const uint32_t cell = ((__float_as_uint(fy) << 10) | (__float_as_uint(fx) << 3)) & ((LMS_LUT_G * LMS_LUT_G - 1) << 3);
      ent = *reinterpret_cast<const float2*>(reinterpret_cast<const unsigned char*>(s_lut) + cell);
      out = (fx < glo) | (fx > ghi) | (fy < glo) | (fy > ghi) | (fx != fx) | (fy != fy);
    }
    {
      const float2 pp[4] = {u2, u3, w2, w3};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        A[k] = fmaf(ep.x, pp[k].x, A[k]);
        B[k] = fmaf(ep.x, pp[k].y, B[k]);
        C[k] = fmaf(ep.y, pp[k].x, C[k]);
        D[k] = fmaf(ep.y, pp[k].y, D[k]);
      }
    }
    const float2 yh = filt(v0, v1, u0, u1);
    const float q5 = dot2(u0, v0), q4 = dot2(u1, v1);
    const float r = mu2 * (((q5 + q4) + qa) + qb);
    // straight-line FAST assumption (gamma = 1, ref = the cell's point); SLOW cells
    // (rare) recompute e below.  Keeping yhat, r and y_{n+1} ahead of the branch lets
    // them fill the latency of the table load.
    float2 e, yn;
    if (MODE == 1) {
      const float2 ref = s_pts[pk];
      e = make_float2(ref.x - y.x, ref.y - y.y);
      yn = make_float2(fmaf(r, e.x, yh.x), fmaf(r, e.y, yh.y));
    } else {
      e = make_float2(ent.x - y.x, ent.y - y.y);
      yn = make_float2(fmaf(r, e.x, yh.x), fmaf(r, e.y, yh.y));
      // the NaN of a SLOW entry propagates into yn (so the branch needs yhat and r first)
      if (out | isnan(yn.x)) {
        const uint32_t w = out ? LMS_BRUTE : __float_as_uint(ent.y);
        float d1 = INF, d2 = INF;
        int k1 = 0;
        if (w == LMS_BRUTE) {
#pragma unroll 1
          for (int k = 0; k < a.m; ++k) {
            const float dx = y.x - s_pts[k].x, dy = y.y - s_pts[k].y;
            const float d = fmaf(dx, dx, dy * dy);
            const bool bt = d < d1;
            d2 = bt ? d1 : fminf(d2, d);
            k1 = bt ? k : k1;
            d1 = bt ? d : d1;
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int k = (int)((w >> (8 * jj)) & 0xffu);  // 128 = padding (point at infinity)
            const float dx = y.x - s_pts[k].x, dy = y.y - s_pts[k].y;
            const float d = fmaf(dx, dx, dy * dy);
            const bool bt = d < d1;
            d2 = bt ? d1 : fminf(d2, d);
            k1 = bt ? k : k1;
            d1 = bt ? d : d1;
          }
        }
        const float2 ref = s_pts[k1];
        float gamma = 1.0f;
        if (MODE == 0) gamma = fminf(1.0f, fmaxf(d2 - d1, 0.f) * a.inv_tau);
        gated += (gamma < 1.0f) ? 1u : 0u;
        e = make_float2(gamma * (ref.x - y.x), gamma * (ref.y - y.y));
        yn = make_float2(fmaf(r, e.x, yh.x), fmaf(r, e.y, yh.y));
      }
    }
    esum = fmaf(e.x, e.x, fmaf(e.y, e.y, esum));
    y = yn;  // y_{n+1}
    ep = make_float2(mu2 * e.x, mu2 * e.y);
    qa = q5;
    qb = q4;
    R[(2 * q) & 7] = make_float2(nx.x, nx.y);      // W[2j+8]
    R[(2 * q + 1) & 7] = make_float2(nx.z, nx.w);  // W[2j+9]
  };
  using P0 = Phase<0>;
  using P1 = Phase<1>;
  using P2 = Phase<2>;
  using P3 = Phase<3>;
  const float2* W = nullptr;
  int n = 0;
#pragma unroll 1
  for (int sa = 0; sa < a.K; sa += LMS_CHUNK) {
    const int sb = min(a.K, sa + LMS_CHUNK);
    if (sa > 0) __syncwarp();  // every lane is done with the previous window
    W = load_window(sa, sb, sa == 0 && MODE != 1);
#pragma unroll
    for (int i = 0; i < 8; ++i) R[i] = W[i];
    qa = dot2(R[3], R[5]);
    qb = dot2(R[2], R[4]);
    if (sa == 0) y = filt(R[5], R[4], R[3], R[2]);
    n = sb - sa;
    const int n4 = n & ~3;
#pragma unroll 1
    for (int j = 0; j < n4; j += 4) {
      step(P0{}, W, j);
      step(P1{}, W, j + 1);
      step(P2{}, W, j + 2);
      step(P3{}, W, j + 3);
    }
    if (n4 < n) step(P0{}, W, n4);
    if (n4 + 1 < n) step(P1{}, W, n4 + 1);
    if (n4 + 2 < n) step(P2{}, W, n4 + 2);
  }
  // the update of the last step: e_{K-1} with u_{K-1} = (W[2n+3], W[2n+2], W[2n+1], W[2n]) of the last window
  {
    const float2 lastu[4] = {W[2 * n + 3], W[2 * n + 2], W[2 * n + 1], W[2 * n]};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      A[k] = fmaf(ep.x, lastu[k].x, A[k]);
      B[k] = fmaf(ep.x, lastu[k].y, B[k]);
      C[k] = fmaf(ep.y, lastu[k].x, C[k]);
      D[k] = fmaf(ep.y, lastu[k].y, D[k]);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // w = ((A + D) + i (C - B)) / 2,  g = ((A - D) + i (C + B)) / 2
      a.taps[(int64_t)c * 8 + k] = make_float2(0.5f * (A[k] + D[k]), 0.5f * (C[k] - B[k]));
      a.taps[(int64_t)c * 8 + 4 + k] = make_float2(0.5f * (A[k] - D[k]), 0.5f * (C[k] + B[k]));
    }
    if (gated) atomicAdd(&a.counts[b * 8 + C_GATED], (unsigned long long)gated);
    bool bad = !(esum / (float)a.K <= 1.0f);
#pragma unroll
    for (int k = 0; k < 4; ++k) bad |= !isfinite(A[k] + B[k] + C[k] + D[k]);
    if (bad) atomicOr(&a.counts[b * 8 + C_FLAGS], 1ull);
  }
}

template <int MODE>
__global__ void __launch_bounds__(32) kk_lms_kernel(LmsArgs a) {
  extern __shared__ __align__(128) unsigned char lms_smem[];
  __shared__ float2 s_pts[129];
  __shared__ __align__(8) uint64_t s_bar;
  if ((int)blockIdx.x >= a.nchains) return;
  lms_warp_body<MODE>(a, lms_smem, s_pts, &s_bar, (int)blockIdx.x, (int)threadIdx.x);
}

static size_t lms_smem_bytes(int mode, int K) {
  const size_t lut = (mode == 1) ? 0 : LMS_LUT_BYTES;
  return lut + (size_t)(2 * min(K, LMS_CHUNK) + 16) * sizeof(float2);
}

cudaError_t lms_setup() {
  cudaError_t e = cudaFuncSetAttribute(kk_lms_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LMS_SMEM_MAX);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kk_lms_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LMS_SMEM_MAX);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kk_lms_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LMS_SMEM_MAX);
  return e;
}

cudaError_t launch_lms(const LmsArgs& a, cudaStream_t s) {
  if (a.nchains < 1) return cudaSuccess;
  const int mode = (a.mode == 1) ? 1 : (a.mode == 2 || !(a.inv_tau > 0.f)) ? 2 : 0;
  const size_t sm = lms_smem_bytes(mode, a.K);
  if (mode == 1)
    kk_lms_kernel<1><<<a.nchains, 32, sm, s>>>(a);
  else if (mode == 2)
    kk_lms_kernel<2><<<a.nchains, 32, sm, s>>>(a);
  else
    kk_lms_kernel<0><<<a.nchains, 32, sm, s>>>(a);
  return cudaGetLastError();
}

int lms_lanes_ctas(int nchains) { return (nchains + LMSL_MAXW * 32 - 1) / (LMSL_MAXW * 32); }

cudaError_t launch_lms_lanes(const LmsArgs& a, cudaStream_t s) {
  if (a.nchains < 1) return cudaSuccess;
  static bool attr_done = false;
  if (!attr_done) {
    for (cudaError_t e : {cudaFuncSetAttribute(kk_lms_lanes_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(LMS_LUT_BYTES + 129 * sizeof(float2))),
                          cudaFuncSetAttribute(kk_lms_lanes_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(LMS_LUT_BYTES + 129 * sizeof(float2))),
                          cudaFuncSetAttribute(kk_lms_lanes_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(LMS_LUT_BYTES + 129 * sizeof(float2)))})
      if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int ctas = lms_lanes_ctas(a.nchains);
  const int threads = LMSL_MAXW * 32;  // chains spread over all warps (lms_lanes_body)
  const int mode = (a.mode == 1) ? 1 : (a.mode == 2 || !(a.inv_tau > 0.f)) ? 2 : 0;
  const size_t sm = LMS_LUT_BYTES + 129 * sizeof(float2);
  if (mode == 1)
    kk_lms_lanes_kernel<1><<<ctas, threads, sm, s>>>(a);
  else if (mode == 2)
    kk_lms_lanes_kernel<2><<<ctas, threads, sm, s>>>(a);
  else
    kk_lms_lanes_kernel<0><<<ctas, threads, sm, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Kernel 4: packed 12-bit ADC samples -> int16 codes (S0 ingest of the packed input
// format, kk_rx_submit_batch_packed12).  Two two's-complement 12-bit codes per 3 bytes,
// little-endian: b0 = c0[7:0], b1 = c0[11:8] | c1[3:0] << 4, b2 = c1[11:4].  One thread
// per 8 samples (12 bytes in, 16 bytes out); memory-bound (3.5 B per sample).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) kk_unpack12_kernel(const uint8_t* __restrict__ src, int16_t* __restrict__ dst,
                                                          int64_t n8) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n8) return;
  const uint32_t* s = reinterpret_cast<const uint32_t*>(src + 12 * t);
  const uint32_t w0 = __ldg(s), w1 = __ldg(s + 1), w2 = __ldg(s + 2);
  // 96 bits = 8 codes of 12 bits, code k at bit 12 k
  auto code = [&](int k) -> int16_t {
    const int bit = 12 * k;
    uint32_t v;
    if (bit + 12 <= 32) v = w0 >> bit;
    else if (bit < 32) v = (w0 >> bit) | (w1 << (32 - bit));
    else if (bit + 12 <= 64) v = w1 >> (bit - 32);
    else if (bit < 64) v = (w1 >> (bit - 32)) | (w2 << (64 - bit));
    else v = w2 >> (bit - 64);
    return (int16_t)((int32_t)(v << 20) >> 20);  // sign-extend 12 bits
  };
  uint4 o;
  o.x = (uint16_t)code(0) | ((uint32_t)(uint16_t)code(1) << 16);
  o.y = (uint16_t)code(2) | ((uint32_t)(uint16_t)code(3) << 16);
  o.z = (uint16_t)code(4) | ((uint32_t)(uint16_t)code(5) << 16);
  o.w = (uint16_t)code(6) | ((uint32_t)(uint16_t)code(7) << 16);
  reinterpret_cast<uint4*>(dst)[t] = o;
}

cudaError_t launch_unpack12(const uint8_t* src, int16_t* dst, int64_t n_samples, cudaStream_t s) {
  const int64_t n8 = n_samples / 8;
  if (n8 <= 0) return cudaSuccess;
  kk_unpack12_kernel<<<(unsigned)((n8 + 255) / 256), 256, 0, s>>>(src, dst, n8);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Init-time training of the static equaliser (NEXT row of SURVEY 8(f); PAPER l.53:
// "optimized offline using a training sequence every time that the data acquisition
// is initialized").  Least squares  min_h sum_n |sum_t h_t E_s[4n + 101 - t] - s_n|^2
// (+ ridge), reading R4, in fp64: the normal equations R h = b with
//   R[t1][t2] = sum_n conj(A[n][t1]) A[n][t2],  b[t] = sum_n conj(A[n][t]) s_n,
//   A[n][t] = E_s[4 (n_first + n) + 101 - t],
// accumulated by kk_gram_kernel (one 16 x 16 tile of R per CTA, the last tile row = b),
// then solved by kk_chol_solve_kernel (one CTA, right-looking Cholesky, fp64).
// ---------------------------------------------------------------------------
constexpr int GRAM_T = 16;
constexpr int CHOL_MAX_N = 256;  // largest static-EQ length the single-CTA solve stages in shared memory

__global__ void __launch_bounds__(256) kk_gram_kernel(const float2* __restrict__ es, int64_t pos_first,
                                                      const float2* __restrict__ sym, int n_count, int ntap,
                                                      double2* __restrict__ R, double2* __restrict__ bvec) {
  // tile (bx, by) of R; by == ceil(ntap/16) means the right-hand side b
  const int t1 = blockIdx.y * GRAM_T + (threadIdx.x / GRAM_T);
  const int t2 = blockIdx.x * GRAM_T + (threadIdx.x % GRAM_T);
  const int nt = (ntap + GRAM_T - 1) / GRAM_T;
  const bool rhs = (int)blockIdx.y == nt;
  if (rhs && blockIdx.x > 0) return;
  const int half = ntap / 2;
  // this CTA's slice of the training symbols and its partial-sum plane
  const int chunk = (n_count + GRAM_SPLIT - 1) / GRAM_SPLIT;
  const int nlo = (int)blockIdx.z * chunk, nhi = min(n_count, nlo + chunk);
  R += (int64_t)blockIdx.z * ntap * ntap;
  bvec += (int64_t)blockIdx.z * ntap;
  double sr = 0.0, si = 0.0;
  if (!rhs && t1 < ntap && t2 < ntap && t2 >= t1) {
    for (int n = nlo; n < nhi; ++n) {
      const int64_t base = pos_first + 4 * (int64_t)n + half;
      const float2 a1 = es[base - t1], a2 = es[base - t2];
      // conj(a1) * a2
      sr += (double)a1.x * a2.x + (double)a1.y * a2.y;
      si += (double)a1.x * a2.y - (double)a1.y * a2.x;
    }
    R[(int64_t)t1 * ntap + t2] = make_double2(sr, si);
    R[(int64_t)t2 * ntap + t1] = make_double2(sr, -si);
  } else if (rhs && threadIdx.x < GRAM_T) {
    for (int t = threadIdx.x; t < ntap; t += GRAM_T) {
      double br = 0.0, bi = 0.0;
      for (int n = nlo; n < nhi; ++n) {
        const float2 a = es[pos_first + 4 * (int64_t)n + half - t];
        const float2 s = sym[n];
        br += (double)a.x * s.x + (double)a.y * s.y;
        bi += (double)a.x * s.y - (double)a.y * s.x;
      }
      bvec[t] = make_double2(br, bi);
    }
  }
}

// (R + ridge * tr(R)/n * I) h = b, R Hermitian positive definite (n <= CHOL_MAX_N), in place;
// one CTA of 1024 threads, fp64; R in global / L2, the pivot column and the right-hand side
// staged in fixed shared arrays of CHOL_MAX_N entries.  R and b arrive as
// GRAM_SPLIT partial planes, summed here in a fixed order (deterministic).
__global__ void __launch_bounds__(1024) kk_chol_solve_kernel(double2* __restrict__ R, double2* __restrict__ b, int n,
                                                             double ridge, float* __restrict__ out) {
  __shared__ double s_tr;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    double2 t = R[i];
    for (int z = 1; z < GRAM_SPLIT; ++z) {
      const double2 q = R[(int64_t)z * n * n + i];
      t.x += q.x;
      t.y += q.y;
    }
    R[i] = t;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double2 t = b[i];
    for (int z = 1; z < GRAM_SPLIT; ++z) {
      const double2 q = b[(int64_t)z * n + i];
      t.x += q.x;
      t.y += q.y;
    }
    b[i] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int k = 0; k < n; ++k) tr += R[(int64_t)k * n + k].x;
    s_tr = tr;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) R[(int64_t)k * n + k].x += ridge * s_tr / n;
  __syncthreads();
  // Cholesky R = L L^H (lower triangle overwritten); column k of L staged in shared memory,
  // the trailing update one row per warp (j <= i over the lanes)
  __shared__ double2 s_col[CHOL_MAX_N];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int k = 0; k < n; ++k) {
    const double d = sqrt(R[(int64_t)k * n + k].x);
    const double inv = 1.0 / d;
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) {
      double2 v = R[(int64_t)i * n + k];
      v = make_double2(v.x * inv, v.y * inv);
      R[(int64_t)i * n + k] = v;
      s_col[i] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) R[(int64_t)k * n + k] = make_double2(d, 0.0);
    // trailing update R[i][j] -= L[i][k] conj(L[j][k]), k < j <= i
    for (int i = k + 1 + warp; i < n; i += nwarp) {
      const double2 li = s_col[i];
      for (int j = k + 1 + lane; j <= i; j += 32) {
        const double2 lj = s_col[j];
        double2 r = R[(int64_t)i * n + j];
        r.x -= li.x * lj.x + li.y * lj.y;
        r.y -= li.y * lj.x - li.x * lj.y;
        R[(int64_t)i * n + j] = r;
      }
    }
    __syncthreads();
  }
  // forward L y = b, backward L^H h = y: column-oriented substitution, the right-hand side
  // in shared memory, one pivot per step and the n - i remaining updates spread over the CTA
  __shared__ double2 s_b[CHOL_MAX_N];
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_b[i] = b[i];
  __syncthreads();
  for (int i = 0; i < n; ++i) {
    const double d = R[(int64_t)i * n + i].x;
    const double2 yi = make_double2(s_b[i].x / d, s_b[i].y / d);
    __syncthreads();
    if (threadIdx.x == 0) s_b[i] = yi;
    for (int j = i + 1 + threadIdx.x; j < n; j += blockDim.x) {  // y_j -= L[j][i] y_i
      const double2 l = R[(int64_t)j * n + i];
      s_b[j].x -= l.x * yi.x - l.y * yi.y;
      s_b[j].y -= l.x * yi.y + l.y * yi.x;
    }
    __syncthreads();
  }
  for (int i = n - 1; i >= 0; --i) {
    const double d = R[(int64_t)i * n + i].x;
    const double2 hi = make_double2(s_b[i].x / d, s_b[i].y / d);
    __syncthreads();
    if (threadIdx.x == 0) s_b[i] = hi;
    for (int j = threadIdx.x; j < i; j += blockDim.x) {  // y_j -= conj(L[i][j]) h_i
      const double2 l = R[(int64_t)i * n + j];
      s_b[j].x -= l.x * hi.x + l.y * hi.y;
      s_b[j].y -= l.x * hi.y - l.y * hi.x;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    out[2 * i] = (float)s_b[i].x;
    out[2 * i + 1] = (float)s_b[i].y;
  }
}

// ---------------------------------------------------------------------------
// Frame synchronisation (oracle.train.frame_sync): correlation
// of the symbol-instant field y_n = E_s[4 (n0 + n)], n < L, with the known pattern
// points over every cyclic lag k of the pattern,
//   c(k) = sum_n y_n conj(p[(n0 + n + k) mod P]),   n_off = argmax_k |c(k)| (lowest k on ties).
// One thread per lag; y and the points in shared memory, pattern bytes coalesced across
// lags; per-warp max of (|c|^2, k) -> one 64-bit atomicMax per warp (|c|^2 bits in the
// high word -- order-preserving for non-negative floats -- and ~k in the low word so
// equal magnitudes keep the lowest k); sum of |c|^2 for the mean sidelobe level.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) kk_fsync_kernel(const float2* __restrict__ es, int64_t es_first, int L,
                                                       const uint8_t* __restrict__ pattern, int64_t P, int64_t n0,
                                                       const float2* __restrict__ pts, int m,
                                                       unsigned long long* __restrict__ best, double* __restrict__ sum2,
                                                       float2* __restrict__ cval) {
  extern __shared__ float2 fs_y[];  // L field samples, then the points
  float2* fs_p = fs_y + L;
  for (int i = threadIdx.x; i < L; i += blockDim.x) fs_y[i] = es[es_first + 4 * (int64_t)i];
  for (int i = threadIdx.x; i < m; i += blockDim.x) fs_p[i] = pts[i];
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float cr = 0.f, ci = 0.f;
  if (k < P) {
    int64_t idx = (n0 + k) % P;
    for (int n = 0; n < L; ++n) {
      const float2 y = fs_y[n], p = fs_p[pattern[idx]];
      cr = fmaf(y.x, p.x, fmaf(y.y, p.y, cr));  // y conj(p)
      ci = fmaf(y.y, p.x, fmaf(-y.x, p.y, ci));
      idx = (idx + 1 == P) ? 0 : idx + 1;
    }
    if (cval) cval[k] = make_float2(cr, ci);
  }
  const float mag = (k < P) ? fmaf(cr, cr, ci * ci) : 0.f;
  unsigned long long key = (k < P) ? (((unsigned long long)__float_as_uint(mag) << 32) | (unsigned)(~(unsigned)k)) : 0ull;
  double sm = (double)mag;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
    key = ok > key ? ok : key;
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(best, key);
    atomicAdd(sum2, sm);
  }
}

cudaError_t launch_frame_sync(const float2* es, int64_t es_first, int L, const uint8_t* pattern, int64_t P, int64_t n0,
                              const float2* pts, int m, unsigned long long* best, double* sum2, float2* cval,
                              cudaStream_t s) {
  const size_t sm = (size_t)(L + m) * sizeof(float2);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kk_fsync_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  const int64_t blocks = (P + 255) / 256;
  kk_fsync_kernel<<<(unsigned)blocks, 256, sm, s>>>(es, es_first, L, pattern, P, n0, pts, m, best, sum2, cval);
  return cudaGetLastError();
}

cudaError_t launch_train_fir(const float2* es, int64_t pos_first, const float2* sym, int n_count, int ntap, double ridge,
                             double2* R, double2* b, float* out, cudaStream_t s) {
  if (ntap < 1 || ntap > CHOL_MAX_N) return cudaErrorInvalidValue;  // s_col / s_b of kk_chol_solve_kernel
  const int nt = (ntap + GRAM_T - 1) / GRAM_T;
  kk_gram_kernel<<<dim3(nt, nt + 1, GRAM_SPLIT), GRAM_T * GRAM_T, 0, s>>>(es, pos_first, sym, n_count, ntap, R, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  kk_chol_solve_kernel<<<1, 1024, 0, s>>>(R, b, ntap, ridge, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// GMI of constellations in complex AWGN (NEXT row 4 of SURVEY 8(f); the
// GS optimiser evaluates "the GMI for the AWGN channel" after every move).  Standard BICM
// GMI, Es = 1, N0 = 10^(-SNR/10), expectation over the noise by 2-D
// Gauss-Hermite quadrature (nodes t_a + i t_b, weights w_a w_b / pi):
//   GMI = nb - (1/M) sum_k sum_q W_q sum_i log2( sum_j e^{-|y-p_j|^2/N0} /
//                                                 sum_{j: b_i(j) = b_i(k)} e^{-|y-p_j|^2/N0} ),
//   y = p_k + sqrt(N0) (t_a + i t_b).
// One CTA per candidate constellation, one thread per (point k, node q); exponentials
// shifted by the nearest point, sums and logs in fp64.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) kk_gmi_kernel(const float2* __restrict__ pts, const uint8_t* __restrict__ labs,
                                                     int m, int nb, const double2* __restrict__ nodes,
                                                     const double* __restrict__ wts, int nq, double n0,
                                                     double* __restrict__ out) {
  __shared__ float2 s_p[256];
  __shared__ int s_l[256];
  __shared__ double s_red[256];
  const int c = blockIdx.x;
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    s_p[j] = pts[(int64_t)c * m + j];
    s_l[j] = labs[(int64_t)c * m + j];
  }
  __syncthreads();
  const double sq = sqrt(n0), inv = 1.0 / n0;
  double acc = 0.0;
  for (int idx = threadIdx.x; idx < m * nq; idx += blockDim.x) {
    const int k = idx / nq, q = idx - k * nq;
    const double yx = (double)s_p[k].x + sq * nodes[q].x, yy = (double)s_p[k].y + sq * nodes[q].y;
    double dmin = 1e300;
    for (int j = 0; j < m; ++j) {
      const double dx = yx - s_p[j].x, dy = yy - s_p[j].y;
      dmin = fmin(dmin, dx * dx + dy * dy);
    }
    double den = 0.0, num[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int lk = s_l[k];
    for (int j = 0; j < m; ++j) {
      const double dx = yx - s_p[j].x, dy = yy - s_p[j].y;
      const double e = exp(-(dx * dx + dy * dy - dmin) * inv);
      den += e;
      const int same = ~(s_l[j] ^ lk);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < nb && ((same >> i) & 1)) num[i] += e;
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < nb) s += log2(den / num[i]);
    acc += wts[q] * s;
  }
  s_red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s_red[threadIdx.x] += s_red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = (double)nb - s_red[0] / m;
}

cudaError_t launch_gmi(const float2* pts, const uint8_t* labs, int m, int nb, const double2* nodes, const double* wts,
                       int nq, double n0, int n_cand, double* out, cudaStream_t s) {
  kk_gmi_kernel<<<n_cand, 256, 0, s>>>(pts, labs, m, nb, nodes, wts, nq, n0, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Kernel 3: fixed-tap WL apply, decision, demap, count from materialised x2
// (used when sub_block < buffer: several tap sets per buffer)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) kk_apply_kernel(ApplyArgs a) {
  __shared__ float2 s_pts[128];
  __shared__ uint8_t s_lab[128];
  __shared__ unsigned s_red[2][4];
  for (int i = threadIdx.x; i < a.m; i += blockDim.x) {
    s_pts[i] = a.pts[i];
    s_lab[i] = a.labels[i];
  }
  __syncthreads();
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned se = 0, be = 0;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x / a.n_sym;
  if (n < a.total) {
    const int64_t nl = n - b * a.n_sym;
    const int64_t chain = b * a.nsub + nl / a.L;
    float2 w[4], g[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      w[k] = a.taps[chain * 8 + k];
      g[k] = a.taps[chain * 8 + 4 + k];
    }
    const float2* xp = a.x2 + b * (a.n_sym * 2) + 2 * nl;
    const float2 y = wl_out(w, g, xp[1], xp[0], xp[-1], xp[-2]);
    const int d = decide(y, a.lut, s_pts, a.m);
    a.out[n] = s_lab[d];
    if (a.pattern) {
      int64_t pi = (a.n_off0 + n) % a.P;
      if (pi < 0) pi += a.P;
      const int ref = a.pattern[pi];
      se = (ref != d) ? 1u : 0u;
      be = __popc((unsigned)(s_lab[d] ^ s_lab[ref]));
    }
  }
  se = warp_sum(se);
  be = warp_sum(be);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_red[0][warp] = se;
    s_red[1][warp] = be;
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.pattern) {
    unsigned ts = 0, tb = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      ts += s_red[0][k];
      tb += s_red[1][k];
    }
    if (ts) atomicAdd(&a.counts[b * 8 + C_SYMERR], (unsigned long long)ts);
    if (tb) atomicAdd(&a.counts[b * 8 + C_BITERR], (unsigned long long)tb);
  }
}

cudaError_t launch_apply(const ApplyArgs& a, cudaStream_t s) {
  const int64_t grid = (a.total + 127) / 128;
  if (grid < 1) return cudaSuccess;
  kk_apply_kernel<<<(unsigned)grid, 128, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace kk
