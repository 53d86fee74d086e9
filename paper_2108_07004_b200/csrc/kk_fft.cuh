// kk_fft.cuh -- warp-level register/shared-memory FFT building blocks (sm_100a).
//
// The KK chain needs 1024-point complex FFTs (Hilbert, "a pair of
// 100% overlap-save 1024-point FFTs"; static EQ, l.47 "another pair of FFTs")
// and a 512-point inverse FFT after the 4->2 spectral fold.  One warp owns one
// transform: 32 lanes x 32 complex registers.  A 1024-point transform is the
// four-step factorisation 1024 = 32 x 32:
//   pass A: 32-point DFT over the register index (in registers, no memory)
//   twiddle W_1024^(lane*r) from a 32x32 shared table
//   one 32x32 transpose through a per-warp padded shared tile (re, then im)
//   pass B: 32-point DFT over the register index
// so each point crosses shared memory once per transform (not once per radix-2
// stage as a shared-memory Stockham would).
//
// The 32-point DFT is radix-2 decimation in TIME with the twiddle folded into
// the butterfly as FFMAs: for w = c(1 + i t) (t = tan),
//   p = b.x - t b.y, q = b.y + t b.x;  a +- w b = (a.x +- c p, a.y +- c q)
// = 6 FP32 instructions per general butterfly (8 for mul-then-add), 4 for
// trivial twiddles; all twiddle constants are immediates.
//
// Code size matters (an early version with every transform inlined at five
// call sites was instruction-fetch bound, 271 KB of SASS): there is exactly ONE
// copy of the 32-point and of the 16-point DFT; passes and transforms are loops
// (#pragma unroll 1) around them, and every inverse transform is computed as
// conj(DFT(conj(x))).
//
// Layout contract ("lane layout"): element e of a length-1024 sequence lives in
// lane (e % 32), register (e / 32), for inputs and outputs alike.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace kk {

__host__ __device__ constexpr int brev(int k, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((k >> i) & 1) << (bits - 1 - i);
  return r;
}

// cos(2*pi*m/32), m = 0..31 (correctly rounded float literals)
__host__ __device__ constexpr float cos32(int m) {
  constexpr float t[8] = {1.0f, 0.98078528040323043f, 0.92387953251128674f, 0.83146961230254524f,
                          0.70710678118654752f, 0.55557023301960218f, 0.38268343236508977f,
                          0.19509032201612825f};
  m &= 31;
  return (m < 8) ? t[m] : (m == 8) ? 0.0f : (m < 16) ? -t[16 - m] : (m < 24) ? -t[m - 16]
         : (m == 24) ? 0.0f : t[32 - m];
}
__host__ __device__ constexpr float sin32(int m) { return cos32(m - 8); }

// Complex arithmetic on the packed FP32x2 instructions of sm_100 (FADD2 / FMUL2 / FFMA2:
// one issue slot for both halves of a float2).  The kernel is instruction-issue bound
// (DESIGN.md section 6), so this halves the issue cost of the FFT arithmetic.  ptxas
// folds the operand permutations used below into the instructions' own modifiers:
// swapped halves (.LO_HI), a per-half sign (.NP), a negated operand and a broadcast scalar
// or immediate -- checked in the SASS (cuobjdump).  Each half is an IEEE fma /
// add / mul, identical to the scalar instruction.  -DKK_F32X2=0 restores scalar code.
#ifndef KK_F32X2
#define KK_F32X2 1
#endif
#if KK_F32X2
typedef unsigned long long kk_u64;
__device__ __forceinline__ kk_u64 f2p(float2 a) {
  kk_u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 p2f(kk_u64 v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  kk_u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2p(a)), "l"(f2p(b)));
  return p2f(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  kk_u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2p(a)), "l"(f2p(b)));
  return p2f(r);
}
// a * b + c per half
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  kk_u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2p(a)), "l"(f2p(b)), "l"(f2p(c)));
  return p2f(r);
}
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return add2(a, b); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return add2(a, make_float2(-b.x, -b.y)); }
// a b = b.x a + b.y (-a.y, a.x): FMUL2 + FFMA2
__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
  return fma2(make_float2(-a.y, a.x), make_float2(b.y, b.y), mul2(a, make_float2(b.x, b.x)));
}
#else
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
#endif
__device__ __forceinline__ float2 c_conj(float2 a) { return make_float2(a.x, -a.y); }

// ---------------------------------------------------------------------------
// Per-lane tables in tensor memory (TMEM).  Every table the transforms read per lane --
// the 1024-point twiddles W^(lane r), the 512-point twiddles and the static-EQ spectrum
// H[lane + 32 k] -- depends only on the lane index, so each thread can hold its own copy in
// its TMEM lane (tcgen05.ld 32x32b: thread t of a warp reads TMEM lane 32 (warp % 4) + t).
// That moves ~0.33 shared-memory wavefronts per ADC sample (22 % of the kernel's shared
// traffic) onto the TMEM read path, which nothing else in this kernel uses (no tensor-core
// work: DESIGN.md "No tensor cores").  -DKK_TMEM_TABLES=0 restores the shared-memory tables.
#ifndef KK_TMEM_TABLES
#define KK_TMEM_TABLES 1
#endif
constexpr int TM_TW1024 = 0;   // columns 2(r-1), 2(r-1)+1: W1024^(lane r), r = 1..31 (+2 pad columns)
constexpr int TM_TW512 = 64;   // W512^(lane r), r = 1..15 (+2 pad)
constexpr int TM_H = 96;       // H[lane + 32 k], k = 0..31
constexpr int TM_NCOLS = 160;
constexpr int TM_ALLOC = 256;  // allocation: power of two >= TM_NCOLS

// 4 complex values (8 TMEM columns) of this thread's lane; asynchronous until tm_wait
__device__ __forceinline__ void tm_ld4(uint32_t taddr, float2 (&t)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(t[0].x), "=f"(t[0].y), "=f"(t[1].x), "=f"(t[1].y), "=f"(t[2].x), "=f"(t[2].y), "=f"(t[3].x),
                 "=f"(t[3].y)
               : "r"(taddr));
}
// completes every earlier tm_ld4 of this thread; t = the registers of the one to be used next
// (tied so no use of them can be scheduled before the wait)
__device__ __forceinline__ void tm_wait(float2 (&t)[4]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(t[0].x), "+f"(t[0].y), "+f"(t[1].x), "+f"(t[1].y), "+f"(t[2].x), "+f"(t[2].y), "+f"(t[3].x),
                 "+f"(t[3].y)::"memory");
}
__device__ __forceinline__ void tm_st2(uint32_t taddr, float2 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// v[r] *= table[r] for r = R0 .. R0 + 4 NCH - 1 (r < NR), table columns col0 + 2 (r - R0), chunks of 4
// pipelined one ahead (TMEM load latency ~12 cycles)
template <int N, int R0, int NR, int NCH>
__device__ __forceinline__ void tm_twiddle(float2 (&v)[N], uint32_t taddr) {
  float2 t[2][4];
  tm_ld4(taddr, t[0]);
  tm_wait(t[0]);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    if (c + 1 < NCH) tm_ld4(taddr + 8 * (c + 1), t[(c + 1) & 1]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = R0 + 4 * c + j;
      if (r < NR) v[r] = c_mul(v[r], t[c & 1][j]);
    }
    if (c + 1 < NCH) tm_wait(t[(c + 1) & 1]);
  }
}

// a * exp(-2*pi*i*m/32) (used outside the butterflies)
__device__ __forceinline__ float2 tw32(float2 a, int m) {
  m &= 31;
  if (m == 0) return a;
  if (m == 16) return make_float2(-a.x, -a.y);
  if (m == 8) return make_float2(a.y, -a.x);
  if (m == 24) return make_float2(-a.y, a.x);
  const float c = cos32(m);
  const float s = -sin32(m);
#if KK_F32X2
  // c a + s (-a.y, a.x)
  return fma2(make_float2(-a.y, a.x), make_float2(s, s), mul2(a, make_float2(c, c)));
#else
  return make_float2(fmaf(a.x, c, -a.y * s), fmaf(a.x, s, a.y * c));
#endif
}

// DIT butterfly: (a, b) <- (a + w b, a - w b), w = exp(-2 pi i m / 32), m compile-time.
__device__ __forceinline__ void bfly(float2& a, float2& b, int m) {
  m &= 31;
  if (m == 0) {
    const float2 t = b;
    b = c_sub(a, t);
    a = c_add(a, t);
  } else if (m == 8) {  // w = -i: w b = (b.y, -b.x)
    const float2 t = make_float2(b.y, -b.x);
    b = c_sub(a, t);
    a = c_add(a, t);
  } else if (m == 24) {  // w = +i
    const float2 t = make_float2(-b.y, b.x);
    b = c_sub(a, t);
    a = c_add(a, t);
  } else if (m == 16) {
    const float2 t = make_float2(-b.x, -b.y);
    b = c_sub(a, t);
    a = c_add(a, t);
  } else {
    const float c = cos32(m);
    const float s = -sin32(m);
#if KK_F32X2
    // w = c (1 + i t), t = s / c (|t| <= tan(7 pi / 16) ~ 5.03; the result's rounding error
    // stays <= (|c| + |s|) eps |b|): pq = b + t (-b.y, b.x) [one FFMA2 with a swapped,
    // half-negated operand], then a +- c pq [two FFMA2 with a broadcast immediate]
    const float t = s / c;
    const float2 a0 = a;
    const float2 pq = (m == 4 || m == 12 || m == 20 || m == 28)
                          ? c_add(b, (t > 0) ? make_float2(-b.y, b.x) : make_float2(b.y, -b.x))
                          : fma2(make_float2(b.y, b.x), make_float2(-t, t), b);
    a = fma2(pq, make_float2(c, c), a0);
    b = fma2(pq, make_float2(-c, -c), a0);
#else
    if (m == 4 || m == 12 || m == 20 || m == 28) {
      // |t| == 1: p = b.x - t b.y, q = b.y + t b.x are plain adds
      const float t = s / c;
      const float p = (t > 0) ? b.x - b.y : b.x + b.y;
      const float q = (t > 0) ? b.y + b.x : b.y - b.x;
      const float2 a0 = a;
      a = make_float2(fmaf(c, p, a0.x), fmaf(c, q, a0.y));
      b = make_float2(fmaf(-c, p, a0.x), fmaf(-c, q, a0.y));
    } else if (m < 4 || (m > 12 && m < 20) || m > 28) {
      // |cos| > |sin|: factor cos
      const float t = s / c;
      const float p = fmaf(-t, b.y, b.x), q = fmaf(t, b.x, b.y);
      const float2 a0 = a;
      a = make_float2(fmaf(c, p, a0.x), fmaf(c, q, a0.y));
      b = make_float2(fmaf(-c, p, a0.x), fmaf(-c, q, a0.y));
    } else {
      // |sin| > |cos|: w = s (ct + i) with ct = c/s:  w b = s (ct b.x - b.y, ct b.y + b.x)
      const float ct = c / s;
      const float p = fmaf(ct, b.x, -b.y), q = fmaf(ct, b.y, b.x);
      const float2 a0 = a;
      a = make_float2(fmaf(s, p, a0.x), fmaf(s, q, a0.y));
      b = make_float2(fmaf(-s, p, a0.x), fmaf(-s, q, a0.y));
    }
#endif
  }
}

// Forward DFT of length N (N in {16, 32}) over the register index, radix-2
// decimation in time, in place on BIT-REVERSED input storage:
//   on entry v[brev(n)] holds x[n]; on exit v[k] holds X[k] = sum_n x[n] e^{-2 pi i n k / N}.
// (DIT wants t[k] = x[brev(k)]; with that storage t is v itself, so no register
// permutation is ever materialised.  Producers write their data bit-reversed for free.)
template <int N>
__device__ __forceinline__ void dft_brin(float2 (&v)[N]) {
  constexpr int LOGN = (N == 16) ? 4 : 5;
#pragma unroll
  for (int st = 0; st < LOGN; ++st) {
    const int half = 1 << st;  // butterfly span
#pragma unroll
    for (int start = 0; start < N; start += 2 * half) {
#pragma unroll
      for (int j = 0; j < half; ++j) bfly(v[start + j], v[start + j + half], j * (32 / (2 * half)));
    }
  }
}

// Forward 1024-point DFT of one warp:
//   in : x[lane + 32 n2] at v[brev5(n2)]  (lane layout, registers bit-reversed)
//   out: X[lane + 32 k2] at v[k2]          (lane layout, natural)
//   X[k] = sum_n x[n] e^{-2 pi i n k / 1024}
// scr: this warp's tile (31 x 33 float2 + pad); tw: shared table tw[r*32 + l] = e^{-2 pi i r l / 1024} (no TMEM).
// One copy of the 32-point DFT: the two passes are a loop.
// tm: this warp's TMEM table address (lane quarter, column 0) when KK_TMEM_TABLES.
// The transpose goes through a 32 x 33 float2 tile whose rows 0..30 are scr + 33 r and whose
// row 31 is `pad` (32 float2 at a bank offset of scr + 1023, i.e. pad = scr - 1 mod 16
// float2): every access is base + immediate (no per-access address arithmetic) and both
// directions are conflict-free (store: 16 consecutive float2 per half-warp; load at column
// n: lanes hit banks (l + n) mod 16), so the tile fits the warp's 1024-float2 slice + pad.
__device__ __forceinline__ void fft1024(float2 (&v)[32], int lane, float* __restrict__ scr,
                                        const float2* __restrict__ tw, uint32_t tm,
                                        float2* __restrict__ pad) {
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    dft_brin<32>(v);
    if (pass == 0) {
#if KK_TMEM_TABLES
      tm_twiddle<32, 1, 32, 8>(v, tm + TM_TW1024);
#else
#pragma unroll
      for (int r = 1; r < 32; ++r) v[r] = c_mul(v[r], tw[r * 32 + lane]);
#endif
      float2* s2 = reinterpret_cast<float2*>(scr);
#pragma unroll
      for (int r = 0; r < 31; ++r) s2[r * 33 + lane] = v[r];
      pad[lane] = v[31];
      __syncwarp();
      const float2* row = (lane < 31) ? s2 + 33 * lane : pad;
#pragma unroll
      for (int n = 0; n < 32; ++n) v[brev(n, 5)] = row[n];
      __syncwarp();
    }
  }
}

// Forward 512-point DFT of the folded spectrum, one warp:
//   in : Z[lane + 32*k2] at z[brev4(k2)], k2 in [0,16)   (registers bit-reversed)
//   out: lane (2*r1 + h) gets z[r2] = X[r1 + 16*(r2 + 16*h)],  X[r] = sum_k Z[k] e^{-2 pi i k r / 512}
// scr: this warp's tile (>= 16 x 34 float2, 8-B aligned); tw512[r1*32 + l] = e^{-2 pi i r1 l / 512} (shared).
// The inverse transform the method needs is conj(DFT(conj(Z))), done by the caller.
__device__ __forceinline__ void fft512_pairs(float2 (&z)[16], int lane, float* __restrict__ scr,
                                             const float2* __restrict__ tw512, uint32_t tm) {
  const int h = lane & 1, r1 = lane >> 1;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    dft_brin<16>(z);
    if (pass == 0) {
#if KK_TMEM_TABLES
      tm_twiddle<16, 1, 16, 4>(z, tm + TM_TW512);
#else
#pragma unroll
      for (int r = 1; r < 16; ++r) z[r] = c_mul(z[r], tw512[r * 32 + lane]);
#endif
      // one 64-bit transpose through 16 rows of 34 float2 (row stride = 2 mod 16 bank pairs:
      // stores of a row and the lanes' (r1, h) reads of column pairs are both conflict-free)
      float2* s2 = reinterpret_cast<float2*>(scr);
#pragma unroll
      for (int r = 0; r < 16; ++r) s2[r * 34 + lane] = z[r];
      __syncwarp();
      const float2* row = s2 + r1 * 34 + h;
#pragma unroll
      for (int j = 0; j < 16; ++j) z[brev(j, 4)] = row[2 * j];
      __syncwarp();
    }
  }
  // radix-2 across the lane pair: X[r2] = E[r2] + W32^{r2} O[r2], X[r2+16] = E[r2] - W32^{r2} O[r2].
  // The odd lane twiddles its own O first; then out = sgn * mine + other (no selects on the data path).
  const float sg = h ? -1.0f : 1.0f;
#pragma unroll
  for (int r2 = 0; r2 < 16; ++r2) {
    const float2 t = tw32(z[r2], r2);
    const float2 mine = h ? t : z[r2];
    float2 other;
    other.x = __shfl_xor_sync(0xffffffffu, mine.x, 1);
    other.y = __shfl_xor_sync(0xffffffffu, mine.y, 1);
#if KK_F32X2
    z[r2] = fma2(mine, make_float2(sg, sg), other);
#else
    z[r2] = make_float2(fmaf(sg, mine.x, other.x), fmaf(sg, mine.y, other.y));
#endif
  }
}

}  // namespace kk
