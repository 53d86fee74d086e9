// kk_fft.cuh -- warp-level register/shared-memory FFT building blocks (sm_100a).
//
// The KK chain needs 1024-point complex FFTs (Hilbert, "a pair of
// 100% overlap-save 1024-point FFTs"; static EQ, l.47 "another pair of FFTs")
// and a 512-point inverse FFT after the 4->2 spectral fold.  One warp owns one
// transform: 32 lanes x 32 complex registers.  A 1024-point transform is the
// four-step factorisation 1024 = 32 x 32:
//   pass A: 32-point DFT over the register index (in registers, no memory)
//   twiddle W_1024^(lane*r) from a 32x32 shared table
//   one 32x32 transpose through a per-warp padded shared tile
//   pass B: 32-point DFT over the register index
// so each point crosses shared memory once per transform (not once per radix-2
// stage as a shared-memory Stockham would), and all butterflies are FP32
// FFMA/FADD with compile-time twiddles (immediate operands).
//
// Layout contract ("lane layout"): element e of a length-1024 sequence lives in
// lane (e % 32), register (e / 32).  Forward and inverse transforms both take
// and return this layout, so FFT -> pointwise -> IFFT needs no reordering.
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

__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 c_mulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}

// a * exp(S*2*pi*i*m/32), m a compile-time constant after unrolling; S = -1 forward, +1 inverse.
template <int S>
__device__ __forceinline__ float2 tw32(float2 a, int m) {
  m &= 31;
  if (m == 0) return a;
  if (m == 16) return make_float2(-a.x, -a.y);
  if (m == 8) return (S > 0) ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);    // *(+-i)
  if (m == 24) return (S > 0) ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
  const float c = cos32(m);
  const float s = (S > 0) ? sin32(m) : -sin32(m);
  if (m == 4 || m == 12 || m == 20 || m == 28) {
    // |c| == |s| == sqrt(1/2): (a.x c - a.y s, a.x s + a.y c) with one multiply each
    return make_float2((a.x * (c > 0 ? 1.f : -1.f) - a.y * (s > 0 ? 1.f : -1.f)) * 0.70710678118654752f,
                       (a.x * (s > 0 ? 1.f : -1.f) + a.y * (c > 0 ? 1.f : -1.f)) * 0.70710678118654752f);
  }
  return make_float2(fmaf(a.x, c, -a.y * s), fmaf(a.x, s, a.y * c));
}

// In-register radix-2 decimation-in-frequency DFT of length N (N | 32) over v[0..N):
//   V[k] = sum_n v[n] exp(S*2*pi*i*n*k/N),  result V[k] stored at v[brev(k)].
template <int N, int S>
__device__ __forceinline__ void dft_dif(float2 (&v)[N]) {
  constexpr int LOGN = (N == 2) ? 1 : (N == 4) ? 2 : (N == 8) ? 3 : (N == 16) ? 4 : 5;
#pragma unroll
  for (int st = 0; st < LOGN; ++st) {
    const int span = N >> (st + 1);
#pragma unroll
    for (int start = 0; start < N; start += 2 * span) {
#pragma unroll
      for (int j = 0; j < span; ++j) {
        float2 a = v[start + j], b = v[start + j + span];
        v[start + j] = c_add(a, b);
        // twiddle W_{2 span}^j = W_32^{j * 32 / (2 span)}
        v[start + j + span] = tw32<S>(c_sub(a, b), j * (32 / (2 * span)));
      }
    }
  }
}

// Natural-order DFT over the register index: v[k] = sum_n v_in[n] W_N^{S n k}.
template <int N, int S>
__device__ __forceinline__ void dft_reg(float2 (&v)[N]) {
  dft_dif<N, S>(v);
  float2 t[N];
#pragma unroll
  for (int k = 0; k < N; ++k) t[k] = v[brev(k, (N == 16) ? 4 : 5)];
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = t[k];
}

// 1024-point DFT of one warp, lane layout in and out.
//   S = -1: X[k] = sum_n x[n] e^{-2 pi i n k / 1024}
//   S = +1: x[n] = sum_k X[k] e^{+2 pi i n k / 1024}   (unnormalised)
// scr: this warp's 32 x 33 float2 tile; tw: shared table tw[r*32 + l] = e^{-2 pi i r l / 1024}.
template <int S>
__device__ __forceinline__ void fft1024(float2 (&v)[32], int lane, float2* __restrict__ scr,
                                        const float2* __restrict__ tw) {
  dft_dif<32, S>(v);  // v[brev(r)] = pass-A output index r
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    float2 t = v[brev(r, 5)];
    if (r != 0) {
      const float2 w = tw[r * 32 + lane];
      t = (S < 0) ? c_mul(t, w) : c_mulc(t, w);
    }
    scr[r * 33 + lane] = t;
  }
  __syncwarp();
#pragma unroll
  for (int n = 0; n < 32; ++n) v[n] = scr[lane * 33 + n];
  __syncwarp();
  dft_reg<32, S>(v);
}

// Inverse 512-point DFT after the spectral fold, one warp.
//   in : z[k2] = Z[lane + 32*k2], k2 in [0,16)
//   out: lane (2*r1 + h) gets o[r2] = x[r1 + 16*(r2 + 16*h)], r1 in [0,16), r2 in [0,16)
//        x[r] = sum_k Z[k] e^{+2 pi i k r / 512}  (unnormalised)
// scr: this warp's tile (>= 16 x 34 float2); tw512[r1*32 + l] = e^{-2 pi i r1 l / 512}.
__device__ __forceinline__ void ifft512_fold_out(float2 (&z)[16], int lane, float2* __restrict__ scr,
                                                 const float2* __restrict__ tw512, float2 (&o)[16]) {
  dft_dif<16, +1>(z);  // z[brev4(r1)] = sum_k2 Z[lane+32k2] w16^{k2 r1}
#pragma unroll
  for (int r1 = 0; r1 < 16; ++r1) {
    float2 t = z[brev(r1, 4)];
    if (r1 != 0) t = c_mulc(t, tw512[r1 * 32 + lane]);
    scr[r1 * 34 + lane] = t;
  }
  __syncwarp();
  const int h = lane & 1, r1 = lane >> 1;
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j] = scr[r1 * 34 + 2 * j + h];
  __syncwarp();
  dft_reg<16, +1>(o);  // o[r2] = sum_j A[2j+h][r1] w16^{j r2}  (E for h=0, O for h=1)
#pragma unroll
  for (int r2 = 0; r2 < 16; ++r2) {
    const float2 mine = o[r2];
    float2 other;
    other.x = __shfl_xor_sync(0xffffffffu, mine.x, 1);
    other.y = __shfl_xor_sync(0xffffffffu, mine.y, 1);
    const float2 ev = h ? other : mine;
    const float2 od = tw32<+1>(h ? mine : other, r2);  // W_32^{+r2} O[r2]
    o[r2] = h ? c_sub(ev, od) : c_add(ev, od);
  }
}

}  // namespace kk
