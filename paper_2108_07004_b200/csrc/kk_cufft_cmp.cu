// kk_cufft_cmp.cu -- cuFFT-based COMPARISON pipeline for S1-S4 (libkkrx_cufft.so).
//
// Not the product path (see include/kk_cufft_cmp.h): the north star asks for cuFFT
// "reported only as a comparison".  This is the conventional multi-kernel design --
// every intermediate (packed Hilbert windows, phi, E_s, EQ spectra, folded spectra) is
// materialised in HBM between library FFT calls -- so bench.py can set the fused chain
// kernel (libkkrx.so) beside it on the same synthetic buffers.
//
// Per buffer (positions buffer-local, N = buffer_len):
//   pairs p in [-1, NP - 1): Hilbert blocks 2p, 2p+1 keep [1024 p, 1024 p + 1024)
//   E_s on [-1024, -1024 + LES), LES = 768 * QL (a multiple of 768, >= N + 2048), so the
//   EQ windows of all buffers sit at one uniform distance (idist = 768) in one array
//   EQ blocks q in [0, QL): window E_s[768 q - 128, 768 q + 896) -> x2 [384 q, 384 q + 384)
#include <cuda_runtime.h>
#include <cufft.h>

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <map>
#include <vector>

#include "kk_cufft_cmp.h"

namespace {

constexpr int HB = 1024;   // Hilbert FFT length
constexpr int NF = 1024;   // EQ overlap-save FFT length
constexpr int KEEP = 768;  // EQ outputs per block at 4 sps
constexpr int FIR_TAPS = 203;

struct Plans {
  cufftHandle hil = 0, eq = 0, inv512 = 0;
  bool ok = false;
};

}  // namespace

struct kk_cmp {
  int64_t N = 0, NP = 0, QL = 0, LES = 0;
  int max_batch = 0;
  float dc = 0, a_hat = 0, vmin = 1;
  int64_t tb = 0;
  float2* H = nullptr;     // DFT_1024 of h placed circularly (unnormalised)
  float2* work1 = nullptr; // packed Hilbert windows, then EQ spectra Y
  float2* work2 = nullptr; // E_s, then folded spectra Z
  std::map<int, Plans> plans;
};

namespace {

// per-buffer 2-D grids (blockIdx.y = buffer) keep the index arithmetic 32-bit; the
// transcendental functions are the same MUFU forms the fused chain kernel uses
__global__ void k_pack(const int16_t* __restrict__ codes, float2* __restrict__ W, int64_t N, int per_buf, float dc,
                       float vmin) {
  const int64_t b = blockIdx.y;
  const int16_t* src = codes + b * N;
  float2* dst = W + b * (int64_t)per_buf;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < per_buf; r += gridDim.x * blockDim.x) {
    const int p = (r >> 10) - 1, m = r & (HB - 1);
    const int pos1 = HB * p - 256 + m;  // window of block 2p: 512 (2p) - 256 + m
    const float v1 = fmaxf((float)src[pos1] + dc, vmin), v2 = fmaxf((float)src[pos1 + 512] + dc, vmin);
    dst[r] = make_float2(0.5f * __logf(v1), 0.5f * __logf(v2));
  }
}

// Phi = +i sgn(k) L (reading R1), the 1/1024 of the unnormalised inverse folded in
__global__ void k_mask(float2* __restrict__ W, int64_t total) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx % HB);
    const float s = (k == 0 || k == HB / 2) ? 0.f : (k < HB / 2 ? 1.f : -1.f) * (1.0f / HB);
    const float2 z = W[idx];
    W[idx] = make_float2(-z.y * s, z.x * s);
  }
}

__global__ void k_s3(const int16_t* __restrict__ codes, const float2* __restrict__ W, float2* __restrict__ Es,
                     int64_t N, int64_t NP, int LES, float dc, float vmin, float a_hat, int64_t tb, float inv_n2) {
  const int64_t b = blockIdx.y;
  const int16_t* src = codes + b * N;
  const float2* wb = W + b * NP * HB;
  float2* dst = Es + b * (int64_t)LES;
  const bool pow2 = (N & (N - 1)) == 0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < LES; e += gridDim.x * blockDim.x) {
    const int n = e - 1024;
    const int p = (e >> 10) - 1;  // floor(n / 1024), n >= -1024
    const int r = n - HB * p;
    const float2 z = wb[(int64_t)(p + 1) * HB + 256 + (r & 511)];
    const float phi = (r < 512) ? z.x : z.y;
    const float v = fmaxf((float)src[n] + dc, vmin);
    const float a = sqrtf(v);
    float sp, cp;
    __sincosf(phi, &sp, &cp);  // |phi| of a few rad
    int64_t t = tb * (int64_t)n;
    t = pow2 ? (t & (N - 1)) : ((t % N) + N) % N;
    float st, ct;
    sincospif((float)t * inv_n2, &st, &ct);  // theta_n = 2 pi t / N
    const float ex = a * cp - a_hat, ey = a * sp;
    dst[e] = make_float2(ex * ct - ey * st, ex * st + ey * ct);
  }
}

// Z_k = (Y_k H_k + Y_{k+512} H_{k+512}) / 1024: the 4->2 fold (S4) and the 1/NF
__global__ void k_fold(const float2* __restrict__ Y, const float2* __restrict__ H, float2* __restrict__ Z,
                       int64_t total) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = idx / (NF / 2);
    const int k = (int)(idx % (NF / 2));
    const float2 y0 = Y[g * NF + k], y1 = Y[g * NF + k + NF / 2], h0 = H[k], h1 = H[k + NF / 2];
    const float zx = y0.x * h0.x - y0.y * h0.y + y1.x * h1.x - y1.y * h1.y;
    const float zy = y0.x * h0.y + y0.y * h0.x + y1.x * h1.y + y1.y * h1.x;
    Z[idx] = make_float2(zx * (1.0f / NF), zy * (1.0f / NF));
  }
}

__global__ void k_extract(const float2* __restrict__ Z, float2* __restrict__ x2, int64_t N, int64_t QL) {
  const int64_t b = blockIdx.y;
  const int half = (int)(N / 2);
  const float2* zb = Z + b * QL * (NF / 2);
  float2* dst = x2 + b * (int64_t)half;
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < half; m += gridDim.x * blockDim.x) {
    const int q = m / (KEEP / 2);
    dst[m] = zb[(int64_t)q * (NF / 2) + 64 + (m - q * (KEEP / 2))];
  }
}

int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  return (int)(g > 148 * 32 ? 148 * 32 : g);
}

dim3 grid2(int64_t per_buf, int nbuf) {
  int64_t g = (per_buf + 255) / 256;
  const int64_t cap = (148 * 32 + nbuf - 1) / nbuf;
  return dim3((unsigned)(g > cap ? cap : g), (unsigned)nbuf);
}

Plans* get_plans(kk_cmp* h, int nbuf) {
  auto it = h->plans.find(nbuf);
  if (it != h->plans.end()) return &it->second;
  Plans p;
  int n1[1] = {HB};
  const int bh = (int)(nbuf * h->NP), be = (int)(nbuf * h->QL);
  bool ok = cufftPlanMany(&p.hil, 1, n1, nullptr, 1, HB, nullptr, 1, HB, CUFFT_C2C, bh) == CUFFT_SUCCESS;
  int ne[1] = {NF}, inem[1] = {NF}, onem[1] = {NF};
  ok = ok && cufftPlanMany(&p.eq, 1, ne, inem, 1, KEEP, onem, 1, NF, CUFFT_C2C, be) == CUFFT_SUCCESS;
  int n5[1] = {NF / 2};
  ok = ok && cufftPlanMany(&p.inv512, 1, n5, nullptr, 1, NF / 2, nullptr, 1, NF / 2, CUFFT_C2C, be) == CUFFT_SUCCESS;
  p.ok = ok;
  if (!ok) {
    if (p.hil) cufftDestroy(p.hil);
    if (p.eq) cufftDestroy(p.eq);
    if (p.inv512) cufftDestroy(p.inv512);
    return nullptr;
  }
  return &(h->plans[nbuf] = p);
}

}  // namespace

extern "C" {

int kk_cmp_create(kk_cmp_t** out, int64_t buffer_len, int max_batch, float dc_offset, float a_hat, float v_min,
                  int64_t tone_bin, const float* fir, int fir_len) {
  if (!out || buffer_len <= 0 || buffer_len % 1024 != 0 || max_batch <= 0 || !fir || fir_len != FIR_TAPS ||
      !(v_min > 0.f))
    return -1;
  *out = nullptr;
  kk_cmp* h = new kk_cmp();
  h->N = buffer_len;
  h->max_batch = max_batch;
  h->dc = dc_offset;
  h->a_hat = a_hat;
  h->vmin = v_min;
  h->tb = ((tone_bin % buffer_len) + buffer_len) % buffer_len;
  h->QL = (buffer_len + 2048 + KEEP - 1) / KEEP;
  h->LES = KEEP * h->QL;
  h->NP = (h->LES + HB - 1) / HB;
  // unnormalised DFT_1024 of h placed circularly (tap i at index i mod 1024), fp64
  std::vector<float2> Hh(NF);
  for (int k = 0; k < NF; ++k) {
    std::complex<double> acc = 0;
    for (int t = 0; t < FIR_TAPS; ++t) {
      const int i = t - FIR_TAPS / 2;
      const double ang = -2.0 * M_PI * (double)(((int64_t)k * (i + NF)) % NF) / NF;
      acc += std::complex<double>(fir[2 * t], fir[2 * t + 1]) * std::complex<double>(std::cos(ang), std::sin(ang));
    }
    Hh[k] = make_float2((float)acc.real(), (float)acc.imag());
  }
  const size_t w1 = (size_t)max_batch * (size_t)(h->QL * NF > h->NP * HB ? h->QL * NF : h->NP * HB);
  const size_t w2 = (size_t)max_batch * (size_t)h->LES + 4096;  // + the last EQ window's overrun
  if (cudaMalloc(&h->H, NF * sizeof(float2)) != cudaSuccess || cudaMalloc(&h->work1, w1 * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&h->work2, w2 * sizeof(float2)) != cudaSuccess) {
    kk_cmp_destroy(h);
    return -2;
  }
  if (cudaMemcpy(h->H, Hh.data(), NF * sizeof(float2), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(h->work2, 0, w2 * sizeof(float2)) != cudaSuccess) {
    kk_cmp_destroy(h);
    return -3;
  }
  *out = h;
  return 0;
}

int kk_cmp_halo(const kk_cmp_t* h, int64_t* left, int64_t* right) {
  if (!h || !left || !right) return -1;
  *left = 1024 + 256;                          // first pair window starts at -1024 - 256
  *right = -1024 + h->NP * HB + 256 - h->N;    // last pair window ends at -1024 + NP*1024 + 256
  return 0;
}

int kk_cmp_x2(kk_cmp_t* h, const int16_t* codes, int nbuf, float* x2, void* stream) {
  if (!h || !codes || !x2 || nbuf <= 0 || nbuf > h->max_batch) return -1;
  Plans* p = get_plans(h, nbuf);
  if (!p) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  if (cufftSetStream(p->hil, st) != CUFFT_SUCCESS || cufftSetStream(p->eq, st) != CUFFT_SUCCESS ||
      cufftSetStream(p->inv512, st) != CUFFT_SUCCESS)
    return -3;
  const int64_t tw = (int64_t)nbuf * h->NP * HB, tz = (int64_t)nbuf * h->QL * (NF / 2);
  cufftComplex* W = reinterpret_cast<cufftComplex*>(h->work1);
  k_pack<<<grid2(h->NP * HB, nbuf), 256, 0, st>>>(codes, h->work1, h->N, (int)(h->NP * HB), h->dc, h->vmin);
  if (cufftExecC2C(p->hil, W, W, CUFFT_FORWARD) != CUFFT_SUCCESS) return -3;
  k_mask<<<grid_for(tw), 256, 0, st>>>(h->work1, tw);
  if (cufftExecC2C(p->hil, W, W, CUFFT_INVERSE) != CUFFT_SUCCESS) return -3;
  k_s3<<<grid2(h->LES, nbuf), 256, 0, st>>>(codes, h->work1, h->work2, h->N, h->NP, (int)h->LES, h->dc, h->vmin,
                                              h->a_hat, h->tb, (float)(2.0 / (double)h->N));
  // EQ windows straight from E_s (window of block q of buffer b at b*LES + 768 q + 896)
  if (cufftExecC2C(p->eq, reinterpret_cast<cufftComplex*>(h->work2 + 896), W, CUFFT_FORWARD) != CUFFT_SUCCESS)
    return -3;
  k_fold<<<grid_for(tz), 256, 0, st>>>(h->work1, h->H, h->work2, tz);
  cufftComplex* Z = reinterpret_cast<cufftComplex*>(h->work2);
  if (cufftExecC2C(p->inv512, Z, Z, CUFFT_INVERSE) != CUFFT_SUCCESS) return -3;
  k_extract<<<grid2(h->N / 2, nbuf), 256, 0, st>>>(h->work2, reinterpret_cast<float2*>(x2), h->N, h->QL);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int kk_cmp_launches(const kk_cmp_t* h, int nbuf) { return (h && nbuf > 0) ? 9 : 0; }

int kk_cmp_destroy(kk_cmp_t* h) {
  if (!h) return 0;
  for (auto& kv : h->plans) {
    cufftDestroy(kv.second.hil);
    cufftDestroy(kv.second.eq);
    cufftDestroy(kv.second.inv512);
  }
  cudaFree(h->H);
  cudaFree(h->work1);
  cudaFree(h->work2);
  delete h;
  return 0;
}

}  // extern "C"
