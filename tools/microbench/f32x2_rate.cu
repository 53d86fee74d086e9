// Throughput / latency of scalar FP32 vs packed FP32x2 (FFMA2/FADD2) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f32x2_rate f32x2_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ float ffma1(float a, float b, float c) { float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ float fadd1(float a, float b) { float r; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }

template <int ILP>
__global__ void k_ffma(float* out, int iters, float m) {
  float acc[ILP];
  for (int j = 0; j < ILP; ++j) acc[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc[j] = ffma1(acc[j], m, 0.5f);
  float s = 0; for (int j = 0; j < ILP; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP>
__global__ void k_fadd(float* out, int iters, float m) {
  float acc[ILP];
  for (int j = 0; j < ILP; ++j) acc[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc[j] = fadd1(acc[j], m);
  float s = 0; for (int j = 0; j < ILP; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP>
__global__ void k_ffma2(float* out, int iters, float m) {
  u64 acc[ILP];
  for (int j = 0; j < ILP; ++j) { float2 f = make_float2(threadIdx.x * 1e-3f + j, j); acc[j] = *(u64*)&f; }
  float2 mm = make_float2(m, m), hh = make_float2(0.5f, 0.5f);
  u64 M = *(u64*)&mm, H = *(u64*)&hh;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc[j] = ffma2(acc[j], M, H);
  float s = 0; for (int j = 0; j < ILP; ++j) { float2 f = *(float2*)&acc[j]; s += f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP>
__global__ void k_fadd2(float* out, int iters, float m) {
  u64 acc[ILP];
  for (int j = 0; j < ILP; ++j) { float2 f = make_float2(threadIdx.x * 1e-3f + j, j); acc[j] = *(u64*)&f; }
  float2 mm = make_float2(m, m);
  u64 M = *(u64*)&mm;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc[j] = fadd2(acc[j], M);
  float s = 0; for (int j = 0; j < ILP; ++j) { float2 f = *(float2*)&acc[j]; s += f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
float run(K k, int blocks, int threads, int iters, float* out) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<blocks, threads>>>(out, iters, 0.999f);
  cudaEventRecord(a);
  k<<<blocks, threads>>>(out, iters, 0.999f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 26);
  const int iters = 1 << 16;
  for (int warps : {4, 8, 16, 32}) {
    const int blocks = sms, threads = 32 * warps;
    const double inst = (double)blocks * warps * iters * 8;  // warp-instructions (ILP 8)
    float t1 = run(k_ffma<8>, blocks, threads, iters, out), t2 = run(k_ffma2<8>, blocks, threads, iters, out);
    float t3 = run(k_fadd<8>, blocks, threads, iters, out), t4 = run(k_fadd2<8>, blocks, threads, iters, out);
    // per SM sub-partition per cycle at the measured clock -> report warp-inst/ns/SM and lane-ops/ns/SM
    printf("warps/SM %2d  FFMA %.3f  FFMA2 %.3f  FADD %.3f  FADD2 %.3f  (warp-instructions per ns per SM; x32 / x64 lanes)\n",
           warps, inst / sms / (t1 * 1e6), inst / sms / (t2 * 1e6), inst / sms / (t3 * 1e6), inst / sms / (t4 * 1e6));
  }
  // latency: one dependent chain per warp, 1 warp per SM
  {
    const double inst = (double)sms * 1 * iters * 1;
    float t1 = run(k_ffma<1>, sms, 32, iters, out), t2 = run(k_ffma2<1>, sms, 32, iters, out);
    printf("dependent chain: FFMA %.2f ns/inst  FFMA2 %.2f ns/inst\n", t1 * 1e6 / (iters), t2 * 1e6 / (iters));
  }
  cudaFree(out);
  return 0;
}
