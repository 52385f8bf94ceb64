// Microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) issue/pipe throughput on sm_100a.
// Each thread runs ITERS iterations of 8 independent FMA chains (FFMA) or 4 independent
// FFMA2 chains (same FMA count), optionally interleaved with integer ALU work.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
template <int ALU>
__global__ void k_ffma(float* out, int iters, float s) {
  float a[8];
  unsigned x = threadIdx.x;
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 0.001f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], s, 0.5f * k + s);
#pragma unroll
    for (int q = 0; q < ALU; ++q) x = (x ^ (x << 3)) + q;
  }
  float t = 0;
  for (int k = 0; k < 8; ++k) t += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t + x;
}
template <int ALU>
__global__ void k_ffma2(float* out, int iters, float s) {
  u64 a[4], sv, cv[4];
  unsigned x = threadIdx.x;
  float2 ss = make_float2(s, s);
  sv = *reinterpret_cast<u64*>(&ss);
  for (int k = 0; k < 4; ++k) {
    float2 v = make_float2(threadIdx.x * 0.001f + 2 * k, threadIdx.x * 0.001f + 2 * k + 1);
    a[k] = *reinterpret_cast<u64*>(&v);
    float2 c = make_float2(0.5f * (2 * k) + s, 0.5f * (2 * k + 1) + s);
    cv[k] = *reinterpret_cast<u64*>(&c);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = f2fma(a[k], sv, cv[k]);
#pragma unroll
    for (int q = 0; q < ALU; ++q) x = (x ^ (x << 3)) + q;
  }
  float t = 0;
  for (int k = 0; k < 4; ++k) {
    float2 v = *reinterpret_cast<float2*>(&a[k]);
    t += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t + x;
}
template <typename K>
float run(K kern, float* out, int iters, int blocks, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters, 0.999f);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, iters, 0.999f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 8, iters = 20000;
  float* out;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  const double fmas = (double)blocks * threads * iters * 8;
  float t;
  t = run(k_ffma<0>, out, iters, blocks, threads);
  printf("FFMA  alu0: %.3f ms  %.1f TFMA/s\n", t, fmas / t / 1e9);
  t = run(k_ffma2<0>, out, iters, blocks, threads);
  printf("FFMA2 alu0: %.3f ms  %.1f TFMA/s\n", t, fmas / t / 1e9);
  t = run(k_ffma<4>, out, iters, blocks, threads);
  printf("FFMA  alu4: %.3f ms  %.1f TFMA/s\n", t, fmas / t / 1e9);
  t = run(k_ffma2<4>, out, iters, blocks, threads);
  printf("FFMA2 alu4: %.3f ms  %.1f TFMA/s\n", t, fmas / t / 1e9);
  t = run(k_ffma<8>, out, iters, blocks, threads);
  printf("FFMA  alu8: %.3f ms  %.1f TFMA/s\n", t, fmas / t / 1e9);
  t = run(k_ffma2<8>, out, iters, blocks, threads);
  printf("FFMA2 alu8: %.3f ms  %.1f TFMA/s\n", t, fmas / t / 1e9);
  return 0;
}
