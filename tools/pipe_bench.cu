// Micro-benchmark of per-SM issue rates on B200 for the instruction mix of the
// render kernels (FFMA, FFMA2, FMUL2, FMNMX, FSEL, FSETP, SEL, MUFU.EX2).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipe_bench tools/pipe_bench.cu
// Prints warp-instructions per cycle per SM for each op (4.0 = one per SMSP per clock).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r, x, y, z;
  x = *reinterpret_cast<unsigned long long*>(&a);
  y = *reinterpret_cast<unsigned long long*>(&b);
  z = *reinterpret_cast<unsigned long long*>(&c);
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(y), "l"(z));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int OP>
__global__ void k(float* out, float s0, float s1, long long* cyc) {
  float a[kChains], b[kChains];
  float2 p[kChains];
  int iv[kChains];
  for (int c = 0; c < kChains; ++c) {
    a[c] = s0 + threadIdx.x * 1e-3f + c;
    b[c] = s1 - c * 1e-3f;
    p[c] = make_float2(a[c], b[c]);
    iv[c] = threadIdx.x + c;
  }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (OP == 0) a[c] = fmaf(a[c], b[c], s0);            // FFMA (reg, reg, const)
      if (OP == 1) a[c] = fmaf(a[c], b[c], b[(c + 1) % kChains]);  // FFMA 3-reg
      if (OP == 2) p[c] = ffma2(p[c], p[(c + 1) % kChains], p[(c + 2) % kChains]);  // FFMA2
      if (OP == 3) a[c] = fminf(-a[c], b[c]);               // FMNMX
      if (OP == 4) a[c] = (a[c] > b[c]) ? b[(c + 1) % kChains] : a[c];  // FSETP + FSEL
      if (OP == 5) a[c] = ex2(a[c]);                        // MUFU.EX2
      if (OP == 6) iv[c] = (iv[c] & 1) ? iv[(c + 1) % kChains] : (iv[c] ^ 0x55);  // LOP3+SEL
      if (OP == 7) a[c] = a[c] * b[c];                      // FMUL
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
  for (int c = 0; c < kChains; ++c) acc += a[c] + p[c].x + p[c].y + (float)iv[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps_per_sm) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 32 * warps_per_sm;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * nsm * threads);
  cudaMalloc(&cyc, sizeof(long long) * nsm);
  k<OP><<<nsm, threads>>>(out, 0.5f, 0.999f, cyc);
  k<OP><<<nsm, threads>>>(out, 0.5f, 0.999f, cyc);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < nsm; ++i) mean += h[i];
  mean /= nsm;
  const double ops = (double)kIters * kChains * warps_per_sm;  // warp-instructions per SM
  printf("%-22s warps/SM %3d: %.3f warp-inst/clk/SM\n", name, warps_per_sm, ops / mean);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {16, 32}) {
    run<0>("FFMA reg,reg,const", w);
    run<1>("FFMA 3-reg", w);
    run<2>("FFMA2 (pairs)", w);
    run<7>("FMUL", w);
    run<3>("FMNMX", w);
    run<4>("FSETP+FSEL (x2 inst)", w);
    run<5>("MUFU.EX2", w);
    run<6>("LOP3+SEL (x2 inst)", w);
  }
  return 0;
}
