// FFMA vs FFMA2 throughput (lane-ops per clock per SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k1(float* out, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A83126F;" : "+f"(a[i]));
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* out, int iters) {
  uint64_t a[8];
  for (int i = 0; i < 8; ++i) { float2 f = make_float2(0.001f * (threadIdx.x + i), 0.002f * i); a[i] = *reinterpret_cast<uint64_t*>(&f); }
  const float2 cb = make_float2(0.99f, 0.98f), cc = make_float2(0.001f, 0.002f);
  const uint64_t b = *reinterpret_cast<const uint64_t*>(&cb), c = *reinterpret_cast<const uint64_t*>(&cc);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(b), "l"(c));
  float s = 0; for (int i = 0; i < 8; ++i) { float2 f = *reinterpret_cast<float2*>(&a[i]); s += f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int threads : {128, 256, 512, 1024}) {
    float ms1 = 0, ms2 = 0;
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0); k1<<<148, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms1, e0, e1);
      cudaEventRecord(e0); k2<<<148, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms2, e0, e1);
    }
    const double ops = 148.0 * threads * iters * 16;  // lane-FMAs (both kernels)
    printf("threads %4d: FFMA %.1f  FFMA2 %.1f lane-FMA/clk/SM (clock %.0f MHz)\n", threads,
           ops / (ms1 * 1e-3) / 148 / (clk * 1e3), ops / (ms2 * 1e-3) / 148 / (clk * 1e3), clk / 1e3);
  }
  return 0;
}
