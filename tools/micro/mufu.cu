// Throughput of MUFU.EX2 vs FFMA2 on one SM-resident workload (microbenchmark).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ex2(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A83126F;" : "+f"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int threads : {128, 256, 512, 1024}) {
    for (int w = 0; w < 2; ++w) {
      k_ex2<<<148, threads>>>(out, iters); k_ffma<<<148, threads>>>(out, iters);
      cudaEventRecord(e0); k_ex2<<<148, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = 148.0 * threads * iters * 8;
      cudaEventRecord(e0); k_ffma<<<148, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms2; cudaEventElapsedTime(&ms2, e0, e1);
      if (w) printf("threads %4d: ex2 %.2f ops/clk/SM (at 1.92GHz)  ffma %.2f ops/clk/SM\n", threads,
                    ops / (ms * 1e-3) / 148 / 1.92e9, ops / (ms2 * 1e-3) / 148 / 1.92e9);
    }
  }
  return 0;
}
