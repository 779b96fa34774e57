// Issue rates of the epilogue's instruction mix on one SM-resident workload
// (microbenchmark, not product code): ops per clock per SM of
// I2F (s32 -> f32), the pack to f16x2 (F2FP), MUFU.EX2, FFMA2, FFMA, the
// magic-number int->float alternative (IADD + FADD) and HMNMX2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_rates alu_rates.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

constexpr int N = 8;

__global__ void k_i2f(float* out, int iters) {
  int a[N];
  float s = 0;
  for (int i = 0; i < N; ++i) a[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      float f;
      asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(a[i]));
      a[i] ^= __float_as_int(f);
    }
  }
  for (int i = 0; i < N; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_pack(float* out, int iters) {
  float a[N];
  uint32_t acc = 0;
  for (int i = 0; i < N; ++i) a[i] = 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      uint32_t h;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(a[i]), "f"(a[(i + 1) % N]));
      acc ^= h;
      a[i] = __int_as_float(__float_as_int(a[i]) ^ (h & 1));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc + a[0];
}

__global__ void k_ex2(float* out, int iters) {
  float a[N];
  for (int i = 0; i < N; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0;
  for (int i = 0; i < N; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(float* out, int iters) {
  float a[N];
  for (int i = 0; i < N; ++i) a[i] = 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A83126F;" : "+f"(a[i]));
  float s = 0;
  for (int i = 0; i < N; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, int iters) {
  uint64_t a[N];
  const uint64_t b = 0x3F7FFFFF3F7FFFFFull, c = 0x3A83126F3A83126Full;
  for (int i = 0; i < N; ++i) a[i] = 0x3A83126F3A83126Full + threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(b), "l"(c));
  uint64_t s = 0;
  for (int i = 0; i < N; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(s & 0xFFFF);
}

// int -> float via the 1.5 * 2^23 magic (IADD + FADD), exact for |x| < 2^22
__global__ void k_magic(float* out, int iters) {
  int a[N];
  for (int i = 0; i < N; ++i) a[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      float f;
      asm volatile("{.reg .s32 t; add.s32 t, %1, 0x4B400000; mov.b32 %0, t;}" : "=f"(f) : "r"(a[i]));
      asm volatile("sub.f32 %0, %0, 0f4B400000;" : "+f"(f));
      a[i] ^= __float_as_int(f) & 1;
    }
  }
  float s = 0;
  for (int i = 0; i < N; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_hmax2(float* out, int iters) {
  __half2 a[N];
  for (int i = 0; i < N; ++i) a[i] = __floats2half2_rn(0.001f * (threadIdx.x + i), -0.5f);
  const __half2 b = __floats2half2_rn(0.25f, 0.75f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      uint32_t x = *reinterpret_cast<uint32_t*>(&a[i]);
      asm volatile("max.f16x2 %0, %0, %1;" : "+r"(x) : "r"(*reinterpret_cast<const uint32_t*>(&b)));
      asm volatile("xor.b32 %0, %0, 0x00010001;" : "+r"(x));
      a[i] = *reinterpret_cast<__half2*>(&x);
    }
  float s = 0;
  for (int i = 0; i < N; ++i) s += __low2float(a[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K kern, int ops_per_iter_elem, float* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 512, iters = 4096;
  kern<<<148, threads>>>(out, iters);
  cudaEventRecord(e0);
  kern<<<148, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int mhz = 0;
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
  const double ops = 148.0 * threads * iters * N * ops_per_iter_elem;
  printf("%-28s %7.1f ops/clk/SM (at %d MHz)\n", name, ops / (ms * 1e-3) / 148 / (mhz * 1e3), mhz / 1000);
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 1024 * 4);
  run("I2F s32->f32 (+LOP)", k_i2f, 1, out);
  run("F2FP f32x2->f16x2 (+LOP2)", k_pack, 1, out);
  run("MUFU.EX2", k_ex2, 1, out);
  run("FFMA", k_ffma, 1, out);
  run("FFMA2 (pairs)", k_ffma2, 1, out);
  run("magic IADD+FADD (+LOP)", k_magic, 1, out);
  run("HMNMX2 (+LOP)", k_hmax2, 1, out);
  return 0;
}
