// GELU epilogue tails compared on the GPU over 2^28 points per range: the
// round-2 select tail (0.5 y) * (y >= 0 ? 2 - e : e) and the select-free
// 0.5 * fma(-|y|, e, y + |y|), both with the product's P7 / P11 exponent fits
// (gemm_tc.cu).  Counts fp16 outputs that differ from RN16(RN32(GELU_fp64)),
// the oracle's rounding point (DESIGN R2).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 gelu_tail.cu -o /tmp/gelu_tail
#include <cstdio>
#include <cuda_fp16.h>
#include <math.h>

__device__ __forceinline__ float ex2a(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float expo(float s) {
  const float c7[8] = {3.84035457e-06f, -4.82531614e-05f, 2.16719927e-04f, 8.50132710e-05f,
                       -7.01780897e-03f, 5.24765067e-02f, 4.59211707e-01f, 1.15110505e+00f};
  const float c11[12] = {1.91209187e-10f, -8.90500740e-09f, 1.86934614e-07f, -2.33101059e-06f,
                         1.90286646e-05f, -1.03522529e-04f, 3.35359509e-04f, -6.75584961e-05f,
                         -6.90312125e-03f, 5.24297878e-02f, 4.59220439e-01f, 1.15110457e+00f};
  const float sc = fminf(s, 6.5f);
  float p7 = 0.0f, p11 = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) p7 = __fmaf_rn(p7, s, c7[k]);
#pragma unroll
  for (int k = 0; k < 12; ++k) p11 = __fmaf_rn(p11, sc, c11[k]);
  return s <= 2.5f ? s * p7 : sc * p11;
}
__device__ __forceinline__ float tail_sel(float y, float e) { return (0.5f * y) * (y >= 0.0f ? 2.0f - e : e); }
__device__ __forceinline__ float tail_fma(float y, float e) {
  const float s = fabsf(y);
  return 0.5f * __fmaf_rn(-s, e, y + s);
}
// the 1/2 folded into the exponent: e' = 2^-(s P(s) + 1), GELU = relu(y) - s e'
template <int D>
__device__ __forceinline__ float gelu_relu_form(float y) {
  const float s = fabsf(y);
  const float c7[8] = {3.84035457e-06f, -4.82531614e-05f, 2.16719927e-04f, 8.50132710e-05f,
                       -7.01780897e-03f, 5.24765067e-02f, 4.59211707e-01f, 1.15110505e+00f};
  const float c6[7] = {-1.05019162e-05f, 6.65890184e-05f, 3.93992959e-04f, -7.36664515e-03f,
                       5.26866466e-02f, 4.59151894e-01f, 1.15111077e+00f};
  const float c11[12] = {1.91209187e-10f, -8.90500740e-09f, 1.86934614e-07f, -2.33101059e-06f,
                         1.90286646e-05f, -1.03522529e-04f, 3.35359509e-04f, -6.75584961e-05f,
                         -6.90312125e-03f, 5.24297878e-02f, 4.59220439e-01f, 1.15110457e+00f};
  const float sc = fminf(s, 6.5f);
  float p7 = 0.0f, p11 = 0.0f;
  if (D == 7) {
#pragma unroll
    for (int k = 0; k < 8; ++k) p7 = __fmaf_rn(p7, s, c7[k]);
  } else {
#pragma unroll
    for (int k = 0; k < 7; ++k) p7 = __fmaf_rn(p7, s, c6[k]);
  }
#pragma unroll
  for (int k = 0; k < 12; ++k) p11 = __fmaf_rn(p11, sc, c11[k]);
  const float a = s <= 2.5f ? __fmaf_rn(s, p7, 1.0f) : __fmaf_rn(sc, p11, 1.0f);
  return __fmaf_rn(-s, ex2a(-a), fmaxf(y, 0.0f));
}
struct Stat {
  unsigned long long n, flip[4], diff;
};
__global__ void k(Stat* st, float lo, float hi, unsigned long long n) {
  unsigned long long f0 = 0, f1 = 0, f2 = 0, f3 = 0, d = 0, c = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const float y = lo + (hi - lo) * (float)((double)i / (double)n);
    const double ref = 0.5 * (double)y * erfc(-(double)y / sqrt(2.0));
    const __half r16 = __float2half_rn((float)ref);
    const float e = ex2a(-expo(fabsf(y)));
    const __half a = __float2half_rn(tail_sel(y, e)), b = __float2half_rn(tail_fma(y, e));
    f0 += __half_as_ushort(a) != __half_as_ushort(r16);
    f1 += __half_as_ushort(b) != __half_as_ushort(r16);
    f2 += __half_as_ushort(__float2half_rn(gelu_relu_form<7>(y))) != __half_as_ushort(r16);
    f3 += __half_as_ushort(__float2half_rn(gelu_relu_form<6>(y))) != __half_as_ushort(r16);
    d += __half_as_ushort(a) != __half_as_ushort(b);
    ++c;
  }
  atomicAdd(&st->n, c);
  atomicAdd(&st->flip[0], f0);
  atomicAdd(&st->flip[1], f1);
  atomicAdd(&st->flip[2], f2);
  atomicAdd(&st->flip[3], f3);
  atomicAdd(&st->diff, d);
}
int main() {
  Stat* st;
  cudaMallocManaged(&st, sizeof(Stat));
  const float rl[4][2] = {{-2.0f, 2.0f}, {-7.0f, 7.0f}, {-0.5f, 0.5f}, {-12.0f, 12.0f}};
  for (auto& r : rl) {
    cudaMemset(st, 0, sizeof(Stat));
    k<<<148 * 8, 256>>>(st, r[0], r[1], 1ull << 28);
    cudaDeviceSynchronize();
    printf("gelu y in [%g,%g]: fp16 flips vs oracle: select tail %.5f%%, fma tail %.5f%%, relu form %.5f%%, relu form deg6 %.5f%%; "
           "tails differ %.5f%%\n", r[0], r[1], 100.0 * st->flip[0] / st->n, 100.0 * st->flip[1] / st->n,
           100.0 * st->flip[2] / st->n, 100.0 * st->flip[3] / st->n, 100.0 * st->diff / st->n);
  }
  return 0;
}
