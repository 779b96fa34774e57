// Accuracy of the exp / GELU evaluations used (or considered) in the
// attention softmax and the FFN1 GEMM epilogue, against fp64 references
// computed on the device (microbenchmark, not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp_accuracy exp_accuracy.cu
// For each candidate: max |err| in fp32 ulps of the reference, fraction of
// results that differ from the correctly rounded fp32 value, and (GELU) the
// fraction whose fp16 rounding differs from RN16(RN32(exact)) -- the quantity
// that decides whether the GPU's stored activations match the oracle's.
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// exp(x), x <= 0: Cody-Waite split of x*log2(e) into n + f, |f| <= 1/2,
// 2^f by a degree-6 polynomial on the FMA pipe, 2^n by exponent insertion.
__device__ __forceinline__ float exp_poly(float x) {
  const float L2E = 1.44269502f, L2E_LO = 1.925963033e-08f;
  const float t = fmaxf(x * L2E, -126.0f);
  const float n = rintf(t);
  float f = fmaf(x, L2E, -n);
  f = fmaf(x, L2E_LO, f);
  // 2^f on [-0.5, 0.5]
  float p = 1.5345805e-4f;
  p = fmaf(p, f, 1.3399931e-3f);
  p = fmaf(p, f, 9.6184891e-3f);
  p = fmaf(p, f, 5.5503286e-2f);
  p = fmaf(p, f, 2.4022646e-1f);
  p = fmaf(p, f, 6.9314718e-1f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((int)n << 23));
}

// exp(x): same split, 2^f on MUFU
__device__ __forceinline__ float exp_cw_mufu(float x) {
  const float L2E = 1.44269502f, L2E_LO = 1.925963033e-08f;
  const float t = fmaxf(x * L2E, -126.0f);
  const float n = rintf(t);
  float f = fmaf(x, L2E, -n);
  f = fmaf(x, L2E_LO, f);
  return __int_as_float(__float_as_int(ex2a(f)) + ((int)n << 23));
}

struct Stat {
  unsigned long long n, miss, flip16;
  unsigned maxulp;
};

__device__ __forceinline__ void acc(Stat& st, float got, double ref, bool f16) {
  const float r32 = (float)ref;
  const unsigned ulp = (unsigned)llabs((long long)__float_as_int(got) - (long long)__float_as_int(r32));
  st.maxulp = ulp > st.maxulp ? ulp : st.maxulp;
  st.miss += got != r32;
  st.flip16 += f16 && __half2float(__float2half_rn(got)) != __half2float(__float2half_rn(r32));
  st.n += 1;
}
__device__ void flush(Stat* g, const Stat& l) {
  atomicAdd(&g->n, l.n);
  atomicAdd(&g->miss, l.miss);
  atomicAdd(&g->flip16, l.flip16);
  atomicMax(&g->maxulp, l.maxulp);
}

// exp on x in [lo, 0]: candidate 0 = ex2.approx(x * log2e), 1 = Cody-Waite + MUFU,
// 2 = Cody-Waite + polynomial
__global__ void k_exp(Stat* st, float lo, unsigned long long n) {
  Stat l[3] = {};
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const float x = lo * (float)((double)i / (double)n);
    const double ref = exp((double)x);
    acc(l[0], ex2a(x * 1.44269502f), ref, true);
    acc(l[1], exp_cw_mufu(x), ref, true);
    acc(l[2], exp_poly(x), ref, true);
  }
  for (int c = 0; c < 3; ++c) flush(&st[c], l[c]);
}

// GELU candidates: 0 = the round-1 degree-6 2^(-s P6(s)) with MUFU;
// 1 = degree-10 fit, MUFU; 2 = degree-10 fit, polynomial 2^x
__device__ __forceinline__ float gelu_p(float y, int deg11, int poly) {
  const float s = fminf(fabsf(y), deg11 ? 6.5f : 5.6568542f);
  float p;
  if (deg11) {
    const float c[12] = {1.91209187e-10f, -8.90500740e-09f, 1.86934614e-07f, -2.33101059e-06f, 1.90286646e-05f,
                         -1.03522529e-04f, 3.35359509e-04f, -6.75584961e-05f, -6.90312125e-03f, 5.24297878e-02f,
                         4.59220439e-01f, 1.15110457e+00f};
    p = c[0];
#pragma unroll
    for (int k = 1; k < 12; ++k) p = fmaf(p, s, c[k]);
  } else {
    p = 1.7657696e-06f;
    p = fmaf(p, s, -6.0254122e-05f);
    p = fmaf(p, s, 9.2013367e-04f);
    p = fmaf(p, s, -8.4673585e-03f);
    p = fmaf(p, s, 5.3876434e-02f);
    p = fmaf(p, s, 4.5855144e-01f);
    p = fmaf(p, s, 1.1512122f);
  }
  const float a = -s * p;
  float e;
  if (poly) {
    const float n = rintf(fmaxf(a, -126.0f));
    const float f = a - n;
    float q = 1.5345805e-4f;
    q = fmaf(q, f, 1.3399931e-3f);
    q = fmaf(q, f, 9.6184891e-3f);
    q = fmaf(q, f, 5.5503286e-2f);
    q = fmaf(q, f, 2.4022646e-1f);
    q = fmaf(q, f, 6.9314718e-1f);
    q = fmaf(q, f, 1.0f);
    e = __int_as_float(__float_as_int(q) + ((int)n << 23));
  } else {
    e = ex2a(a);
  }
  return (0.5f * y) * (y >= 0.0f ? 2.0f - e : e);
}

__global__ void k_gelu(Stat* st, float lo, float hi, unsigned long long n) {
  Stat l[3] = {};
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const float y = lo + (hi - lo) * (float)((double)i / (double)n);
    const double ref = 0.5 * (double)y * erfc(-(double)y / sqrt(2.0));
    acc(l[0], gelu_p(y, 0, 0), ref, true);
    acc(l[1], gelu_p(y, 1, 0), ref, true);
    acc(l[2], gelu_p(y, 1, 1), ref, true);
  }
  for (int c = 0; c < 3; ++c) flush(&st[c], l[c]);
}

int main() {
  Stat* st;
  cudaMallocManaged(&st, 3 * sizeof(Stat));
  const char* en[3] = {"ex2.approx(x*log2e)", "Cody-Waite + ex2.approx", "Cody-Waite + poly6"};
  for (float lo : {-1.0f, -20.0f}) {
    cudaMemset(st, 0, 3 * sizeof(Stat));
    k_exp<<<148 * 8, 256>>>(st, lo, 1ull << 28);
    cudaDeviceSynchronize();
    for (int c = 0; c < 3; ++c)
      printf("exp x in [%g,0] %-26s max %u ulp, %.5f%% not correctly rounded, %.5f%% fp16 flips\n", lo, en[c],
             st[c].maxulp, 100.0 * st[c].miss / st[c].n, 100.0 * st[c].flip16 / st[c].n);
  }
  const char* gn[3] = {"deg6 + ex2.approx (r1)", "deg11 + ex2.approx", "deg11 + poly6 exp2"};
  const float rl[3][2] = {{-2.0f, 2.0f}, {-7.0f, 7.0f}, {-0.5f, 0.5f}};
  for (auto& r : rl) {
    cudaMemset(st, 0, 3 * sizeof(Stat));
    k_gelu<<<148 * 8, 256>>>(st, r[0], r[1], 1ull << 28);
    cudaDeviceSynchronize();
    for (int c = 0; c < 3; ++c)
      printf("gelu y in [%g,%g] %-24s max %u ulp, %.5f%% not correctly rounded, %.5f%% fp16 flips\n", r[0], r[1],
             gn[c], st[c].maxulp, 100.0 * st[c].miss / st[c].n, 100.0 * st[c].flip16 / st[c].n);
  }
  return 0;
}
