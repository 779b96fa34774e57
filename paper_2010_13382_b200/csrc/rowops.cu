// rowops.cu -- the HBM-bound row kernels of the encoder forward and the
// one-time weight packing kernels.
//
//   embed_ln   X = LN(E_tok[id] + P'[t]) -> fp16 (+ s8 rows)
//   add_ln     Y = LN(a + r) -> fp16 (+ s8 rows)   (post-LN residual, a6/a10)
//   quant_rows (q, s) = Q8row(x16)                                (a4/a8)
//   pooler / classifier: logits = Wc tanh(Wp x0 + bp) + bc        (a11)
//   cast_f16 / quant_weight / add_row: weight packing at load     (a0)
//
// Row kernels: one warp per row, the whole row held in registers as 16-byte
// chunks (8 elements; chunk c of lane l covers columns 8*(l + 32c)), so every
// global access is a 16-byte vector and each row is read from HBM exactly
// once; warp-shuffle reductions; two-pass mean / variance in fp32.
// Q8row (DESIGN R6-R8): scale = amax/127 (IEEE division, 1.0 for an all-zero
// row), q = clamp(RNE(x/scale), -127, 127), computed from the fp16-ROUNDED
// value so the result does not depend on where the quantizer is fused (R12).
// No fast-math anywhere in this file.
#include "ff_kernels.h"
#include "ptx.cuh"
#include "quant.cuh"

namespace ff {

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Q8row of 8 fp16-rounded values (R6-R8), packed s8x8.
__device__ __forceinline__ uint2 quant8(const float (&f)[8], float sc, float rs) {
  uint2 o;
  o.x = q8_quant4(make_float2(f[0], f[1]), make_float2(f[2], f[3]), sc, rs);
  o.y = q8_quant4(make_float2(f[4], f[5]), make_float2(f[6], f[7]), sc, rs);
  return o;
}

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __half22float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// LayerNorm of a row held as v[c][0..7] at columns 8*(lane + 32c) (< H), then
// R16 store and optional Q8row.  All lanes of the warp participate.  Packed
// fp32 pair arithmetic (FADD2 / FFMA2 / FMUL2) throughout; two-pass mean /
// variance.
template <int NCH>
__device__ __forceinline__ void ln_store(float (&v)[NCH][8], int H, int lane, const float* __restrict__ g,
                                         const float* __restrict__ b, float eps, __half* y16, int8_t* yq, float* ys) {
  float2 s2 = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int c = 0; c < NCH; ++c)
    if (8 * (lane + 32 * c) < H) {
#pragma unroll
      for (int j = 0; j < 8; j += 2) s2 = add2(s2, make_float2(v[c][j], v[c][j + 1]));
    }
  const float mean = __fdiv_rn(warp_sum(s2.x + s2.y), (float)H);
  const float2 mean2 = make_float2(mean, mean);
  float2 q2 = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int c = 0; c < NCH; ++c)
    if (8 * (lane + 32 * c) < H) {
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float2 d = sub2(make_float2(v[c][j], v[c][j + 1]), mean2);
        v[c][j] = d.x;  // v now holds the deviations
        v[c][j + 1] = d.y;
        q2 = fma2(d, d, q2);
      }
    }
  const float var = __fdiv_rn(warp_sum(q2.x + q2.y), (float)H);
  const float rstd = 1.0f / sqrtf(var + eps);
  const float2 rstd2 = make_float2(rstd, rstd);
  __half2 amax2 = __float2half2_rn(0.0f);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = 8 * (lane + 32 * c);
    if (col < H) {
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(g + col));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(g + col + 4));
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(b + col));
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(b + col + 4));
      const float2 gv[4] = {make_float2(g0.x, g0.y), make_float2(g0.z, g0.w), make_float2(g1.x, g1.y),
                            make_float2(g1.z, g1.w)};
      const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                            make_float2(b1.z, b1.w)};
      uint32_t pk[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 y = fma2(mul2(make_float2(v[c][2 * j], v[c][2 * j + 1]), rstd2), gv[j], bv[j]);
        const __half2 h = __floats2half2_rn(y.x, y.y);
        amax2 = __hmax2(amax2, __habs2(h));
        const float2 hf = __half22float2(h);  // keep the fp16-rounded values for Q8row
        v[c][2 * j] = hf.x;
        v[c][2 * j + 1] = hf.y;
        pk[j] = *reinterpret_cast<const uint32_t*>(&h);
      }
      *reinterpret_cast<uint4*>(y16 + col) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  }
  if (yq == nullptr) return;
  const float amax = warp_max(fmaxf(__low2float(amax2), __high2float(amax2)));
  const float sc = q8_scale(amax);
  const float rs = __frcp_rn(sc);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = 8 * (lane + 32 * c);
    if (col < H) {
      *reinterpret_cast<uint2*>(yq + col) = quant8(v[c], sc, rs);
    }
  }
  if (lane == 0) *ys = sc;
}

template <int NCH>
__global__ void __launch_bounds__(256) embed_ln_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ mask,
                                                      int M, int S, int H, int V, const float* __restrict__ tok,
                                                      const float* __restrict__ pos, const float* __restrict__ g,
                                                      const float* __restrict__ b, float eps, __half* x16, int ldx,
                                                      int8_t* xq, int ldq, float* xs, int* err_flag) {
  griddep_wait();
  griddep_launch();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= M) return;
  int id = ids[row];
  const int t = row % S;
  if (lane == 0) {
    const int mk = mask[row];
    int bad = 0;
    if (id < 0 || id >= V) bad |= 1;
    if (mk != 0 && mk != 1) bad |= 2;
    if (t == 0 && mk != 1) bad |= 4;
    if (bad) atomicOr(err_flag, bad);
  }
  if (id < 0 || id >= V) id = 0;  // keep the gather in bounds; the row is flagged
  const float* e = tok + (size_t)id * H;
  const float* p = pos + (size_t)t * H;
  float v[NCH][8];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = 8 * (lane + 32 * c);
    if (col < H) {
      const float4 a0 = __ldg(reinterpret_cast<const float4*>(e + col));
      const float4 a1 = __ldg(reinterpret_cast<const float4*>(e + col + 4));
      const float4 p0 = __ldg(reinterpret_cast<const float4*>(p + col));
      const float4 p1 = __ldg(reinterpret_cast<const float4*>(p + col + 4));
      v[c][0] = __fadd_rn(a0.x, p0.x);
      v[c][1] = __fadd_rn(a0.y, p0.y);
      v[c][2] = __fadd_rn(a0.z, p0.z);
      v[c][3] = __fadd_rn(a0.w, p0.w);
      v[c][4] = __fadd_rn(a1.x, p1.x);
      v[c][5] = __fadd_rn(a1.y, p1.y);
      v[c][6] = __fadd_rn(a1.z, p1.z);
      v[c][7] = __fadd_rn(a1.w, p1.w);
    }
  }
  ln_store<NCH>(v, H, lane, g, b, eps, x16 + (size_t)row * ldx, xq ? xq + (size_t)row * ldq : nullptr,
                xs ? xs + row : nullptr);
}

template <int NCH>
__global__ void __launch_bounds__(256) add_ln_kernel(const __half* __restrict__ a, int lda, const __half* __restrict__ r,
                                                    int ldr, int M, int H, const float* __restrict__ g,
                                                    const float* __restrict__ b, float eps, __half* y16, int ldy,
                                                    int8_t* yq, int ldq, float* ys) {
  griddep_wait();
  griddep_launch();
  // one row per warp (measured faster than a grid-stride loop with prefetch,
  // which lowers occupancy); all 2*NCH 16-byte loads are issued up front
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= M) return;
  uint4 ua[NCH], ur[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = 8 * (lane + 32 * c);
    if (col < H) {
      ua[c] = __ldcs(reinterpret_cast<const uint4*>(a + (size_t)row * lda + col));
      ur[c] = __ldcs(reinterpret_cast<const uint4*>(r + (size_t)row * ldr + col));
    }
  }
  float v[NCH][8];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    if (8 * (lane + 32 * c) < H) {
      float fa[8], fr[8];
      unpack8(ua[c], fa);
      unpack8(ur[c], fr);
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float2 t = add2(make_float2(fa[j], fa[j + 1]), make_float2(fr[j], fr[j + 1]));
        v[c][j] = t.x;
        v[c][j + 1] = t.y;
      }
    }
  }
  ln_store<NCH>(v, H, lane, g, b, eps, y16 + (size_t)row * ldy, yq ? yq + (size_t)row * ldq : nullptr,
                ys ? ys + row : nullptr);
}

// One warp per row, the row in registers (NCH 16-byte chunks per lane).
template <int NCH>
__global__ void __launch_bounds__(256) quant_rows_kernel(const __half* __restrict__ x, int ldx, int M, int K,
                                                        int8_t* __restrict__ q, int ldq, float* __restrict__ scale) {
  griddep_wait();
  griddep_launch();
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * 8;
  int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  uint4 un[NCH];  // next row, prefetched
  auto load_row = [&](int rw) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int col = 8 * (lane + 32 * c);
      if (rw < M && col < K) un[c] = __ldcs(reinterpret_cast<const uint4*>(x + (size_t)rw * ldx + col));
    }
  };
  load_row(row);
  for (; row < M; row += stride) {
  int8_t* qr = q + (size_t)row * ldq;
  uint4 u[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) u[c] = un[c];
  load_row(row + stride);
  __half2 amax2 = __float2half2_rn(0.0f);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    if (8 * (lane + 32 * c) < K) {
      const __half2* hw = reinterpret_cast<const __half2*>(&u[c]);
#pragma unroll
      for (int j = 0; j < 4; ++j) amax2 = __hmax2(amax2, __habs2(hw[j]));
    }
  }
  const float amax = warp_max(fmaxf(__low2float(amax2), __high2float(amax2)));
  const float sc = q8_scale(amax);
  const float rs = __frcp_rn(sc);
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int col = 8 * (lane + 32 * c);
    if (col < K) {
      float f[8];
      unpack8(u[c], f);
      *reinterpret_cast<uint2*>(qr + col) = quant8(f, sc, rs);
    }
  }
  if (lane == 0) scale[row] = sc;
  }
}

// Persistent grid for the row kernels: enough resident warps to keep ~2 rows
// per warp in flight without a long tail.
inline unsigned row_grid(int M) {
  const unsigned want = (unsigned)((M + 7) / 8);
  // measured on B200: one row per warp with many short CTAs (no cap) beats a
  // persistent grid of 2-4 CTAs/SM for these kernels; the grid-stride loop
  // keeps them correct for any grid size
  (void)kNumSMs;
  return want;
}

// Generic fallback (K not a multiple of 8 or unaligned rows): element-wise.
__global__ void __launch_bounds__(256) quant_rows_scalar_kernel(const __half* __restrict__ x, int ldx, int M, int K,
                                                               int8_t* __restrict__ q, int ldq,
                                                               float* __restrict__ scale) {
  griddep_wait();
  griddep_launch();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= M) return;
  const __half* xr = x + (size_t)row * ldx;
  float amax = 0.0f;
  for (int c = lane; c < K; c += 32) amax = fmaxf(amax, fabsf(__half2float(xr[c])));
  amax = warp_max(amax);
  const float sc = q8_scale(amax);
  for (int c = lane; c < K; c += 32) q[(size_t)row * ldq + c] = q8_quant1(__half2float(xr[c]), sc);
  if (lane == 0) scale[row] = sc;
}

// Pooler + classifier, fp32 (DESIGN R15).
// pooler_kernel: split-K partial products of the [B x H] x [H x H]^T pooler
// GEMM.  CTA = 64 sequences x 64 output features j x one K-slice (kPoolK
// columns); the x0 rows (fp16 -> fp32) and Wp rows of the slice are staged in
// smem with 16-byte loads (rows padded by 4 floats); each thread owns 4
// sequences x 4 features (float4 k-steps: 8 LDS.128 per 64 FFMA).
// part[ks][b][j] = sum over slice ks of Wp[j][k] x0_b[k].
// head_kernel: CTA per sequence, thread per feature j: pooled_j =
// tanh(sum_ks part[ks][b][j] + bp[j]) (fixed order), then logits[b][c] =
// Wc[c] . pooled + bc[c] by a fixed-order block reduction.
constexpr int kPoolT = 64, kPoolK = 128, kPoolLd = kPoolK + 4;
constexpr size_t kPoolSmem = 2 * kPoolT * kPoolLd * sizeof(float);
__global__ void __launch_bounds__(256) pooler_kernel(const __half* __restrict__ x16, int ldx, int B, int S, int H,
                                                    const float* __restrict__ Wp, int cps, float* __restrict__ part) {
  griddep_wait();
  griddep_launch();
  extern __shared__ __align__(16) float psm[];
  float* xs = psm;
  float* ws = psm + kPoolT * kPoolLd;
  const int j0 = blockIdx.x * kPoolT, b0 = blockIdx.y * kPoolT, ks = blockIdx.z;
  const int tid = threadIdx.x;
  const int tb = tid >> 4, tj = tid & 15;  // sequences b0 + tb + 16u, features j0 + tj + 16v
  float acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0f;
  const int kend = min(H, (ks + 1) * cps * kPoolK);
  for (int k0 = ks * cps * kPoolK; k0 < kend; k0 += kPoolK) {
    const int kw = min(kPoolK, kend - k0);
    // x0 slice: 64 rows x kw fp16 (8 per 16-byte load); Wp slice: 64 rows x kw fp32 (4 per load)
    for (int i = tid; i < kPoolT * (kPoolK / 8); i += 256) {
      const int bb = i / (kPoolK / 8), kk = (i - bb * (kPoolK / 8)) * 8;
      float f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (b0 + bb < B && kk < kw) {
        const __half* src = x16 + (size_t)(b0 + bb) * S * ldx + k0 + kk;
        if (kk + 8 <= kw) {
          unpack8(*reinterpret_cast<const uint4*>(src), f);
        } else {
          for (int e = 0; e < kw - kk; ++e) f[e] = __half2float(src[e]);
        }
      }
      float4* d = reinterpret_cast<float4*>(xs + bb * kPoolLd + kk);
      d[0] = make_float4(f[0], f[1], f[2], f[3]);
      d[1] = make_float4(f[4], f[5], f[6], f[7]);
    }
    for (int i = tid; i < kPoolT * (kPoolK / 4); i += 256) {
      const int jj = i / (kPoolK / 4), kk = (i - jj * (kPoolK / 4)) * 4;
      float4 v = make_float4(0, 0, 0, 0);
      if (j0 + jj < H && kk < kw) {
        const float* src = Wp + (size_t)(j0 + jj) * H + k0 + kk;
        if (kk + 4 <= kw && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
          v = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          float t[4] = {0, 0, 0, 0};
          for (int e = 0; e < min(4, kw - kk); ++e) t[e] = __ldg(src + e);
          v = make_float4(t[0], t[1], t[2], t[3]);
        }
      }
      *reinterpret_cast<float4*>(ws + jj * kPoolLd + kk) = v;
    }
    __syncthreads();
#pragma unroll 2
    for (int k = 0; k < kPoolK; k += 4) {
      float4 xv[4], wv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = *reinterpret_cast<const float4*>(xs + (tb + 16 * u) * kPoolLd + k);
#pragma unroll
      for (int v = 0; v < 4; ++v) wv[v] = *reinterpret_cast<const float4*>(ws + (tj + 16 * v) * kPoolLd + k);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          acc[u][v] = __fmaf_rn(xv[u].x, wv[v].x, acc[u][v]);
          acc[u][v] = __fmaf_rn(xv[u].y, wv[v].y, acc[u][v]);
          acc[u][v] = __fmaf_rn(xv[u].z, wv[v].z, acc[u][v]);
          acc[u][v] = __fmaf_rn(xv[u].w, wv[v].w, acc[u][v]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int b = b0 + tb + 16 * u, j = j0 + tj + 16 * v;
      if (b < B && j < H) part[((size_t)ks * B + b) * H + j] = acc[u][v];
    }
}

constexpr int kHeadThreads = 256, kHeadClasses = 8;
__global__ void __launch_bounds__(kHeadThreads) head_kernel(const float* __restrict__ part, int nks, int B, int H,
                                                           int C, const float* __restrict__ bp,
                                                           const float* __restrict__ Wc, const float* __restrict__ bc,
                                                           float* __restrict__ logits) {
  griddep_wait();
  griddep_launch();
  __shared__ float red[kHeadThreads / 32][kHeadClasses];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int c0 = 0; c0 < C; c0 += kHeadClasses) {
    float acc[kHeadClasses];
#pragma unroll
    for (int c = 0; c < kHeadClasses; ++c) acc[c] = 0.0f;
    for (int j = tid; j < H; j += kHeadThreads) {
      float z = 0.0f;
      for (int ks = 0; ks < nks; ++ks) z += part[((size_t)ks * B + b) * H + j];
      const float pj = tanhf(z + bp[j]);
#pragma unroll
      for (int c = 0; c < kHeadClasses; ++c)
        if (c0 + c < C) acc[c] = __fmaf_rn(__ldg(Wc + (size_t)(c0 + c) * H + j), pj, acc[c]);
    }
#pragma unroll
    for (int c = 0; c < kHeadClasses; ++c) {
      const float v = warp_sum(acc[c]);
      if (lane == 0) red[warp][c] = v;
    }
    __syncthreads();
    if (tid < kHeadClasses && c0 + tid < C) {
      float v = 0.0f;
      for (int w = 0; w < kHeadThreads / 32; ++w) v += red[w][tid];
      logits[(size_t)b * C + c0 + tid] = v + bc[c0 + tid];
    }
    __syncthreads();
  }
}

__global__ void cast_f16_kernel(const float* __restrict__ src, int N, int K, __half* __restrict__ dst, int ldd) {
  griddep_wait();
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)N * K) return;
  const int n = (int)(i / K), k = (int)(i - (size_t)n * K);
  dst[(size_t)n * ldd + k] = __float2half_rn(src[i]);
}

// Per-output-channel symmetric int8 weights (R7-R8).
__global__ void __launch_bounds__(256) quant_weight_kernel(const float* __restrict__ src, int N, int K,
                                                          int8_t* __restrict__ dst, int ldd, float* __restrict__ scale) {
  griddep_wait();
  const int n = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (n >= N) return;
  const float* w = src + (size_t)n * K;
  float amax = 0.0f;
  for (int k = lane; k < K; k += 32) amax = fmaxf(amax, fabsf(w[k]));
  amax = warp_max(amax);
  const float sc = q8_scale(amax);
  for (int k = lane; k < K; k += 32) dst[(size_t)n * ldd + k] = q8_quant1(w[k], sc);
  if (lane == 0) scale[n] = sc;
}

__global__ void add_row_kernel(const float* __restrict__ src, int N, int K, const float* __restrict__ row,
                               float* __restrict__ dst) {
  griddep_wait();
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)N * K) return;
  dst[i] = __fadd_rn(src[i], row[i % K]);
}

inline int chunks_for(int K) { return (K + 255) / 256; }  // 16-byte chunks per lane

}  // namespace

cudaError_t launch_embed_ln(const int32_t* ids, const int32_t* mask, int B, int S, int H, int V, const float* tok,
                            const float* pos, const float* g, const float* b, float eps, __half* x16, int ldx,
                            int8_t* xq, int ldq, float* xs, int* err_flag, cudaStream_t s) {
  const int M = B * S;
  const unsigned grid = (M + 7) / 8;
  switch (chunks_for(H)) {
    case 1: launch_ex(embed_ln_kernel<1>, dim3(grid), dim3(256), 0, s, 0,ids, mask, M, S, H, V, tok, pos, g, b, eps, x16, ldx, xq, ldq, xs, err_flag); break;
    case 2: launch_ex(embed_ln_kernel<2>, dim3(grid), dim3(256), 0, s, 0,ids, mask, M, S, H, V, tok, pos, g, b, eps, x16, ldx, xq, ldq, xs, err_flag); break;
    case 3: launch_ex(embed_ln_kernel<3>, dim3(grid), dim3(256), 0, s, 0,ids, mask, M, S, H, V, tok, pos, g, b, eps, x16, ldx, xq, ldq, xs, err_flag); break;
    default: launch_ex(embed_ln_kernel<4>, dim3(grid), dim3(256), 0, s, 0,ids, mask, M, S, H, V, tok, pos, g, b, eps, x16, ldx, xq, ldq, xs, err_flag); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_add_ln(const __half* a, int lda, const __half* r, int ldr, int M, int H, const float* g,
                          const float* b, float eps, __half* y16, int ldy, int8_t* yq, int ldq, float* ys,
                          cudaStream_t s) {
  const unsigned grid = row_grid(M);
  switch (chunks_for(H)) {
    case 1: launch_ex(add_ln_kernel<1>, dim3(grid), dim3(256), 0, s, 0,a, lda, r, ldr, M, H, g, b, eps, y16, ldy, yq, ldq, ys); break;
    case 2: launch_ex(add_ln_kernel<2>, dim3(grid), dim3(256), 0, s, 0,a, lda, r, ldr, M, H, g, b, eps, y16, ldy, yq, ldq, ys); break;
    case 3: launch_ex(add_ln_kernel<3>, dim3(grid), dim3(256), 0, s, 0,a, lda, r, ldr, M, H, g, b, eps, y16, ldy, yq, ldq, ys); break;
    default: launch_ex(add_ln_kernel<4>, dim3(grid), dim3(256), 0, s, 0,a, lda, r, ldr, M, H, g, b, eps, y16, ldy, yq, ldq, ys); break;
  }
  return cudaGetLastError();
}

// ---------------------------------------------- per-tensor u8 (DESIGN R22)
namespace {

// mm[0] = bits of max(0, max x), mm[1] = bits of max(0, -min x): both
// non-negative floats, whose bit patterns order like the values, so an
// integer atomicMax is an exact (order-independent) float max.
__global__ void __launch_bounds__(256) tensor_minmax_kernel(const __half* __restrict__ x, int ldx, int M, int K,
                                                           unsigned* __restrict__ mm) {
  griddep_wait();
  griddep_launch();
  float hi = 0.0f, nlo = 0.0f;
  const int kc = K / 8;  // 16-byte chunks per row (K % 8 == 0)
  const size_t n = (size_t)M * kc;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / kc, c = i - r * kc;
    float f[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(x + r * ldx + c * 8)), f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      hi = fmaxf(hi, f[j]);
      nlo = fmaxf(nlo, -f[j]);
    }
  }
  hi = warp_max(hi);
  nlo = warp_max(nlo);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(mm, __float_as_uint(hi));
    atomicMax(mm + 1, __float_as_uint(nlo));
  }
}

// q = clamp(RNE(x / scale) + zp, 0, 255), scale = (hi - lo) / 255 (1 for an
// all-zero tensor), zp = clamp(RNE(-lo / scale), 0, 255); IEEE divisions as
// in the definition.  qp[0] = scale, qp[1] = zp for the GEMM epilogue.
__global__ void __launch_bounds__(256) tensor_quant_kernel(const __half* __restrict__ x, int ldx, int M, int K,
                                                          const unsigned* __restrict__ mm, uint8_t* __restrict__ q,
                                                          int ldq, float* __restrict__ qp) {
  griddep_wait();
  griddep_launch();
  const float hi = __uint_as_float(mm[0]), nlo = __uint_as_float(mm[1]);
  float sc = __fdiv_rn(__fadd_rn(hi, nlo), 255.0f);  // (hi - lo) / 255 with lo = -nlo
  if (sc == 0.0f) sc = 1.0f;
  const float zp = fminf(fmaxf(rintf(__fdiv_rn(nlo, sc)), 0.0f), 255.0f);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    qp[0] = sc;
    qp[1] = zp;
  }
  // x / sc as the correctly rounded quotient without a division per element
  // (Markstein's correction with rs = RN(1 / sc), as q8_quant4 / div2_cr),
  // RNE via the 1.5 * 2^23 magic add (|x / sc| <= 255): bit-identical to
  // rintf(__fdiv_rn(x, sc)).
  const float rs = __frcp_rn(sc);
  const float2 rs2 = make_float2(rs, rs), nsc2 = make_float2(-sc, -sc);
  const float2 kMagic = make_float2(12582912.0f, 12582912.0f);
  const int kc = K / 8;
  const size_t n = (size_t)M * kc;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / kc, c = i - r * kc;
    float f[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(x + r * ldx + c * 8)), f);
    uint32_t b[8];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const float2 xv = make_float2(f[j], f[j + 1]);
      const float2 t = mul2(xv, rs2);
      const float2 qv = fma2(fma2(t, nsc2, xv), rs2, t);
      const float2 rn = sub2(add2(qv, kMagic), kMagic);  // RNE(q), exact for |q| < 2^22
      b[j] = (uint32_t)fminf(fmaxf(rn.x + zp, 0.0f), 255.0f);
      b[j + 1] = (uint32_t)fminf(fmaxf(rn.y + zp, 0.0f), 255.0f);
    }
    *reinterpret_cast<uint2*>(q + r * ldq + c * 8) =
        make_uint2(b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24), b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24));
  }
}

// colsum[n] = sum_k wq[n][k] (the zero-point correction of u8 x s8 GEMMs).
__global__ void __launch_bounds__(256) weight_colsum_kernel(const int8_t* __restrict__ wq, int ldw, int N, int K,
                                                           int* __restrict__ colsum) {
  griddep_wait();
  const int n = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (n >= N) return;
  int acc = 0;
  for (int k = lane; k < K; k += 32) acc += wq[(size_t)n * ldw + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) colsum[n] = acc;
}

}  // namespace

cudaError_t launch_quant_tensor(const __half* x, int ldx, int M, int K, unsigned* mm, uint8_t* q, int ldq, float* qp,
                                cudaStream_t s) {
  if (K % 8 || ldx % 8 || ldq % 8) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(mm, 0, 2 * sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  launch_ex(tensor_minmax_kernel, dim3(2 * kNumSMs), dim3(256), 0, s, 0, x, ldx, M, K, mm);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  launch_ex(tensor_quant_kernel, dim3(4 * kNumSMs), dim3(256), 0, s, 0, x, ldx, M, K, (const unsigned*)mm, q, ldq, qp);
  return cudaGetLastError();
}

cudaError_t launch_weight_colsum(const int8_t* wq, int ldw, int N, int K, int* colsum, cudaStream_t s) {
  launch_ex(weight_colsum_kernel, dim3((N + 7) / 8), dim3(256), 0, s, 0, wq, ldw, N, K, colsum);
  return cudaGetLastError();
}

cudaError_t launch_quant_rows(const __half* x, int ldx, int M, int K, int8_t* q, int ldq, float* scale,
                              cudaStream_t s) {
  unsigned grid = (M + 7) / 8;
  const bool vec = (K % 8 == 0) && (ldx % 8 == 0) && (ldq % 8 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(q) & 7) == 0) && K <= 4096;
  if (!vec) {
    launch_ex(quant_rows_scalar_kernel, dim3(grid), dim3(256), 0, s, 0,x, ldx, M, K, q, ldq, scale);
    return cudaGetLastError();
  }
  grid = row_grid(M);
  const int n = chunks_for(K);
  if (n <= 1) launch_ex(quant_rows_kernel<1>, dim3(grid), dim3(256), 0, s, 0,x, ldx, M, K, q, ldq, scale);
  else if (n <= 2) launch_ex(quant_rows_kernel<2>, dim3(grid), dim3(256), 0, s, 0,x, ldx, M, K, q, ldq, scale);
  else if (n <= 4) launch_ex(quant_rows_kernel<4>, dim3(grid), dim3(256), 0, s, 0,x, ldx, M, K, q, ldq, scale);
  else if (n <= 6) launch_ex(quant_rows_kernel<6>, dim3(grid), dim3(256), 0, s, 0,x, ldx, M, K, q, ldq, scale);
  else if (n <= 8) launch_ex(quant_rows_kernel<8>, dim3(grid), dim3(256), 0, s, 0,x, ldx, M, K, q, ldq, scale);
  else if (n <= 12) launch_ex(quant_rows_kernel<12>, dim3(grid), dim3(256), 0, s, 0,x, ldx, M, K, q, ldq, scale);
  else launch_ex(quant_rows_kernel<16>, dim3(grid), dim3(256), 0, s, 0,x, ldx, M, K, q, ldq, scale);
  return cudaGetLastError();
}

cudaError_t launch_head(const __half* x16, int ldx, int B, int S, int H, int C, const float* Wp, const float* bp,
                        const float* Wc, const float* bc, float* part, float* logits, cudaStream_t s,
                        int seq_stride) {
  // seq_stride: rows between consecutive sequences' first tokens (S; 1 when
  // they are compact, FF_OPT_CLS_LAST_LAYER); the split-K geometry depends on
  // S only, so both layouts sum in the same order
  // nks K slices of cps kPoolK-column chunks; part holds nks x B x H floats,
  // within the caller's B x S x H scratch (nks <= S)
  const int chunks = (H + kPoolK - 1) / kPoolK;
  const int cps = (chunks + min(chunks, S) - 1) / min(chunks, S);
  const int nks = (chunks + cps - 1) / cps;
  dim3 grid((H + kPoolT - 1) / kPoolT, (B + kPoolT - 1) / kPoolT, nks);
  launch_ex(pooler_kernel, grid, dim3(256), kPoolSmem, s, 0, x16, ldx, B, seq_stride < 0 ? S : seq_stride, H, Wp, cps,
            part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  launch_ex(head_kernel, dim3(B), dim3(kHeadThreads), 0, s, 0, (const float*)part, nks, B, H, C, bp, Wc, bc, logits);
  return cudaGetLastError();
}

cudaError_t prepare_row_kernels() {
  return cudaFuncSetAttribute(pooler_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPoolSmem);
}

cudaError_t launch_cast_f16(const float* src, int N, int K, __half* dst, int ldd, cudaStream_t s) {
  const size_t n = (size_t)N * K;
  launch_ex(cast_f16_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, 0,src, N, K, dst, ldd);
  return cudaGetLastError();
}

cudaError_t launch_quant_weight(const float* src, int N, int K, int8_t* dst, int ldd, float* scale, cudaStream_t s) {
  launch_ex(quant_weight_kernel, dim3((N + 7) / 8), dim3(256), 0, s, 0,src, N, K, dst, ldd, scale);
  return cudaGetLastError();
}

cudaError_t launch_add_row(const float* src, int N, int K, const float* row, float* dst, cudaStream_t s) {
  const size_t n = (size_t)N * K;
  launch_ex(add_row_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, 0,src, N, K, row, dst);
  return cudaGetLastError();
}

}  // namespace ff
