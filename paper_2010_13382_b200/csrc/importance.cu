// importance.cu -- structured-pruning importance scores on the GPU (SURVEY
// 8(f) NEXT-3): "we add a mask variable to each attention head
// for the gradient computation of the heads.  Next, we run forward and
// backward passes of the model on the entire validation data set, then the
// absolute values of the gradients are accumulated."
//
// One ff_score_batch call = the fp32 encoder forward of the UNPRUNED model
// with every activation the backward needs kept in the workspace, the
// classifier's mean cross-entropy (DESIGN R24), then the reverse pass layer by
// layer down to layer 0's input, reducing on the way
//   dL/dxi[l,h] = sum_{t, j in head h} ctx[t,j] * dctx[t,j]     (head mask, R23)
//   dL/dnu[l,f] = sum_t act[t,f] * dact[t,f]                     (FFN-unit mask)
// and adding their absolute values to fp64 score arrays.
// Masks are 1, so the forward is the plain encoder (post-LN BERT, R1-R4, R10,
// R16); the masked keys get probability 0 and padded rows carry no gradient.
//
// fp32 throughout; every contraction runs on a generic strided batched SIMT
// SGEMM (128x128 tiles / 8x8 per thread for the linears, 64x64 / 4x4 for the
// per-head attention products) -- this pass runs once over a validation set,
// offline; it is not the serving hot path.  Parity against
// the fp64 oracle (oracle/importance.py) in tests/test_gpu_importance.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fastformers.h"
#include "ff_kernels.h"

namespace {

thread_local std::string g_serr;

// Makes the scorer's device current for one API call, restoring the caller's.
struct SDev {
  int prev = -1;
  explicit SDev(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~SDev() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
ff_status sfail(ff_status s, const std::string& msg) {
  g_serr = msg;
  return s;
}
#define SC_CK(x)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) return sfail(FF_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------------ SGEMM
// C[z](m, n) (+)= alpha * sum_k A[z](m, k) * B[z](k, n) (+ bias[n]) with
// z = b * nh + h and arbitrary element strides: every transpose of the
// forward / backward contractions is a stride choice.
struct SG {
  const float* A;
  long long sAb, sAh, sAm, sAk;
  const float* B;
  long long sBb, sBh, sBk, sBn;
  float* C;
  long long sCb, sCh, sCm;  // n stride 1
  const float* bias;
  int M, N, K, nh;
  float alpha;
  int accumulate;
};

constexpr int TBM = 64, TBN = 64, TBK = 16;

__global__ void __launch_bounds__(256) sgemm_kernel(SG g) {
  __shared__ float As[TBK][TBM + 4];
  __shared__ float Bs[TBK][TBN + 4];
  const int z = blockIdx.z, zb = z / g.nh, zh = z - zb * g.nh;
  const float* A = g.A + zb * g.sAb + zh * g.sAh;
  const float* B = g.B + zb * g.sBb + zh * g.sBh;
  float* C = g.C + zb * g.sCb + zh * g.sCh;
  const int m0 = blockIdx.y * TBM, n0 = blockIdx.x * TBN;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const bool a_kfast = g.sAk == 1, b_nfast = g.sBn == 1;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += TBK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;
      const int mm = a_kfast ? e / TBK : e % TBM, kk = a_kfast ? e % TBK : e / TBM;
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < g.M && k < g.K) ? A[m * g.sAm + k * g.sAk] : 0.0f;
      const int nn = b_nfast ? e % TBN : e / TBK, kb = b_nfast ? e / TBN : e % TBK;
      const int n = n0 + nn, k2 = k0 + kb;
      Bs[kb][nn] = (n < g.N && k2 < g.K) ? B[k2 * g.sBk + n * g.sBn] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TBK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty + 16 * i];
        b[i] = Bs[kk][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= g.N) continue;
      float v = g.alpha * acc[i][j];
      if (g.bias) v += g.bias[n];
      float* c = C + m * g.sCm + n;
      *c = g.accumulate ? *c + v : v;
    }
  }
}

// Large-tile variant for the encoder linears: 128x128 tiles, 8x8 outputs per
// thread (rows ty*4 + {0..3} and 64 + ty*4 + {0..3}, same for columns, so the
// fragment reads are conflict-free LDS.128), k-tiles of 8 double-buffered in
// smem with the next tile's global loads held in registers during the FMAs.
constexpr int LBM = 128, LBN = 128, LBK = 8;

__global__ void __launch_bounds__(256, 2) sgemm128_kernel(SG g) {
  __shared__ __align__(16) float As[2][LBK][LBM + 4];  // +4: conflict-free transposing stores
  __shared__ __align__(16) float Bs[2][LBK][LBN + 4];
  const int z = blockIdx.z, zb = z / g.nh, zh = z - zb * g.nh;
  const float* A = g.A + zb * g.sAb + zh * g.sAh;
  const float* B = g.B + zb * g.sBb + zh * g.sBh;
  float* C = g.C + zb * g.sCb + zh * g.sCh;
  const int m0 = blockIdx.y * LBM, n0 = blockIdx.x * LBN;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const bool a_kfast = g.sAk == 1, b_nfast = g.sBn == 1;
  float ra[4], rb[4];
  auto gload = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;
      const int mm = a_kfast ? e / LBK : e % LBM, kk = a_kfast ? e % LBK : e / LBM;
      const int m = m0 + mm, k = k0 + kk;
      ra[i] = (m < g.M && k < g.K) ? A[m * g.sAm + k * g.sAk] : 0.0f;
      const int nn = b_nfast ? e % LBN : e / LBK, kb = b_nfast ? e / LBN : e % LBK;
      const int n = n0 + nn, k2 = k0 + kb;
      rb[i] = (n < g.N && k2 < g.K) ? B[k2 * g.sBk + n * g.sBn] : 0.0f;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;
      const int mm = a_kfast ? e / LBK : e % LBM, kk = a_kfast ? e % LBK : e / LBM;
      As[buf][kk][mm] = ra[i];
      const int nn = b_nfast ? e % LBN : e / LBK, kb = b_nfast ? e / LBN : e % LBK;
      Bs[buf][kb][nn] = rb[i];
    }
  };
  float acc[8][8] = {};
  gload(0);
  sstore(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < g.K; k0 += LBK) {
    const bool more = k0 + LBK < g.K;
    if (more) gload(k0 + LBK);
#pragma unroll
    for (int kk = 0; kk < LBK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) {
      sstore(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n >= g.N) continue;
      float v = g.alpha * acc[i][j];
      if (g.bias) v += g.bias[n];
      float* c = C + m * g.sCm + n;
      *c = g.accumulate ? *c + v : v;
    }
  }
}

// Split-K for the narrow linears (N = H = 768 at M = 4096 gives 192 big tiles,
// 0.65 of a wave at 2 CTAs per SM): the K range is cut into `splits` equal
// parts computed by one launch (grid z = split, partials to the scorer's own
// split-K scratch `sk`) and summed in a fixed order by splitk_reduce_kernel
// (+ bias, + C if accumulating).
struct SplitKScratch {
  float* ws = nullptr;  // the calling scorer's workspace slice (stream-ordered use)
  size_t cap = 0;       // floats
};

__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits, int M, int N,
                                     const float* __restrict__ bias, float* C, long long sCm, int accumulate) {
  const size_t n_el = (size_t)M * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_el; i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / N), n = (int)(i - (size_t)m * N);
    float v = 0.0f;
    for (int s = 0; s < splits; ++s) v += part[(size_t)s * n_el + i];
    if (bias) v += bias[n];
    float* c = C + m * sCm + n;
    *c = accumulate ? *c + v : v;
  }
}

cudaError_t sgemm(const SG& g, int nz, cudaStream_t s, const SplitKScratch& sk = SplitKScratch()) {
  const long long big_tiles = (long long)((g.N + LBN - 1) / LBN) * ((g.M + LBM - 1) / LBM) * nz;
  if (nz == 1 && g.M >= 256 && g.N >= 256 && big_tiles < 2 * ff::kNumSMs && sk.ws != nullptr) {
    int splits = 0;
    for (int cand = 4; cand >= 2; --cand)
      if (g.K % cand == 0 && g.K / cand >= 256 && (size_t)cand * g.M * g.N <= sk.cap) {
        splits = cand;
        break;
      }
    if (splits > 0) {
      const int klen = g.K / splits;
      SG gs = g;
      gs.K = klen;
      gs.nh = 1;
      gs.sAb = (long long)klen * g.sAk;
      gs.sBb = (long long)klen * g.sBk;
      gs.C = sk.ws;
      gs.sCb = (long long)g.M * g.N;
      gs.sCm = g.N;
      gs.bias = nullptr;
      gs.accumulate = 0;
      dim3 grid((g.N + LBN - 1) / LBN, (g.M + LBM - 1) / LBM, splits);
      sgemm128_kernel<<<grid, 256, 0, s>>>(gs);
      splitk_reduce_kernel<<<4 * ff::kNumSMs, 256, 0, s>>>(sk.ws, splits, g.M, g.N, g.bias, g.C, g.sCm,
                                                            g.accumulate);
      return cudaGetLastError();
    }
  }
  if (g.M >= 256 && g.N >= 256) {
    dim3 grid((g.N + LBN - 1) / LBN, (g.M + LBM - 1) / LBM, nz);
    sgemm128_kernel<<<grid, 256, 0, s>>>(g);
  } else {
    dim3 grid((g.N + TBN - 1) / TBN, (g.M + TBM - 1) / TBM, nz);
    sgemm_kernel<<<grid, 256, 0, s>>>(g);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------- row reductions
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.0f;
  for (int i = 0; i < nw; ++i) t += red[i];  // fixed order: deterministic
  return t;
}
__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = -INFINITY;
  for (int i = 0; i < nw; ++i) t = fmaxf(t, red[i]);
  return t;
}

// y = LN(x) per row (biased variance, eps inside the sqrt); keeps xh and rstd.
// x = a + b (b may be null); embedding variant gathers a row of the tables.
__device__ void ln_row(const float* x, int H, const float* gam, const float* bet, float eps, float* y, float* xh,
                       float* rstd_out, float* red) {
  float s = 0.0f;
  for (int j = threadIdx.x; j < H; j += blockDim.x) s += x[j];
  const float mu = block_sum(s, red) / H;
  float v = 0.0f;
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    const float t = x[j] - mu;
    v += t * t;
  }
  const float rs = rsqrtf(block_sum(v, red) / H + eps);
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    const float h = (x[j] - mu) * rs;
    if (xh) xh[j] = h;
    y[j] = h * gam[j] + bet[j];
  }
  if (threadIdx.x == 0 && rstd_out) *rstd_out = rs;
}

// Input errors (sticky flag, ff_scorer_check): bit 0 token id outside [0, V)
// (read as id 0), bit 1 mask[b][0] != 1 or a mask value not 0/1, bit 2 label
// outside [0, C) (read as 0) -- no out-of-bounds access on bad input.
__global__ void embed_ln_f32_kernel(const int* ids, const int* mask, int S, int H, int V, const float* tok,
                                    const float* pos, const float* type0, const float* g, const float* b, float eps,
                                    float* X, int* err) {
  extern __shared__ float sm[];
  float* row = sm;
  float* red = sm + H;
  const int r = blockIdx.x, si = r % S;
  int id = ids[r];
  if (threadIdx.x == 0) {
    const int mk = mask[r];
    if (id < 0 || id >= V) atomicOr(err, 1);
    if ((mk != 0 && mk != 1) || (si == 0 && mk != 1)) atomicOr(err, 2);
  }
  if (id < 0 || id >= V) id = 0;
  const float* t = tok + (size_t)id * H;
  const float* p = pos + (size_t)si * H;
  for (int j = threadIdx.x; j < H; j += blockDim.x) row[j] = t[j] + p[j] + type0[j];
  ln_row(row, H, g, b, eps, X + (size_t)r * H, nullptr, nullptr, red);
}

__global__ void add_ln_f32_kernel(const float* a, const float* r, int H, const float* g, const float* b, float eps,
                                  float* y, float* xh, float* rstd) {
  extern __shared__ float sm[];
  float* row = sm;
  float* red = sm + H;
  const size_t o = (size_t)blockIdx.x * H;
  for (int j = threadIdx.x; j < H; j += blockDim.x) row[j] = a[o + j] + r[o + j];
  ln_row(row, H, g, b, eps, y + o, xh + o, rstd + blockIdx.x, red);
}

// dX = rstd * (dxh - mean(dxh) - xh * mean(dxh * xh)), dxh = dY * gamma.
__global__ void ln_bwd_kernel(const float* dy, const float* g, const float* xh, const float* rstd, int H, float* dx) {
  extern __shared__ float red[];
  const size_t o = (size_t)blockIdx.x * H;
  float s1 = 0.0f, s2 = 0.0f;
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    const float d = dy[o + j] * g[j];
    s1 += d;
    s2 += d * xh[o + j];
  }
  const float m1 = block_sum(s1, red) / H;
  const float m2 = block_sum(s2, red) / H;
  const float rs = rstd[blockIdx.x];
  for (int j = threadIdx.x; j < H; j += blockDim.x) dx[o + j] = rs * (dy[o + j] * g[j] - m1 - xh[o + j] * m2);
}

// P = softmax(scale * S) over the valid keys of the row (masked keys: 0).
// Rows: z = (b, h), i; S buffer [B, A, S, S].
__global__ void softmax_fwd_kernel(float* P, const int* mask, int S, int A, float scale) {
  __shared__ float red[32];
  const size_t row = blockIdx.x;
  const int b = (int)(row / ((size_t)A * S));
  float* p = P + row * S;
  const int* mk = mask + (size_t)b * S;
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < S; j += blockDim.x)
    if (mk[j]) mx = fmaxf(mx, p[j] * scale);
  mx = block_max(mx, red);
  float sum = 0.0f;
  for (int j = threadIdx.x; j < S; j += blockDim.x) {
    const float e = mk[j] ? expf(p[j] * scale - mx) : 0.0f;
    p[j] = e;
    sum += e;
  }
  const float inv = 1.0f / block_sum(sum, red);
  for (int j = threadIdx.x; j < S; j += blockDim.x) p[j] *= inv;
}

// dS = scale * P * (dP - sum_j P dP), in place on dP.
__global__ void softmax_bwd_kernel(const float* P, float* dP, int S, float scale) {
  __shared__ float red[32];
  const size_t o = (size_t)blockIdx.x * S;
  float s = 0.0f;
  for (int j = threadIdx.x; j < S; j += blockDim.x) s += P[o + j] * dP[o + j];
  const float t = block_sum(s, red);
  for (int j = threadIdx.x; j < S; j += blockDim.x) dP[o + j] = scale * P[o + j] * (dP[o + j] - t);
}

__device__ __forceinline__ float act_f(float u, int act) {
  if (act == ff::ACT_GELU) return 0.5f * u * (1.0f + erff(u * 0.70710678118654752f));
  if (act == ff::ACT_RELU) return fmaxf(u, 0.0f);
  const float c = 0.7978845608028654f;
  return 0.5f * u * (1.0f + tanhf(c * (u + 0.044715f * u * u * u)));
}
__device__ __forceinline__ float act_g(float u, int act) {
  if (act == ff::ACT_GELU)
    return 0.5f * (1.0f + erff(u * 0.70710678118654752f)) + u * expf(-0.5f * u * u) * 0.3989422804014327f;
  if (act == ff::ACT_RELU) return u > 0.0f ? 1.0f : 0.0f;
  const float c = 0.7978845608028654f;
  const float t = tanhf(c * (u + 0.044715f * u * u * u));
  return 0.5f * (1.0f + t) + 0.5f * u * (1.0f - t * t) * c * (1.0f + 3.0f * 0.044715f * u * u);
}
__global__ void act_fwd_kernel(const float* U, float* Aout, size_t n, int act) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    Aout[i] = act_f(U[i], act);
}
__global__ void act_bwd_kernel(const float* U, float* dA, size_t n, int act) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dA[i] *= act_g(U[i], act);
}

// Classifier head of sequence b, forward and backward (block per sequence):
// pool = tanh(Wp x0 + bp), logits = Wc pool + bc, loss_b = CE; writes
// dX[b*S + 0, :] = Wp^T ((Wc^T dlogits) * (1 - pool^2)), dlogits = (p - y) / B.
// Classifier head forward and backward in three launches (the single-CTA-per-
// sequence version was latency-bound: 2 x H^2 MACs on 32 SMs):
// head_pool_kernel (grid B x H/8, warp per pooler output): pool = tanh(Wp x0 + bp);
// head_loss_kernel (CTA per sequence): logits = Wc pool + bc, loss_b = CE,
//   dlogits = (p - y) / B, dpre = (Wc^T dlogits) * (1 - pool^2);
// head_dx_kernel (grid B x H/256, thread per feature): dX[b*S + 0, j] = sum_o Wp[o][j] dpre[o].
__global__ void head_pool_kernel(const float* X, int S, int H, const float* Wp, const float* bp, float* pool) {
  const int b = blockIdx.x, w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int o = blockIdx.y * 8 + w;
  if (o >= H) return;
  const float* x0 = X + (size_t)b * S * H;
  float s = 0.0f;
  for (int j = l; j < H; j += 32) s += Wp[(size_t)o * H + j] * x0[j];
#pragma unroll
  for (int q = 16; q > 0; q >>= 1) s += __shfl_xor_sync(0xffffffffu, s, q);
  if (l == 0) pool[(size_t)b * H + o] = tanhf(s + bp[o]);
}

__global__ void head_loss_kernel(const float* pool_all, int H, int C, int B, const float* Wc, const float* bc,
                                 const int* labels, float* loss_b, float* logits_out, float* dpre_all, int* err) {
  __shared__ float lg[64];
  const int b = blockIdx.x;
  const float* pool = pool_all + (size_t)b * H;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = w; c < C; c += nw) {
    float s = 0.0f;
    for (int j = l; j < H; j += 32) s += Wc[(size_t)c * H + j] * pool[j];
#pragma unroll
    for (int q = 16; q > 0; q >>= 1) s += __shfl_xor_sync(0xffffffffu, s, q);
    if (l == 0) lg[c] = s + bc[c];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = -INFINITY;
    for (int c = 0; c < C; ++c) mx = fmaxf(mx, lg[c]);
    float se = 0.0f;
    for (int c = 0; c < C; ++c) se += expf(lg[c] - mx);
    const float lse = logf(se);
    int lab = labels[b];
    if (lab < 0 || lab >= C) {
      atomicOr(err, 4);
      lab = 0;
    }
    loss_b[b] = lse - (lg[lab] - mx);
    for (int c = 0; c < C; ++c) {
      if (logits_out) logits_out[(size_t)b * C + c] = lg[c];
      lg[c] = (expf(lg[c] - mx - lse) - (c == lab ? 1.0f : 0.0f)) / (float)B;  // dlogits
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    float s = 0.0f;
    for (int c = 0; c < C; ++c) s += Wc[(size_t)c * H + j] * lg[c];
    dpre_all[(size_t)b * H + j] = s * (1.0f - pool[j] * pool[j]);
  }
}

__global__ void head_dx_kernel(const float* dpre_all, int S, int H, const float* Wp, float* dX) {
  const int b = blockIdx.x, j = blockIdx.y * blockDim.x + threadIdx.x;
  if (j >= H) return;
  const float* dpre = dpre_all + (size_t)b * H;
  float s = 0.0f;
  for (int o = 0; o < H; ++o) s += Wp[(size_t)o * H + j] * dpre[o];
  dX[(size_t)b * S * H + j] = s;
}

__global__ void loss_mean_kernel(const float* loss_b, int B, float* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    float s = 0.0f;
    for (int b = 0; b < B; ++b) s += loss_b[b];
    *out = s / B;
  }
}

// colg[chunk][c] = sum over the rows of chunk `blockIdx.y` (of kRowChunks) of
// X[r, c] * dX[r, c] (fixed order): block = 32 columns x 8 row groups.
constexpr int kRowChunks = 16;
__global__ void colprod_kernel(const float* X, const float* dX, int M, int ncols, int ld, float* colg) {
  __shared__ float part[8][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31), rg = threadIdx.x >> 5;
  const int rows = (M + kRowChunks - 1) / kRowChunks;
  const int r0 = blockIdx.y * rows, r1 = min(M, r0 + rows);
  float s = 0.0f;
  if (c < ncols)
    for (int r = r0 + rg; r < r1; r += 8) s += X[(size_t)r * ld + c] * dX[(size_t)r * ld + c];
  part[rg][threadIdx.x & 31] = s;
  __syncthreads();
  if (rg == 0 && c < ncols) {
    float t = 0.0f;
    for (int i = 0; i < 8; ++i) t += part[i][threadIdx.x & 31];
    colg[(size_t)blockIdx.y * ncols + c] = t;
  }
}
// scores[u] += | sum_{c in [u*group, +group)} sum_chunks colg[chunk][c] |
// One warp per unit: strided fp64 partial sums, then a fixed xor-shuffle tree
// (deterministic).
__global__ void group_abs_add_kernel(const float* colg, int ncols, int units, int group, double* scores) {
  const int u = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (u >= units) return;
  double s = 0.0;
  const int n = kRowChunks * group;
  for (int i = lane; i < n; i += 32) {
    const int ch = i / group, j = i - ch * group;
    s += (double)colg[(size_t)ch * ncols + (size_t)u * group + j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) scores[u] += fabs(s);
}

__global__ void copy_kernel(const float* a, float* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

size_t al(size_t x) { return (x + 255) / 256 * 256; }

const char* kSLayer[16] = {
    "attention.self.query.weight", "attention.self.key.weight", "attention.self.value.weight",
    "attention.self.query.bias", "attention.self.key.bias", "attention.self.value.bias",
    "attention.output.dense.weight", "attention.output.dense.bias", "attention.output.LayerNorm.weight",
    "attention.output.LayerNorm.bias", "intermediate.dense.weight", "intermediate.dense.bias",
    "output.dense.weight", "output.dense.bias", "output.LayerNorm.weight", "output.LayerNorm.bias"};

struct XSplit {
  size_t h = 0, l = 0;  // fp16 hi / lo offsets in the weight arena
  size_t s = 0;         // per-row scales (fp32, 2^e)
  int ld = 0;           // row pitch (halves, multiple of 8)
};
inline int round8(int x) { return (x + 7) & ~7; }

struct SLayer {
  int A, D, F;
  size_t wqkv, bqkv, wo, bo, g1, b1, w1, bi1, w2, bi2, g2, b2;  // weight offsets
  size_t X, QKV, P, Cx, Y1, XH1, R1, U, Act, XH2, R2;          // saved activations (workspace)
  // Row-scaled fp16 hi / lo splits of the linears' weights for the tcgen05
  // path (weight arena, written by ff_scorer_finalize): W [N x K] as
  // [N x round8(K)] (forward B operand) and W^T as [K x round8(N)]
  // (input-gradient B operand).
  XSplit qkv, qkvT, o, oT, f1, f1T, f2, f2T;
  uint32_t loaded = 0;
};

}  // namespace

struct ff_scorer {
  ff_config cfg;
  std::vector<int> heads, ffn;
  int device = 0, state = 0;
  std::vector<SLayer> L;
  size_t tok, pos, type0, eg, eb, pw, pb, cw, cb;
  uint32_t top_loaded = 0;
  size_t wbytes = 0, wsbytes = 0;
  size_t Xout, dX, dZ, dY1, dAm, dC, dP, dQKV, colg, lossb, errf, skws, headws, ids, mask, labels;
  size_t xh = 0, xl = 0, xs = 0;  // fp16 hi / lo split of the current linear's input [M x round8(Kmax)], row scales
  size_t tws = 0, tws_floats = 0;  // finalize-time transpose scratch (the split-K region, free then)
  int Dmax = 0, Fmax = 0, Amax = 0, Kmax = 0;
  int tc_linears = 1;     // FF_SCORER_OPT_TC_LINEARS
  uint8_t* dW = nullptr;
  uint8_t* dWS = nullptr;
  float* w(size_t o) const { return reinterpret_cast<float*>(dW + o); }
  float* ws(size_t o) const { return reinterpret_cast<float*>(dWS + o); }
  __half* hw(size_t o) const { return reinterpret_cast<__half*>(dW + o); }
  __half* hws(size_t o) const { return reinterpret_cast<__half*>(dWS + o); }
};

namespace {

void plan_scorer(ff_scorer* m) {
  const ff_config& c = m->cfg;
  const size_t H = c.hidden, M = c.max_tokens, Sm = c.max_positions;
  size_t o = 0;
  auto take = [&](size_t floats) {
    const size_t r = o;
    o = al(o + floats * 4);
    return r;
  };
  m->tok = take((size_t)c.vocab_size * H);
  m->pos = take(Sm * H);
  m->type0 = take(H);
  m->eg = take(H);
  m->eb = take(H);
  m->L.resize(c.num_layers);
  for (int l = 0; l < c.num_layers; ++l) {
    SLayer& P = m->L[l];
    P.A = m->heads[l];
    P.D = P.A * c.head_dim;
    P.F = m->ffn[l];
    m->Dmax = std::max(m->Dmax, P.D);
    m->Fmax = std::max(m->Fmax, P.F);
    m->Amax = std::max(m->Amax, P.A);
    P.wqkv = take((size_t)3 * P.D * H);
    P.bqkv = take((size_t)3 * P.D);
    P.wo = take(H * P.D);
    P.bo = take(H);
    P.g1 = take(H);
    P.b1 = take(H);
    P.w1 = take((size_t)P.F * H);
    P.bi1 = take(P.F);
    P.w2 = take(H * P.F);
    P.bi2 = take(H);
    P.g2 = take(H);
    P.b2 = take(H);
  }
  // fp16 hi / lo splits of the four linears' weights and of their transposes
  auto split = [&](XSplit& x, size_t rows, int cols) {
    x.ld = round8(cols);
    x.h = take((rows * x.ld + 1) / 2);
    x.l = take((rows * x.ld + 1) / 2);
    x.s = take(rows);
  };
  for (int l = 0; l < c.num_layers; ++l) {
    SLayer& P = m->L[l];
    split(P.qkv, 3 * (size_t)P.D, (int)H);
    split(P.qkvT, H, 3 * P.D);
    split(P.o, H, P.D);
    split(P.oT, P.D, (int)H);
    split(P.f1, P.F, (int)H);
    split(P.f1T, H, P.F);
    split(P.f2, H, P.F);
    split(P.f2T, P.F, (int)H);
    m->Kmax = std::max(m->Kmax, std::max((int)H, std::max(3 * P.D, P.F)));
  }
  m->pw = take(H * H);
  m->pb = take(H);
  m->cw = take((size_t)c.num_classes * H);
  m->cb = take(c.num_classes);
  m->wbytes = o;

  o = 0;
  for (int l = 0; l < c.num_layers; ++l) {
    SLayer& P = m->L[l];
    P.X = take(M * H);
    P.QKV = take(M * 3 * P.D);
    P.P = take(M * P.A * Sm);  // [B, A, S, S] = M * A * S floats
    P.Cx = take(M * P.D);
    P.Y1 = take(M * H);
    P.XH1 = take(M * H);
    P.R1 = take(M);
    P.U = take(M * P.F);
    P.Act = take(M * P.F);
    P.XH2 = take(M * H);
    P.R2 = take(M);
  }
  m->Xout = take(M * H);
  m->dX = take(M * H);
  m->dZ = take(M * H);
  m->dY1 = take(M * H);
  m->dAm = take(M * m->Fmax);
  m->dC = take(M * m->Dmax);
  m->dP = take(M * m->Amax * Sm);
  m->dQKV = take(M * 3 * m->Dmax);
  m->colg = take((size_t)kRowChunks * std::max(m->Fmax, m->Dmax));
  {  // split-K partials; at finalize, the fp32 transpose of one weight (the largest fits)
    size_t wmax = 0;
    for (const SLayer& P : m->L) wmax = std::max(wmax, std::max((size_t)3 * P.D * H, (size_t)P.F * H));
    m->tws_floats = std::max(4 * M * std::max((size_t)H, (size_t)m->Dmax), wmax);
    m->skws = m->tws = take(m->tws_floats);
  }
  m->headws = take(2 * M * H);                                     // head: pool, dpre [B x H] each
  m->lossb = take(M);
  m->xh = take((M * round8(m->Kmax) + 1) / 2);
  m->xl = take((M * round8(m->Kmax) + 1) / 2);
  m->xs = take(M);
  m->errf = take(64);
  m->wsbytes = o;
}

SG lin(const float* X, int M, int K, const float* W, const float* bias, float* Y, int N) {
  // Y[M, N] = X[M, K] W[N, K]^T + bias
  SG g{};
  g.A = X; g.sAm = K; g.sAk = 1;
  g.B = W; g.sBk = 1; g.sBn = K;
  g.C = Y; g.sCm = N;
  g.bias = bias; g.M = M; g.N = N; g.K = K; g.nh = 1; g.alpha = 1.0f;
  return g;
}
SG lin_back(const float* dY, int M, int N, const float* W, int K, float* dX, bool acc) {
  // dX[M, K] (+)= dY[M, N] W[N, K]
  SG g{};
  g.A = dY; g.sAm = N; g.sAk = 1;
  g.B = W; g.sBk = K; g.sBn = 1;
  g.C = dX; g.sCm = K;
  g.M = M; g.N = K; g.K = N; g.nh = 1; g.alpha = 1.0f; g.accumulate = acc ? 1 : 0;
  return g;
}

ff_status launch_ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return sfail(FF_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return FF_OK;
}
#define SL(x, what)                                   \
  do {                                                \
    ff_status s_ = launch_ck((x), what);              \
    if (s_ != FF_OK) return s_;                       \
  } while (0)

int rows_threads(int H) { return H >= 512 ? 256 : 128; }

// One linear of the scorer, Y[M x N] (+)= X[M x K] B^T (+ bias) with B the
// split weight operand w ([N x K]: W for Y = X W^T, W^T for dX = dY W): split
// X (row-scaled fp16 hi / lo), then the 3xFP16 tcgen05 GEMM (gemm_x3.cu).  With
// FF_SCORER_OPT_TC_LINEARS = 0 the SIMT SGEMM `g` (same contraction) runs instead.
ff_status linear(ff_scorer* m, const SG& g, const XSplit& w, const SplitKScratch& sk, cudaStream_t s,
                 const char* what) {
  if (!m->tc_linears) {
    SL(sgemm(g, 1, s, sk), what);
    return FF_OK;
  }
  const int K = g.K, kp = round8(K);
  __half* xh = m->hws(m->xh);
  __half* xl = m->hws(m->xl);
  float* xs = m->ws(m->xs);
  SL(ff::launch_split_x3(g.A, g.M, K, (int)g.sAm, xh, xl, kp, xs, s), what);
  const char* err = nullptr;
  const cudaError_t e = ff::launch_gemm_x3(xh, xl, xs, kp, m->hw(w.h), m->hw(w.l), m->w(w.s), w.ld, g.M, g.N, K,
                                           g.bias, g.C, (int)g.sCm, g.accumulate != 0, s, &err, 2, sk.ws, sk.cap);
  if (e != cudaSuccess) return sfail(FF_E_CUDA, std::string(what) + ": " + (err ? err : cudaGetErrorString(e)));
  return FF_OK;
}
#define LIN(g, w, what)                               \
  do {                                                \
    ff_status s_ = linear(m, (g), (w), sk, s, what);  \
    if (s_ != FF_OK) return s_;                       \
  } while (0)

ff_status score_batch(ff_scorer* m, const int* ids, const int* mask, const int* labels, int B, int S, double* hsc,
                      double* fsc, float* loss, float* logits, cudaStream_t s) {
  const ff_config& c = m->cfg;
  const int H = c.hidden, d = c.head_dim, M = B * S, C = c.num_classes;
  const float scale = 1.0f / sqrtf((float)d);
  const int rt = rows_threads(H);
  const size_t lnsm = (size_t)(H + 32) * 4;
  SplitKScratch sk;  // split-K scratch of this scorer (stream-ordered use)
  sk.ws = m->ws(m->skws);
  sk.cap = m->tws_floats;
  // ---- forward, keeping what the backward needs
  int* errf = reinterpret_cast<int*>(m->dWS + m->errf);
  embed_ln_f32_kernel<<<M, rt, lnsm, s>>>(ids, mask, S, H, c.vocab_size, m->w(m->tok), m->w(m->pos), m->w(m->type0),
                                          m->w(m->eg), m->w(m->eb), c.ln_eps, m->ws(m->L[0].X), errf);
  SL(cudaGetLastError(), "embed_ln");
  for (int l = 0; l < c.num_layers; ++l) {
    SLayer& P = m->L[l];
    const int A = P.A, D = P.D, F = P.F;
    float* X = m->ws(P.X);
    float* QKV = m->ws(P.QKV);
    LIN(lin(X, M, H, m->w(P.wqkv), m->w(P.bqkv), QKV, 3 * D), P.qkv, "qkv");
    // S = Q K^T per (b, h) into P, then softmax in place
    SG g{};
    g.A = QKV; g.sAb = (long long)S * 3 * D; g.sAh = d; g.sAm = 3 * D; g.sAk = 1;
    g.B = QKV + D; g.sBb = (long long)S * 3 * D; g.sBh = d; g.sBk = 1; g.sBn = 3 * D;
    g.C = m->ws(P.P); g.sCb = (long long)A * S * S; g.sCh = (long long)S * S; g.sCm = S;
    g.M = S; g.N = S; g.K = d; g.nh = A; g.alpha = 1.0f;
    SL(sgemm(g, B * A, s), "qk");
    softmax_fwd_kernel<<<B * A * S, 128, 0, s>>>(m->ws(P.P), mask, S, A, scale);
    SL(cudaGetLastError(), "softmax");
    // ctx = P V
    g = SG{};
    g.A = m->ws(P.P); g.sAb = (long long)A * S * S; g.sAh = (long long)S * S; g.sAm = S; g.sAk = 1;
    g.B = QKV + 2 * D; g.sBb = (long long)S * 3 * D; g.sBh = d; g.sBk = 3 * D; g.sBn = 1;
    g.C = m->ws(P.Cx); g.sCb = (long long)S * D; g.sCh = d; g.sCm = D;
    g.M = S; g.N = d; g.K = S; g.nh = A; g.alpha = 1.0f;
    SL(sgemm(g, B * A, s), "pv");
    float* O = m->ws(m->dZ);  // scratch for the projection outputs
    LIN(lin(m->ws(P.Cx), M, D, m->w(P.wo), m->w(P.bo), O, H), P.o, "oproj");
    add_ln_f32_kernel<<<M, rt, lnsm, s>>>(O, X, H, m->w(P.g1), m->w(P.b1), c.ln_eps, m->ws(P.Y1), m->ws(P.XH1),
                                          m->ws(P.R1));
    SL(cudaGetLastError(), "ln1");
    LIN(lin(m->ws(P.Y1), M, H, m->w(P.w1), m->w(P.bi1), m->ws(P.U), F), P.f1, "ffn1");
    act_fwd_kernel<<<1184, 256, 0, s>>>(m->ws(P.U), m->ws(P.Act), (size_t)M * F, c.act);
    SL(cudaGetLastError(), "act");
    LIN(lin(m->ws(P.Act), M, F, m->w(P.w2), m->w(P.bi2), O, H), P.f2, "ffn2");
    float* Xn = l + 1 < c.num_layers ? m->ws(m->L[l + 1].X) : m->ws(m->Xout);
    add_ln_f32_kernel<<<M, rt, lnsm, s>>>(O, m->ws(P.Y1), H, m->w(P.g2), m->w(P.b2), c.ln_eps, Xn, m->ws(P.XH2),
                                          m->ws(P.R2));
    SL(cudaGetLastError(), "ln2");
  }
  // ---- head: loss and the gradient at position 0 of the last layer
  SC_CK(cudaMemsetAsync(m->ws(m->dX), 0, (size_t)M * H * 4, s));
  {
    float* pool = m->ws(m->headws);
    float* dpre = pool + (size_t)B * H;
    head_pool_kernel<<<dim3(B, (H + 7) / 8), 256, 0, s>>>(m->ws(m->Xout), S, H, m->w(m->pw), m->w(m->pb), pool);
    head_loss_kernel<<<B, 256, 0, s>>>(pool, H, C, B, m->w(m->cw), m->w(m->cb), labels, m->ws(m->lossb), logits, dpre,
                                       errf);
    head_dx_kernel<<<dim3(B, (H + 255) / 256), 256, 0, s>>>(dpre, S, H, m->w(m->pw), m->ws(m->dX));
  }
  SL(cudaGetLastError(), "head");
  if (loss) {
    loss_mean_kernel<<<1, 32, 0, s>>>(m->ws(m->lossb), B, loss);
    SL(cudaGetLastError(), "loss");
  }
  // ---- backward, layer by layer
  const int sc_ld = std::max(m->Amax, 1);
  for (int l = c.num_layers - 1; l >= 0; --l) {
    SLayer& P = m->L[l];
    const int A = P.A, D = P.D, F = P.F;
    float* dX = m->ws(m->dX);
    float* dZ = m->ws(m->dZ);
    float* dY1 = m->ws(m->dY1);
    float* dAm = m->ws(m->dAm);
    ln_bwd_kernel<<<M, rt, 32 * 4, s>>>(dX, m->w(P.g2), m->ws(P.XH2), m->ws(P.R2), H, dZ);  // d(o2 + y1)
    SL(cudaGetLastError(), "ln2 bwd");
    LIN(lin_back(dZ, M, H, m->w(P.w2), F, dAm, false), P.f2T, "ffn2 bwd");  // d(act * nu)
    colprod_kernel<<<dim3((F + 31) / 32, kRowChunks), 256, 0, s>>>(m->ws(P.Act), dAm, M, F, F, m->ws(m->colg));
    group_abs_add_kernel<<<(F + 3) / 4, 128, 0, s>>>(m->ws(m->colg), F, F, 1, fsc + (size_t)l * m->Fmax);
    act_bwd_kernel<<<1184, 256, 0, s>>>(m->ws(P.U), dAm, (size_t)M * F, c.act);
    copy_kernel<<<1184, 256, 0, s>>>(dZ, dY1, (size_t)M * H);
    LIN(lin_back(dAm, M, F, m->w(P.w1), H, dY1, true), P.f1T, "ffn1 bwd");
    ln_bwd_kernel<<<M, rt, 32 * 4, s>>>(dY1, m->w(P.g1), m->ws(P.XH1), m->ws(P.R1), H, dZ);  // d(o + x)
    SL(cudaGetLastError(), "ln1 bwd");
    float* dC = m->ws(m->dC);
    LIN(lin_back(dZ, M, H, m->w(P.wo), D, dC, false), P.oT, "oproj bwd");
    colprod_kernel<<<dim3((D + 31) / 32, kRowChunks), 256, 0, s>>>(m->ws(P.Cx), dC, M, D, D, m->ws(m->colg));
    group_abs_add_kernel<<<(A + 3) / 4, 128, 0, s>>>(m->ws(m->colg), D, A, d, hsc + (size_t)l * sc_ld);
    // attention backward per (b, h)
    float* QKV = m->ws(P.QKV);
    float* dQKV = m->ws(m->dQKV);
    float* dP = m->ws(m->dP);
    const float* Pm = m->ws(P.P);
    SG g{};  // dP = dC V^T
    g.A = dC; g.sAb = (long long)S * D; g.sAh = d; g.sAm = D; g.sAk = 1;
    g.B = QKV + 2 * D; g.sBb = (long long)S * 3 * D; g.sBh = d; g.sBk = 1; g.sBn = 3 * D;
    g.C = dP; g.sCb = (long long)A * S * S; g.sCh = (long long)S * S; g.sCm = S;
    g.M = S; g.N = S; g.K = d; g.nh = A; g.alpha = 1.0f;
    SL(sgemm(g, B * A, s), "dP");
    g = SG{};  // dV = P^T dC
    g.A = Pm; g.sAb = (long long)A * S * S; g.sAh = (long long)S * S; g.sAm = 1; g.sAk = S;
    g.B = dC; g.sBb = (long long)S * D; g.sBh = d; g.sBk = D; g.sBn = 1;
    g.C = dQKV + 2 * D; g.sCb = (long long)S * 3 * D; g.sCh = d; g.sCm = 3 * D;
    g.M = S; g.N = d; g.K = S; g.nh = A; g.alpha = 1.0f;
    SL(sgemm(g, B * A, s), "dV");
    softmax_bwd_kernel<<<B * A * S, 128, 0, s>>>(Pm, dP, S, scale);  // dP -> dS (scaled)
    SL(cudaGetLastError(), "softmax bwd");
    g = SG{};  // dQ = dS K
    g.A = dP; g.sAb = (long long)A * S * S; g.sAh = (long long)S * S; g.sAm = S; g.sAk = 1;
    g.B = QKV + D; g.sBb = (long long)S * 3 * D; g.sBh = d; g.sBk = 3 * D; g.sBn = 1;
    g.C = dQKV; g.sCb = (long long)S * 3 * D; g.sCh = d; g.sCm = 3 * D;
    g.M = S; g.N = d; g.K = S; g.nh = A; g.alpha = 1.0f;
    SL(sgemm(g, B * A, s), "dQ");
    g = SG{};  // dK = dS^T Q
    g.A = dP; g.sAb = (long long)A * S * S; g.sAh = (long long)S * S; g.sAm = 1; g.sAk = S;
    g.B = QKV; g.sBb = (long long)S * 3 * D; g.sBh = d; g.sBk = 3 * D; g.sBn = 1;
    g.C = dQKV + D; g.sCb = (long long)S * 3 * D; g.sCh = d; g.sCm = 3 * D;
    g.M = S; g.N = d; g.K = S; g.nh = A; g.alpha = 1.0f;
    SL(sgemm(g, B * A, s), "dK");
    if (l > 0) {  // gradient w.r.t. the layer input (residual + QKV path)
      copy_kernel<<<1184, 256, 0, s>>>(dZ, dX, (size_t)M * H);
      LIN(lin_back(dQKV, M, 3 * D, m->w(P.wqkv), H, dX, true), P.qkvT, "qkv bwd");
    }
  }
  return FF_OK;
}

}  // namespace

extern "C" {

const char* ff_scorer_last_error(void) { return g_serr.c_str(); }

ff_status ff_scorer_create(const ff_config* cfg, int32_t cuda_device, ff_scorer** out) {
  if (!cfg || !out) return sfail(FF_E_INVALID, "null argument");
  if (cfg->abi_version != FF_ABI_VERSION) return sfail(FF_E_INVALID, "abi_version mismatch");
  if (cfg->num_layers < 1 || cfg->hidden < 1 || cfg->head_dim < 1 || cfg->vocab_size < 1 ||
      cfg->max_positions < 1 || cfg->num_classes < 1 || cfg->num_classes > 64 || cfg->max_tokens < 1 ||
      !cfg->heads || !cfg->ffn_dim || cfg->act < 0 || cfg->act > 2)
    return sfail(FF_E_INVALID, "invalid config");
  auto* m = new ff_scorer();
  m->cfg = *cfg;
  m->heads.assign(cfg->heads, cfg->heads + cfg->num_layers);
  m->ffn.assign(cfg->ffn_dim, cfg->ffn_dim + cfg->num_layers);
  for (int l = 0; l < cfg->num_layers; ++l)
    if (m->heads[l] < 1 || m->ffn[l] < 1) {
      delete m;
      return sfail(FF_E_INVALID, "heads / ffn_dim must be >= 1");
    }
  m->cfg.heads = m->heads.data();
  m->cfg.ffn_dim = m->ffn.data();
  m->cfg.dtype = nullptr;
  m->device = cuda_device;
  plan_scorer(m);
  *out = m;
  return FF_OK;
}

ff_status ff_scorer_memory(const ff_scorer* m, size_t* weight_bytes, size_t* workspace_bytes) {
  if (!m || !weight_bytes || !workspace_bytes) return sfail(FF_E_INVALID, "null argument");
  *weight_bytes = m->wbytes;
  *workspace_bytes = m->wsbytes;
  return FF_OK;
}

ff_status ff_scorer_bind_memory(ff_scorer* m, void* d_weights, size_t wbytes, void* d_workspace, size_t wsbytes) {
  if (!m || !d_weights || !d_workspace) return sfail(FF_E_INVALID, "null argument");
  if (wbytes < m->wbytes || wsbytes < m->wsbytes) return sfail(FF_E_INVALID, "arena too small");
  if (((uintptr_t)d_weights | (uintptr_t)d_workspace) & 255) return sfail(FF_E_INVALID, "arenas must be 256-B aligned");
  m->dW = static_cast<uint8_t*>(d_weights);
  m->dWS = static_cast<uint8_t*>(d_workspace);
  SDev dg_(m->device);
  SC_CK(cudaMemset(m->dWS + m->errf, 0, 64));
  m->state = 1;
  return FF_OK;
}

ff_status ff_scorer_load_weights(ff_scorer* m, const char* name, const float* host, const int64_t* shape,
                                 int32_t rank, void* stream) {
  if (!m || !name || !host || !shape) return sfail(FF_E_INVALID, "null argument");
  if (m->state < 1) return sfail(FF_E_STATE, "bind memory first");
  std::string n(name);
  for (const char* p : {"bert.", "roberta."})
    if (n.compare(0, std::strlen(p), p) == 0) n = n.substr(std::strlen(p));
  const int H = m->cfg.hidden, d = m->cfg.head_dim;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  size_t numel = 1;
  for (int i = 0; i < rank; ++i) numel *= (size_t)shape[i];
  auto put = [&](size_t off, size_t expect) -> ff_status {
    if (numel != expect) return sfail(FF_E_SHAPE, "wrong shape for " + std::string(name));
    SDev dg_(m->device);
    SC_CK(cudaMemcpyAsync(m->dW + off, host, numel * 4, cudaMemcpyHostToDevice, s));
    SC_CK(cudaStreamSynchronize(s));  // host buffer may be freed after return
    if (m->state == 2) m->state = 1;  // derived TF32 splits are stale: finalize again
    return FF_OK;
  };
  const ff_config& c = m->cfg;
  if (n == "embeddings.word_embeddings.weight") { m->top_loaded |= 1; return put(m->tok, (size_t)c.vocab_size * H); }
  if (n == "embeddings.position_embeddings.weight") {
    // only the first max_positions rows are copied: the table must be 2-D [>= max_positions, hidden]
    if (rank != 2 || shape[1] != H || shape[0] < c.max_positions)
      return sfail(FF_E_SHAPE, "position table must be [>= max_positions, hidden]");
    numel = (size_t)c.max_positions * H;
    m->top_loaded |= 2;
    return put(m->pos, numel);
  }
  if (n == "embeddings.token_type_embeddings.weight") {  // row 0 only (DESIGN R16)
    if (rank != 2 || shape[1] != H || shape[0] < 1)
      return sfail(FF_E_SHAPE, "token-type table must be [>= 1, hidden]");
    numel = H;
    m->top_loaded |= 4;
    return put(m->type0, H);
  }
  if (n == "embeddings.LayerNorm.weight") { m->top_loaded |= 8; return put(m->eg, H); }
  if (n == "embeddings.LayerNorm.bias") { m->top_loaded |= 16; return put(m->eb, H); }
  if (n == "pooler.dense.weight" || n == "classifier.dense.weight") { m->top_loaded |= 32; return put(m->pw, (size_t)H * H); }
  if (n == "pooler.dense.bias" || n == "classifier.dense.bias") { m->top_loaded |= 64; return put(m->pb, H); }
  if (n == "classifier.weight" || n == "classifier.out_proj.weight") { m->top_loaded |= 128; return put(m->cw, (size_t)c.num_classes * H); }
  if (n == "classifier.bias" || n == "classifier.out_proj.bias") { m->top_loaded |= 256; return put(m->cb, c.num_classes); }
  int l = -1, used = 0;
  if (std::sscanf(n.c_str(), "encoder.layer.%d.%n", &l, &used) == 1 && l >= 0 && l < c.num_layers) {
    const std::string key = n.substr(used);
    SLayer& P = m->L[l];
    const size_t D = P.D, F = P.F;
    for (int k = 0; k < 16; ++k) {
      if (key != kSLayer[k]) continue;
      P.loaded |= 1u << k;
      switch (k) {
        case 0: case 1: case 2: return put(P.wqkv + (size_t)k * D * H * 4, D * H);
        case 3: case 4: case 5: return put(P.bqkv + (size_t)(k - 3) * D * 4, D);
        case 6: return put(P.wo, (size_t)H * D);
        case 7: return put(P.bo, H);
        case 8: return put(P.g1, H);
        case 9: return put(P.b1, H);
        case 10: return put(P.w1, F * H);
        case 11: return put(P.bi1, F);
        case 12: return put(P.w2, (size_t)H * F);
        case 13: return put(P.bi2, H);
        case 14: return put(P.g2, H);
        default: return put(P.b2, H);
      }
    }
  }
  (void)d;
  return sfail(FF_E_SHAPE, "unknown tensor " + std::string(name));
}

ff_status ff_scorer_finalize(ff_scorer* m, void* stream) {
  if (!m) return sfail(FF_E_INVALID, "null argument");
  if (m->state < 1) return sfail(FF_E_STATE, "bind memory first");
  if (m->top_loaded != 511u) return sfail(FF_E_STATE, "missing embedding / pooler / classifier tensors");
  for (auto& P : m->L)
    if (P.loaded != 0xFFFFu) return sfail(FF_E_STATE, "missing layer tensors");
  // row-scaled fp16 hi / lo splits of every linear's weight and of its
  // transpose (the B operands of the tcgen05 linears), from the loaded fp32
  // weights; W^T goes through the split-K scratch of the workspace
  SDev dg_(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int H = m->cfg.hidden;
  for (auto& P : m->L) {
    const int D = P.D, F = P.F;
    struct {
      size_t w;
      int n, k;
      XSplit *fwd, *bwd;
    } ws[4] = {{P.wqkv, 3 * D, H, &P.qkv, &P.qkvT}, {P.wo, H, D, &P.o, &P.oT}, {P.w1, F, H, &P.f1, &P.f1T},
               {P.w2, H, F, &P.f2, &P.f2T}};
    for (auto& x : ws) {
      SC_CK(ff::launch_split_x3(m->w(x.w), x.n, x.k, x.k, m->hw(x.fwd->h), m->hw(x.fwd->l), x.fwd->ld,
                                m->w(x.fwd->s), s));
      if ((size_t)x.n * x.k > m->tws_floats) return sfail(FF_E_STATE, "transpose scratch too small");
      float* wt = m->ws(m->tws);
      SC_CK(ff::launch_transpose_f32(m->w(x.w), x.n, x.k, wt, s));
      SC_CK(ff::launch_split_x3(wt, x.k, x.n, x.n, m->hw(x.bwd->h), m->hw(x.bwd->l), x.bwd->ld, m->w(x.bwd->s), s));
    }
  }
  SC_CK(cudaStreamSynchronize(s));
  m->state = 2;
  return FF_OK;
}

ff_status ff_score_batch(ff_scorer* m, const int32_t* d_ids, const int32_t* d_mask, const int32_t* d_labels,
                         int32_t batch, int32_t seq, double* d_head_scores, double* d_ffn_scores, float* d_loss,
                         float* d_logits, void* stream) {
  if (!m || !d_ids || !d_mask || !d_labels || !d_head_scores || !d_ffn_scores)
    return sfail(FF_E_INVALID, "null argument");
  if (m->state != 2) return sfail(FF_E_STATE, "ff_scorer_finalize first");
  if (batch < 1 || seq < 1 || seq > m->cfg.max_positions || (int64_t)batch * seq > m->cfg.max_tokens)
    return sfail(FF_E_SHAPE, "batch * seq exceeds max_tokens or seq > max_positions");
  SDev dg_(m->device);
  return score_batch(m, d_ids, d_mask, d_labels, batch, seq, d_head_scores, d_ffn_scores, d_loss, d_logits,
                     static_cast<cudaStream_t>(stream));
}

ff_status ff_scorer_check(ff_scorer* m, void* stream) {
  if (!m) return sfail(FF_E_INVALID, "null argument");
  if (m->state < 1) return sfail(FF_E_STATE, "bind memory first");
  SDev dg_(m->device);
  SC_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  int flag = 0;
  SC_CK(cudaMemcpy(&flag, m->dWS + m->errf, 4, cudaMemcpyDeviceToHost));
  if (flag) {
    SC_CK(cudaMemset(m->dWS + m->errf, 0, 4));
    std::string why;
    if (flag & 1) why += " token id outside [0, vocab)";
    if (flag & 2) why += " mask value not 0/1 or mask[b,0] != 1";
    if (flag & 4) why += " label outside [0, num_classes)";
    return sfail(FF_E_INPUT, "input error:" + why);
  }
  return FF_OK;
}

ff_status ff_debug_gemm_x3(const float* d_A, int32_t lda, const float* d_B, int32_t ldb, int32_t M, int32_t N,
                           int32_t K, const float* d_bias, float* d_C, int32_t ldc, int32_t accumulate, int32_t kc,
                           void* stream) {
  if (!d_A || !d_B || !d_C) return sfail(FF_E_INVALID, "null argument");
  if (M < 1 || N < 1 || K < 1 || lda < K || ldb < K || ldc < N || kc < 1) return sfail(FF_E_SHAPE, "bad GEMM shape");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int kp = round8(K);
  __half *ah = nullptr, *bh = nullptr;
  float *sa = nullptr, *ws = nullptr;  // row scales; split-K partials, as the scorer provides
  SC_CK(cudaMallocAsync(reinterpret_cast<void**>(&ah), (size_t)2 * M * kp * 2, s));
  SC_CK(cudaMallocAsync(reinterpret_cast<void**>(&bh), (size_t)2 * N * kp * 2, s));
  SC_CK(cudaMallocAsync(reinterpret_cast<void**>(&sa), (size_t)(M + N) * 4, s));
  SC_CK(cudaMallocAsync(reinterpret_cast<void**>(&ws), (size_t)4 * M * N * 4, s));
  __half* al = ah + (size_t)M * kp;
  __half* bl = bh + (size_t)N * kp;
  float* sb = sa + M;
  cudaError_t e = ff::launch_split_x3(d_A, M, K, lda, ah, al, kp, sa, s);
  if (e == cudaSuccess) e = ff::launch_split_x3(d_B, N, K, ldb, bh, bl, kp, sb, s);
  const char* err = nullptr;
  if (e == cudaSuccess)
    e = ff::launch_gemm_x3(ah, al, sa, kp, bh, bl, sb, kp, M, N, K, d_bias, d_C, ldc, accumulate != 0, s, &err, kc,
                           ws, (size_t)4 * M * N);
  cudaFreeAsync(ah, s);
  cudaFreeAsync(bh, s);
  cudaFreeAsync(sa, s);
  cudaFreeAsync(ws, s);
  if (e != cudaSuccess) return sfail(FF_E_CUDA, err ? err : cudaGetErrorString(e));
  return FF_OK;
}

ff_status ff_scorer_set_option(ff_scorer* m, int32_t option, int32_t value) {
  if (!m) return sfail(FF_E_INVALID, "null argument");
  if (option == FF_SCORER_OPT_TC_LINEARS) {
    if (value != 0 && value != 1) return sfail(FF_E_INVALID, "FF_SCORER_OPT_TC_LINEARS takes 0 or 1");
    m->tc_linears = value;
    return FF_OK;
  }
  return sfail(FF_E_INVALID, "unknown scorer option");
}

void ff_scorer_destroy(ff_scorer* m) { delete m; }

}  // extern "C"
