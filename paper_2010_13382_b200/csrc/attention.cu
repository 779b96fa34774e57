// attention.cu -- fused masked-softmax attention over the ragged pruned head
// count of one layer ("multi-head attention node
// fusion"; Q.K^T and P.V in floating point).
//
// For every (sequence b, surviving head h < A'_l, 128-query tile):
//   s_ij = fp32(q_i . k_j) * fp32(1/sqrt(d))        keys with mask 0 excluded (R4)
//   p_ij = exp(s_ij - max_j s_ij) / sum_j exp(.)     fp32, normalized BEFORE
//   P16 = R16(p)                                     the P.V product (R9)
//   ctx_i = R16(sum_j P16_ij v_j)                    fp32 accumulation
// Q, K, V tiles are staged in shared memory (rows padded to d_pad + 8 halves
// so the 32-bit fragment loads are bank-conflict free); QK^T and PV run on the
// tensor cores with mma.sync m16n8k16 (fp16 in, fp32 accumulate); each warp
// owns 16 query rows, so row max / sum are quad-local shuffles.  Keys are
// processed in register chunks of 128: a single pass when S <= 128, else a
// first pass for the row max / sum and a second for P.V (exact normalized
// form, no flash-style rescaling of the output).
// HBM-bound at s <= 256 (reads QKV once, writes ctx once).
#include "ff_kernels.h"
#include "ptx.cuh"

namespace ff {

namespace {

constexpr int QT = 128;  // query rows per CTA (8 warps x 16)
constexpr int KC = 128;  // keys per register chunk

// Copy `rows` rows of d fp16 from global (row pitch ld) into smem rows of
// stride LDS, zero-filling columns [d, DP) and rows [rows, total_rows).
template <int DP, int LDS>
__device__ __forceinline__ void load_tile(__half* dst, const __half* src, int ld, int rows, int total_rows, int d,
                                          bool vec) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (vec) {  // d % 8 == 0, 16-byte aligned rows
    const int cpr = DP / 8;  // uint4 chunks per smem row
    for (int i = tid; i < total_rows * cpr; i += nt) {
      const int r = i / cpr, c = (i - r * cpr) * 8;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < rows && c < d) v = *reinterpret_cast<const uint4*>(src + (size_t)r * ld + c);
      *reinterpret_cast<uint4*>(dst + r * LDS + c) = v;
    }
  } else {
    const int cpr = DP / 2;
    for (int i = tid; i < total_rows * cpr; i += nt) {
      const int r = i / cpr, c = (i - r * cpr) * 2;
      uint32_t v = 0;
      if (r < rows && c < d) v = *reinterpret_cast<const uint32_t*>(src + (size_t)r * ld + c);
      *reinterpret_cast<uint32_t*>(dst + r * LDS + c) = v;
    }
  }
}

template <int DP>
__global__ void __launch_bounds__(256) attention_kernel(const __half* __restrict__ qkv, int ld,
                                                       const int32_t* __restrict__ mask, int S, int A, int d,
                                                       float scale, __half* __restrict__ ctx, int ldc) {
  constexpr int LDS = DP + 8;
  constexpr int NT = KC / 8;  // n-tiles per chunk
  extern __shared__ __align__(16) uint8_t smem[];
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int S16 = (S + 15) & ~15;
  __half* sQ = reinterpret_cast<__half*>(smem);
  __half* sK = sQ + QT * LDS;
  __half* sV = sK + S16 * LDS;
  float* sMask = reinterpret_cast<float*>(sV + S16 * LDS);

  const int D = A * d;
  const size_t tok0 = (size_t)b * S;
  const int q0 = qt * QT;
  const bool vec = ((d & 7) == 0) && ((ld & 7) == 0);
  load_tile<DP, LDS>(sQ, qkv + (tok0 + q0) * ld + h * d, ld, min(QT, S - q0), QT, d, vec);
  load_tile<DP, LDS>(sK, qkv + tok0 * ld + D + h * d, ld, S, S16, d, vec);
  load_tile<DP, LDS>(sV, qkv + tok0 * ld + 2 * D + h * d, ld, S, S16, d, vec);
  for (int i = threadIdx.x; i < S16; i += blockDim.x)
    sMask[i] = (i < S && mask[tok0 + i] != 0) ? 0.0f : -INFINITY;
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = warp * 16;
  if (q0 + r0 >= S) return;
  const int g = lane >> 2, tig = lane & 3;

  uint32_t qf[DP / 16][4];
#pragma unroll
  for (int kk = 0; kk < DP / 16; ++kk)
    ldmatrix_x4(qf[kk], sQ + (r0 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);

  float s[NT][4];
  auto compute_s = [&](int kb) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      if (kb + nt * 8 < S16) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        const __half* krow = sK + (kb + nt * 8 + g) * LDS + tig * 2;
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk) {
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(krow + kk * 16);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(krow + kk * 16 + 8);
          mma_16816(acc, qf[kk], b0, b1);
        }
        const float mk0 = sMask[kb + nt * 8 + tig * 2], mk1 = sMask[kb + nt * 8 + tig * 2 + 1];
        s[nt][0] = __fmul_rn(acc[0], scale) + mk0;
        s[nt][1] = __fmul_rn(acc[1], scale) + mk1;
        s[nt][2] = __fmul_rn(acc[2], scale) + mk0;
        s[nt][3] = __fmul_rn(acc[3], scale) + mk1;
      } else {
        s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = -INFINITY;
      }
    }
  };
  auto quad_max = [](float v) {
    v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
    return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
  };
  auto quad_sum = [](float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v + __shfl_xor_sync(0xffffffffu, v, 2);
  };

  const int nch = (S16 + KC - 1) / KC;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows g and g + 8
  if (nch > 1) {
    for (int c = 0; c < nch; ++c) {
      compute_s(c * KC);
      float c0 = -INFINITY, c1 = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        c0 = fmaxf(c0, fmaxf(s[nt][0], s[nt][1]));
        c1 = fmaxf(c1, fmaxf(s[nt][2], s[nt][3]));
      }
      c0 = fmaxf(m0, quad_max(c0));
      c1 = fmaxf(m1, quad_max(c1));
      float e0 = 0.f, e1 = 0.f;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        e0 += expf(s[nt][0] - c0) + expf(s[nt][1] - c0);
        e1 += expf(s[nt][2] - c1) + expf(s[nt][3] - c1);
      }
      l0 = l0 * expf(m0 - c0) + quad_sum(e0);
      l1 = l1 * expf(m1 - c1) + quad_sum(e1);
      m0 = c0;
      m1 = c1;
    }
  }

  float o[DP / 8][4];
#pragma unroll
  for (int i = 0; i < DP / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;

  for (int c = 0; c < nch; ++c) {
    const int kb = c * KC;
    compute_s(kb);
    if (nch == 1) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        m0 = fmaxf(m0, fmaxf(s[nt][0], s[nt][1]));
        m1 = fmaxf(m1, fmaxf(s[nt][2], s[nt][3]));
      }
      m0 = quad_max(m0);
      m1 = quad_max(m1);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        s[nt][0] = expf(s[nt][0] - m0);
        s[nt][1] = expf(s[nt][1] - m0);
        s[nt][2] = expf(s[nt][2] - m1);
        s[nt][3] = expf(s[nt][3] - m1);
        l0 += s[nt][0] + s[nt][1];
        l1 += s[nt][2] + s[nt][3];
      }
      l0 = quad_sum(l0);
      l1 = quad_sum(l1);
    } else {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        s[nt][0] = expf(s[nt][0] - m0);
        s[nt][1] = expf(s[nt][1] - m0);
        s[nt][2] = expf(s[nt][2] - m1);
        s[nt][3] = expf(s[nt][3] - m1);
      }
    }
    // normalize in fp32, round P to fp16 (R9), then P.V on the tensor cores
#pragma unroll
    for (int t = 0; t < NT / 2; ++t) {
      if (kb + t * 16 < S16) {
        uint32_t pa[4];
        pa[0] = pack_half2(__fdiv_rn(s[2 * t][0], l0), __fdiv_rn(s[2 * t][1], l0));
        pa[1] = pack_half2(__fdiv_rn(s[2 * t][2], l1), __fdiv_rn(s[2 * t][3], l1));
        pa[2] = pack_half2(__fdiv_rn(s[2 * t + 1][0], l0), __fdiv_rn(s[2 * t + 1][1], l0));
        pa[3] = pack_half2(__fdiv_rn(s[2 * t + 1][2], l1), __fdiv_rn(s[2 * t + 1][3], l1));
        const __half* vrow = sV + (kb + t * 16 + (lane & 15)) * LDS;
#pragma unroll
        for (int dn = 0; dn < DP / 8; ++dn) {
          uint32_t b0, b1;
          ldmatrix_x2_trans(b0, b1, vrow + dn * 8);
          mma_16816(o[dn], pa, b0, b1);
        }
      }
    }
  }

  // store ctx rows g and g+8 of this warp, columns < d
  const int qa = q0 + r0 + g, qb = qa + 8;
  __half* ca = ctx + (tok0 + qa) * ldc + h * d;
  __half* cb = ctx + (tok0 + qb) * ldc + h * d;
#pragma unroll
  for (int dn = 0; dn < DP / 8; ++dn) {
    const int col = dn * 8 + tig * 2;
    if (col < d) {  // d is even, so col + 1 < d as well
      if (qa < S) *reinterpret_cast<uint32_t*>(ca + col) = pack_half2(o[dn][0], o[dn][1]);
      if (qb < S) *reinterpret_cast<uint32_t*>(cb + col) = pack_half2(o[dn][2], o[dn][3]);
    }
  }
}

template <int DP>
size_t attn_smem(int S) {
  const int S16 = (S + 15) & ~15;
  return (size_t)(QT + 2 * S16) * (DP + 8) * sizeof(__half) + (size_t)S16 * sizeof(float);
}

template <int DP>
cudaError_t launch_dp(const __half* qkv, int ld, const int32_t* mask, int B, int S, int A, int d, __half* ctx,
                      int ldc, cudaStream_t s) {
  const size_t smem = attn_smem<DP>(S);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  const float scale = (float)(1.0 / sqrt((double)d));  // fp32(1/sqrt(d)) (R10)
  dim3 grid((S + QT - 1) / QT, A, B);
  attention_kernel<DP><<<grid, 256, smem, s>>>(qkv, ld, mask, S, A, d, scale, ctx, ldc);
  return cudaGetLastError();
}

}  // namespace

cudaError_t prepare_attention_kernels() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(attention_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(attention_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess) return e;
  return cudaFuncSetAttribute(attention_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

size_t attention_smem_bytes(int S, int d) {
  if (d <= 32) return attn_smem<32>(S);
  if (d <= 64) return attn_smem<64>(S);
  return attn_smem<128>(S);
}

cudaError_t launch_attention(const __half* qkv, int ldqkv, const int32_t* mask, int B, int S, int A, int d,
                             __half* ctx, int ldctx, cudaStream_t s) {
  if (d <= 32) return launch_dp<32>(qkv, ldqkv, mask, B, S, A, d, ctx, ldctx, s);
  if (d <= 64) return launch_dp<64>(qkv, ldqkv, mask, B, S, A, d, ctx, ldctx, s);
  return launch_dp<128>(qkv, ldqkv, mask, B, S, A, d, ctx, ldctx, s);
}

}  // namespace ff
