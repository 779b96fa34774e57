// attention.cu -- fused masked-softmax attention over the ragged pruned head
// count of one layer ("multi-head attention node
// fusion"; Q.K^T and P.V in floating point).
//
// For every (sequence b, surviving head h < A'_l, 128-query tile):
//   s_ij = fp32(q_i . k_j) * fp32(1/sqrt(d))        keys with mask 0 excluded (R4)
//   p_ij = exp(s_ij - max_j s_ij) / sum_j exp(.)     fp32, normalized BEFORE
//   P16 = R16(p)                                     the P.V product (R9)
//   ctx_i = R16(sum_j P16_ij v_j)                    fp32 accumulation
//
// Persistent kernel: each CTA loops over (b, h, query-tile) work items and
// prefetches the next item's Q/K/V head slices with cp.async into the second
// of two shared-memory buffers while it computes the current one, so the HBM
// reads overlap the math (the kernel is HBM-bound at s <= 256: it reads QKV
// once and writes ctx once).  Smem rows are padded to d_pad + 8 halves so the
// 32-bit fragment loads are bank-conflict free.  QK^T and PV run on the tensor
// cores with mma.sync m16n8k16 (fp16 in, fp32 accumulate); each of the 8 warps
// owns 16 query rows, so row max / sum are quad-local shuffles.  Keys are held
// in register chunks of 128: one pass when S <= 128, else a max/sum pass and a
// P.V pass (exact normalized form, no flash-style output rescaling).
#include "ff_kernels.h"
#include "ptx.cuh"
#include "quant.cuh"

namespace ff {

namespace {

constexpr int QT = 128;  // query rows per work item (8 warps x 16)
constexpr int KC = 128;  // keys per register chunk

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct Item {
  int b, h, qt;
};
__device__ __forceinline__ Item decode(int item, int A, int nqt) {
  Item it;
  it.qt = item % nqt;
  const int bh = item / nqt;
  it.h = bh % A;
  it.b = bh / A;
  return it;
}

// Issue cp.async copies of `rows` rows x d fp16 (row pitch ld) into smem rows of
// stride LDS; rows in [rows, total_rows) and columns [d, DP) are zero-filled.
template <int DP, int LDS>
__device__ __forceinline__ void load_tile_async(__half* dst, const __half* src, int ld, int rows, int total_rows,
                                                int d, bool vec) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (vec) {  // d % 8 == 0, 16-byte aligned rows
    const int cpr = DP / 8;
    for (int i = tid; i < total_rows * cpr; i += nt) {
      const int r = i / cpr, c = (i - r * cpr) * 8;
      const bool ok = r < rows && c < d;
      cp_async16(dst + r * LDS + c, ok ? src + (size_t)r * ld + c : src, ok);
    }
  } else {
    const int cpr = DP / 2;
    for (int i = tid; i < total_rows * cpr; i += nt) {
      const int r = i / cpr, c = (i - r * cpr) * 2;
      const bool ok = r < rows && c < d;
      cp_async4(dst + r * LDS + c, ok ? src + (size_t)r * ld + c : src, ok);
    }
  }
}

template <int DP>
__global__ void __launch_bounds__(256, 1) attention_kernel(const __half* __restrict__ qkv, int ld,
                                                          const int32_t* __restrict__ mask, int B, int S, int A,
                                                          int d, int hs, int hm_rows, float scale,
                                                          __half* __restrict__ ctx, int ldc, int nbuf) {
  constexpr int LDS = DP + 8;
  constexpr int NT = KC / 8;  // n-tiles per chunk
  extern __shared__ __align__(16) uint8_t smem[];
  griddep_wait();
  griddep_launch();
  const int S16 = (S + 15) & ~15;
  const size_t buf_halves = (size_t)(QT + 2 * S16) * LDS;
  const size_t buf_bytes = buf_halves * 2 + (size_t)S16 * 4;
  // QKV sections of A heads of stride hs >= d (hs > d: zero-padded heads,
  // loaded whole so 16-byte copies apply); ctx rows are unpadded (h * d)
  // head slice (t, h) of token r: row-major qkv + r * ld + t * A * hs + h * hs;
  // head-major (hm_rows > 0, ld = 64) qkv + ((t * A + h) * hm_rows + r) * 64
  const size_t sec = hm_rows > 0 ? (size_t)A * hm_rows * 64 : (size_t)A * hs;
  const size_t hst = hm_rows > 0 ? (size_t)hm_rows * 64 : (size_t)hs;
  const int nqt = (S + QT - 1) / QT;
  const int n_items = B * A * nqt;
  const int dl = hs > d ? hs : d;  // columns copied per head (the rest of DP zero-filled)
  const bool vec = ((dl & 7) == 0) && ((ld & 7) == 0);

  auto issue = [&](int item, int buf) {
    const Item it = decode(item, A, nqt);
    uint8_t* base = smem + buf * buf_bytes;
    __half* sQ = reinterpret_cast<__half*>(base);
    __half* sK = sQ + QT * LDS;
    __half* sV = sK + S16 * LDS;
    float* sMask = reinterpret_cast<float*>(base + buf_halves * 2);
    const size_t tok0 = (size_t)it.b * S;
    const int q0 = it.qt * QT;
    load_tile_async<DP, LDS>(sQ, qkv + (tok0 + q0) * ld + it.h * hst, ld, min(QT, S - q0), QT, dl, vec);
    load_tile_async<DP, LDS>(sK, qkv + tok0 * ld + sec + it.h * hst, ld, S, S16, dl, vec);
    load_tile_async<DP, LDS>(sV, qkv + tok0 * ld + 2 * sec + it.h * hst, ld, S, S16, dl, vec);
    for (int i = threadIdx.x; i < S16; i += blockDim.x)
      sMask[i] = (i < S && __ldg(mask + tok0 + i) != 0) ? 0.0f : -INFINITY;
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int r0 = warp * 16;
  constexpr float kLog2e = 1.4426950408889634f;

  int item = blockIdx.x;
  int buf = 0;
  if (item < n_items) issue(item, 0);
  cp_async_commit();
  for (; item < n_items; item += gridDim.x) {
    const int next = item + gridDim.x;
    if (nbuf == 2) {
      if (next < n_items) issue(next, buf ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    const Item it = decode(item, A, nqt);
    uint8_t* base = smem + buf * buf_bytes;
    const __half* sQ = reinterpret_cast<const __half*>(base);
    const __half* sK = sQ + QT * LDS;
    const __half* sV = sK + S16 * LDS;
    const float* sMask = reinterpret_cast<const float*>(base + buf_halves * 2);
    const size_t tok0 = (size_t)it.b * S;
    const int q0 = it.qt * QT;

    if (q0 + r0 < S) {
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
            e0 += ex2((s[nt][0] - c0) * kLog2e) + ex2((s[nt][1] - c0) * kLog2e);
            e1 += ex2((s[nt][2] - c1) * kLog2e) + ex2((s[nt][3] - c1) * kLog2e);
          }
          l0 = l0 * ex2((m0 - c0) * kLog2e) + quad_sum(e0);
          l1 = l1 * ex2((m1 - c1) * kLog2e) + quad_sum(e1);
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
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          s[nt][0] = ex2((s[nt][0] - m0) * kLog2e);
          s[nt][1] = ex2((s[nt][1] - m0) * kLog2e);
          s[nt][2] = ex2((s[nt][2] - m1) * kLog2e);
          s[nt][3] = ex2((s[nt][3] - m1) * kLog2e);
          if (nch == 1) {
            l0 += s[nt][0] + s[nt][1];
            l1 += s[nt][2] + s[nt][3];
          }
        }
        if (nch == 1) {
          l0 = quad_sum(l0);
          l1 = quad_sum(l1);
        }
        const float i0 = __frcp_rn(l0), i1 = __frcp_rn(l1);
        // normalize in fp32 (IEEE e / l), round P to fp16 (R9), then P.V on the tensor cores
#pragma unroll
        for (int t = 0; t < NT / 2; ++t) {
          if (kb + t * 16 < S16) {
            uint32_t pa[4];
            pa[0] = pack_half2(div_cr(s[2 * t][0], l0, i0), div_cr(s[2 * t][1], l0, i0));
            pa[1] = pack_half2(div_cr(s[2 * t][2], l1, i1), div_cr(s[2 * t][3], l1, i1));
            pa[2] = pack_half2(div_cr(s[2 * t + 1][0], l0, i0), div_cr(s[2 * t + 1][1], l0, i0));
            pa[3] = pack_half2(div_cr(s[2 * t + 1][2], l1, i1), div_cr(s[2 * t + 1][3], l1, i1));
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

      const int qa = q0 + r0 + g, qb = qa + 8;
      __half* ca = ctx + (tok0 + qa) * ldc + it.h * d;
      __half* cb = ctx + (tok0 + qb) * ldc + it.h * d;
#pragma unroll
      for (int dn = 0; dn < DP / 8; ++dn) {
        const int col = dn * 8 + tig * 2;
        if (col < d) {  // d is even, so col + 1 < d as well
          if (qa < S) *reinterpret_cast<uint32_t*>(ca + col) = pack_half2(o[dn][0], o[dn][1]);
          if (qb < S) *reinterpret_cast<uint32_t*>(cb + col) = pack_half2(o[dn][2], o[dn][3]);
        }
      }
    }
    __syncthreads();  // everyone is done with `buf` before it is refilled
    if (nbuf == 2) buf ^= 1;
    else if (next < n_items) {
      issue(next, 0);
      cp_async_commit();
    }
  }
  cp_async_wait<0>();
}

template <int DP>
size_t attn_buf_bytes(int S) {
  const int S16 = (S + 15) & ~15;
  return (size_t)(QT + 2 * S16) * (DP + 8) * sizeof(__half) + (size_t)S16 * sizeof(float);
}

constexpr size_t kSmemMax = 227 * 1024;

template <int DP>
cudaError_t launch_dp(const __half* qkv, int ld, const int32_t* mask, int B, int S, int A, int d, int hs,
                      int hm_rows, __half* ctx, int ldc, cudaStream_t s) {
  const size_t one = attn_buf_bytes<DP>(S);
  if (one > kSmemMax) return cudaErrorInvalidValue;
  const int nbuf = 2 * one <= kSmemMax ? 2 : 1;
  const float scale = (float)(1.0 / sqrt((double)d));  // fp32(1/sqrt(d)) (R10)
  const int n_items = B * A * ((S + QT - 1) / QT);
  const int per_sm = 1;  // ~240 registers x 256 threads: one resident CTA per SM
  const int grid = n_items < kNumSMs * per_sm ? n_items : kNumSMs * per_sm;
  launch_ex(attention_kernel<DP>, dim3(grid), dim3(256), nbuf * one, s, 0, qkv, ld, mask, B, S, A, d, hs, hm_rows, scale,
            ctx, ldc,
            nbuf);
  return cudaGetLastError();
}

}  // namespace

cudaError_t prepare_attention_kernels() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(attention_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(attention_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax)) != cudaSuccess) return e;
  return cudaFuncSetAttribute(attention_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
}

size_t attention_smem_bytes(int S, int d) {
  if (d <= 32) return attn_buf_bytes<32>(S);
  if (d <= 64) return attn_buf_bytes<64>(S);
  return attn_buf_bytes<128>(S);
}

cudaError_t launch_attention(const __half* qkv, int ldqkv, const int32_t* mask, int B, int S, int A, int d, int hs,
                             int hm_rows, __half* ctx, int ldctx, cudaStream_t s) {
  const int w = hs > d ? hs : d;
  if (w <= 32) return launch_dp<32>(qkv, ldqkv, mask, B, S, A, d, hs, hm_rows, ctx, ldctx, s);
  if (w <= 64) return launch_dp<64>(qkv, ldqkv, mask, B, S, A, d, hs, hm_rows, ctx, ldctx, s);
  return launch_dp<128>(qkv, ldqkv, mask, B, S, A, d, hs, hm_rows, ctx, ldctx, s);
}

}  // namespace ff
