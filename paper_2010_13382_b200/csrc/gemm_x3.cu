// gemm_x3.cu -- the fp32 linears of the importance scorer (importance.cu;
// SURVEY 8(f) NEXT-3) on the tcgen05 tensor cores.
//
// The scorer must keep fp32 accuracy (its scores are compared with the fp64
// oracle at 1e-4 of a score + 2e-5 of the layer maximum), so a
// single TF32 product (10-bit mantissa operands) is not enough.  Each operand
// is split into two TF32 numbers, x = hi + lo with hi = RN_tf32(x) and
// lo = RN_tf32(x - hi) (|x - hi - lo| <= 2^-22 |x|), and the product is
//   A B^T ~= Ah Bh^T + Ah Bl^T + Al Bh^T        ("3xTF32"; Al Bl^T ~ 2^-22 dropped)
// accumulated in fp32 in TMEM by kind::tf32 MMAs.  Both halves are exact TF32
// values, so the tensor core's treatment of the 13 low mantissa bits of an
// operand (ignored) does not matter.
//
// Operands: A [M x K] and B [N x K], both K-major (row pitch a multiple of 4
// floats: the split buffers are padded with zeros to K rounded up to 4).  The
// forward linear Y = X W^T takes B = W; the input-gradient dX = dY W takes
// B = W^T, split once when the scorer is finalized.
//
// Kernel: persistent, one CTA per SM, 128 x 128 output tiles; warp 0 issues
// the TMA loads of the four 16 KB operand tiles of a 32-float k-block (3-stage
// ring, 192 KB), warp 1 issues 12 MMAs per k-block (4 k-steps x 3 products)
// into one of two 128-column TMEM accumulators, warps 4-7 drain the other
// accumulator (tcgen05.ld -> +bias (+C) -> coalesced row stores through a
// 32 x 33 smem transpose per warp).
#include <algorithm>

#include "ff_kernels.h"
#include "ptx.cuh"

namespace ff {

namespace {

constexpr int X3_TM = 128, X3_TN = 128;
constexpr int X3_KE = 32;                 // fp32 elements per k-block (128 B rows)
constexpr int X3_STAGES = 3;
constexpr int X3_TILE = 128 * 128;        // bytes of one 128-row x 128 B operand tile
constexpr int X3_STAGE = 4 * X3_TILE;     // Ah, Al, Bh, Bl
constexpr int X3_EPI_OFF = X3_STAGES * X3_STAGE;
constexpr int X3_EPI_WARP = 32 * 33 * 4;  // one warp's transpose buffer
constexpr int X3_BAR_OFF = X3_EPI_OFF + 4 * X3_EPI_WARP;
constexpr int X3_SMEM = X3_BAR_OFF + 128 + 1024;  // + barriers + 1024-B alignment slack
constexpr int X3_THREADS = 256;

// kind::tf32 instruction descriptor: D f32 (bits 4-5 = 1), A / B TF32 (bits
// 7-9, 10-12 = 2), both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t x3_idesc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(X3_TN >> 3) << 17) | ((uint32_t)(X3_TM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

struct X3Params {
  float* C;
  const float* bias;
  int M, N, ldc, accumulate;
  int m_tiles, n_tiles, k_blocks;
};

__global__ void __launch_bounds__(X3_THREADS, 1)
    gemm_x3_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                   const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl, X3Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + X3_BAR_OFF);
  uint64_t* empty = full + X3_STAGES;
  uint64_t* tfull = empty + X3_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmAh);
    tma_prefetch(&tmAl);
    tma_prefetch(&tmBh);
    tma_prefetch(&tmBl);
    for (int s = 0; s < X3_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 2 * X3_TN);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = p.m_tiles * p.n_tiles;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mt = tile / p.n_tiles, nt = tile - mt * p.n_tiles;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * X3_STAGE;
          mbar_expect_tx(&full[stage], X3_STAGE);
          tma_load_2d(st, &tmAh, &full[stage], kb * X3_KE, mt * X3_TM, kEvictNormal);
          tma_load_2d(st + X3_TILE, &tmAl, &full[stage], kb * X3_KE, mt * X3_TM, kEvictNormal);
          tma_load_2d(st + 2 * X3_TILE, &tmBh, &full[stage], kb * X3_KE, nt * X3_TN, kEvictLast);
          tma_load_2d(st + 3 * X3_TILE, &tmBl, &full[stage], kb * X3_KE, nt * X3_TN, kEvictLast);
          if (++stage == X3_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = x3_idesc();
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * X3_TN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          uint8_t* st = smem + stage * X3_STAGE;
          const uint64_t ah = make_sw128_desc(st), al = make_sw128_desc(st + X3_TILE);
          const uint64_t bh = make_sw128_desc(st + 2 * X3_TILE), bl = make_sw128_desc(st + 3 * X3_TILE);
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 4 x 8 fp32 (32 B) of K; +2 = +32 B in the >>4 address field
            // small products first: the larger Ah Bh^T term then adds to an accumulator already
            // holding the corrections of this k-step
            mma_tf32(d_tmem, al + 2 * k, bh + 2 * k, idesc, (kb | k) != 0);
            mma_tf32(d_tmem, ah + 2 * k, bl + 2 * k, idesc, 1);
            mma_tf32(d_tmem, ah + 2 * k, bh + 2 * k, idesc, 1);
          }
          mma_commit(&empty[stage]);
          if (++stage == X3_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;  // TMEM lane quadrant = tile rows [32q, 32q + 32)
    float* buf = reinterpret_cast<float*>(smem + X3_EPI_OFF + (warp - 4) * X3_EPI_WARP);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int mt = tile / p.n_tiles, nt = tile - mt * p.n_tiles;
      const int row0 = mt * X3_TM + q * 32;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * X3_TN;
#pragma unroll 1
      for (int c = 0; c < X3_TN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tbase + c * 32, r);
        tmem_wait_ld();
        if (c == X3_TN / 32 - 1) {  // accumulator drained: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) buf[lane * 33 + j] = __uint_as_float(r[j]);
        __syncwarp();
        const int col = nt * X3_TN + c * 32 + lane;
        const bool cok = col < p.N;
        const float b = (p.bias != nullptr && cok) ? __ldg(p.bias + col) : 0.0f;
#pragma unroll 4
        for (int rr = 0; rr < 32; ++rr) {
          const int row = row0 + rr;
          if (row >= p.M) break;
          if (cok) {
            float v = buf[rr * 33 + lane] + b;
            float* dst = p.C + (size_t)row * p.ldc + col;
            if (p.accumulate) v += *dst;
            *dst = v;
          }
        }
        __syncwarp();
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * X3_TN);
  }
}

// hi / lo TF32 split of X [M x K] (pitch ldx) into [M x ldo] (ldo >= K, the
// columns [K, ldo) zero-filled).  One thread per 4 output columns.
__global__ void split_tf32_kernel(const float* __restrict__ X, int M, int K, int ldx, float* __restrict__ hi,
                                  float* __restrict__ lo, int ldo) {
  const int q4 = ldo >> 2;
  const size_t n = (size_t)M * q4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / q4), k0 = (int)(i - (size_t)r * q4) * 4;
    float x[4], h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x[j] = k0 + j < K ? X[(size_t)r * ldx + k0 + j] : 0.0f;
      h[j] = rna_tf32(x[j]);
      l[j] = rna_tf32(x[j] - h[j]);
    }
    *reinterpret_cast<float4*>(hi + (size_t)r * ldo + k0) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(lo + (size_t)r * ldo + k0) = make_float4(l[0], l[1], l[2], l[3]);
  }
}

// Transposed split: W [N x K] (pitch K) -> hi / lo [K x ldo] holding W^T
// (ldo >= N, columns [N, ldo) zero).  32 x 32 smem tiles.
__global__ void split_tf32_t_kernel(const float* __restrict__ W, int N, int K, float* __restrict__ hi,
                                    float* __restrict__ lo, int ldo) {
  __shared__ float t[32][33];
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    t[i][threadIdx.x] = (n < N && k < K) ? W[(size_t)n * K + k] : 0.0f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    if (k < K && n < ldo) {
      const float x = t[threadIdx.x][i];
      const float h = rna_tf32(x);
      hi[(size_t)k * ldo + n] = h;
      lo[(size_t)k * ldo + n] = rna_tf32(x - h);
    }
  }
}

bool encode_f32(CUtensorMap* map, const float* base, int rows, int ld, const char** err) {
  return make_operand_map(map, base, rows, ld, 4, (size_t)ld * 4, 128, err);
}

}  // namespace

cudaError_t launch_gemm_x3(const float* Ah, const float* Al, int lda, const float* Bh, const float* Bl, int ldb,
                           int M, int N, int K, const float* bias, float* C, int ldc, bool accumulate, cudaStream_t s,
                           const char** err) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if ((lda & 3) || (ldb & 3) || K > lda || K > ldb) {
    *err = "gemm_x3: operand pitch must be a multiple of 4 floats and >= K";
    return cudaErrorInvalidValue;
  }
  CUtensorMap ah, al, bh, bl;
  // the maps cover the K-padded width (zeros), so K rounds up to whole k-blocks
  if (!encode_f32(&ah, Ah, M, lda, err) || !encode_f32(&al, Al, M, lda, err) || !encode_f32(&bh, Bh, N, ldb, err) ||
      !encode_f32(&bl, Bl, N, ldb, err))
    return cudaErrorInvalidValue;
  static bool attr_set = false;  // per process; all devices are B200s
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, X3_SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  X3Params p{};
  p.C = C;
  p.bias = bias;
  p.M = M;
  p.N = N;
  p.ldc = ldc;
  p.accumulate = accumulate ? 1 : 0;
  p.m_tiles = (M + X3_TM - 1) / X3_TM;
  p.n_tiles = (N + X3_TN - 1) / X3_TN;
  p.k_blocks = (K + X3_KE - 1) / X3_KE;
  const int tiles = p.m_tiles * p.n_tiles;
  gemm_x3_kernel<<<std::min(tiles, kNumSMs), X3_THREADS, X3_SMEM, s>>>(ah, al, bh, bl, p);
  return cudaGetLastError();
}

cudaError_t launch_split_tf32(const float* X, int M, int K, int ldx, float* hi, float* lo, int ldo, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  const size_t n = (size_t)M * (ldo >> 2);
  const int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)kNumSMs * 8);
  split_tf32_kernel<<<blocks, 256, 0, s>>>(X, M, K, ldx, hi, lo, ldo);
  return cudaGetLastError();
}

cudaError_t launch_split_tf32_t(const float* W, int N, int K, float* hi, float* lo, int ldo, cudaStream_t s) {
  dim3 grid((ldo + 31) / 32, (K + 31) / 32);
  split_tf32_t_kernel<<<grid, dim3(32, 8), 0, s>>>(W, N, K, hi, lo, ldo);
  return cudaGetLastError();
}

}  // namespace ff
