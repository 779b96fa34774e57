// gemm_x3.cu -- the fp32 linears of the importance scorer (importance.cu;
// SURVEY 8(f) NEXT-3) on the tcgen05 tensor cores.
//
// The scorer must keep fp32 accuracy (its scores are compared with the fp64
// oracle at 1e-4 of a score + 2e-5 of the layer maximum), so one
// low-precision product is not enough.  Each operand row r is scaled by a
// power of two 2^-e_r (its largest magnitude maps below 2^14, exact) and split
// into two fp16 numbers, y = x 2^-e_r = hi + lo with hi = RN_fp16(y) and
// lo = RN_fp16(y - hi): 22 significant bits for every element within 2^-17 of
// the row's maximum (smaller ones keep an absolute error <= 2^-39 of it).  The
// product is
//   A B^T ~= 2^(e_a + e_b) (Ah Bh^T + Ah Bl^T + Al Bh^T)     ("3xFP16"; Al Bl^T ~ 2^-22 dropped)
// with fp32 accumulation by kind::f16 MMAs (11-bit x 11-bit products are exact
// in fp32).  Same precision as a hi / lo TF32 split (3xTF32), at half the
// operand bytes and twice the MMA rate (measured: the 3xTF32 form of this
// kernel ran at 0.44 of its peak, bound by operand feed).
//
// The tensor core's fp32 accumulation is not IEEE round-to-nearest (measured
// with 3xTF32: one TMEM accumulator over K = 3072 left errors ~20x the SIMT
// SGEMM's), so the K loop is cut into chunks of `kc` k-blocks (default 2 =
// 128 of K): each chunk accumulates into its own TMEM slot (4-slot ring, 128
// columns each), and the epilogue warps add the chunk results in registers
// with IEEE fp32 adds.
//
// Operands: A [M x K] and B [N x K] fp16 hi / lo, both K-major (row pitch a
// multiple of 8 halves, zero-padded beyond K), with per-row fp32 scales
// 2^e.  The forward linear Y = X W^T takes B = W; the input-gradient
// dX = dY W takes B = W^T, both split once when the scorer is finalized.
//
// Kernel: persistent, one CTA per SM, 128 x 128 output tiles; warp 0 issues
// the TMA loads of the four 16 KB operand tiles of a 64-element k-block
// (3-stage ring, 192 KB), warp 1 issues 12 MMAs per k-block (4 k-steps x 3
// products) into the next free TMEM slot, warps 4-7 add each finished slot
// into their rows' fp32 sums (thread = row, 128 registers) and, after the last
// chunk of a tile, store sum * 2^(e_a + e_b) + bias (+ C) with coalesced row
// stores through a 32 x 33 smem transpose per warp.
#include <algorithm>

#include "ff_kernels.h"
#include "ptx.cuh"

namespace ff {

namespace {

constexpr int X3_TM = 128, X3_TN = 128;
constexpr int X3_KE = 64;                 // fp16 elements per k-block (128 B rows)
constexpr int X3_STAGES = 3;
constexpr int X3_TILE = 128 * 128;        // bytes of one 128-row x 128 B operand tile
constexpr int X3_STAGE = 4 * X3_TILE;     // Ah, Al, Bh, Bl
constexpr int X3_EPI_OFF = X3_STAGES * X3_STAGE;
constexpr int X3_EPI_WARP = 32 * 33 * 4;  // one warp's transpose buffer
constexpr int X3_BAR_OFF = X3_EPI_OFF + 4 * X3_EPI_WARP;
constexpr int X3_SMEM = X3_BAR_OFF + 128 + 1024;  // + barriers + 1024-B alignment slack
constexpr int X3_THREADS = 256;

// kind::f16 instruction descriptor: D f32 (bits 4-5 = 1), A / B fp16 (bits
// 7-9, 10-12 = 0), both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t x3_idesc() {
  return (1u << 4) | ((uint32_t)(X3_TN >> 3) << 17) | ((uint32_t)(X3_TM >> 4) << 24);
}

struct X3Params {
  float* C;
  const float* bias;
  const float* sa;  // per-row scales 2^e of A [M] and of B [N]
  const float* sb;
  int M, N, ldc, accumulate;
  int m_tiles, n_tiles, k_blocks;
  int kc;  // k-blocks per TMEM accumulation chunk
  // split-K (wave quantization of few-tile shapes): unit u = (ks, tile) covers
  // k-blocks [ks * kbps, (ks + 1) * kbps); with splits > 1 each unit writes its
  // plain partial sum to ws[ks] ([M x N]) and x3_splitk_reduce adds them.
  int splits, kbps;
  float* ws;
};
struct X3Unit {
  int mt, nt, ks, kb0, kb1;
};
__device__ __forceinline__ X3Unit x3_unit(const X3Params& p, int u) {
  X3Unit w;
  const int tiles = p.m_tiles * p.n_tiles;
  w.ks = u / tiles;
  const int t = u - w.ks * tiles;
  w.mt = t / p.n_tiles;
  w.nt = t - w.mt * p.n_tiles;
  w.kb0 = w.ks * p.kbps;
  w.kb1 = min(p.k_blocks, w.kb0 + p.kbps);
  return w;
}
constexpr int X3_SLOTS = 4;  // TMEM accumulator ring: 4 x 128 columns = all 512

__global__ void __launch_bounds__(X3_THREADS, 1)
    gemm_x3_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                   const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl, X3Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + X3_BAR_OFF);
  uint64_t* empty = full + X3_STAGES;
  uint64_t* tfull = empty + X3_STAGES;
  uint64_t* tempty = tfull + X3_SLOTS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + X3_SLOTS);
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
    for (int a = 0; a < X3_SLOTS; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, X3_SLOTS * X3_TN);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_units = p.m_tiles * p.n_tiles * p.splits;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const X3Unit w = x3_unit(p, u);
        const int mt = w.mt, nt = w.nt;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
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
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const X3Unit w = x3_unit(p, u);
        uint32_t d_tmem = 0;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          const int kin = (kb - w.kb0) % p.kc;  // k-block index inside its chunk
          if (kin == 0) {             // a new chunk: next TMEM slot
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            d_tmem = tmem_base + acc * X3_TN;
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          uint8_t* st = smem + stage * X3_STAGE;
          const uint64_t ah = make_sw128_desc(st), al = make_sw128_desc(st + X3_TILE);
          const uint64_t bh = make_sw128_desc(st + 2 * X3_TILE), bl = make_sw128_desc(st + 3 * X3_TILE);
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 4 x 16 fp16 (32 B) of K; +2 = +32 B in the >>4 address field
            // small products first: the larger Ah Bh^T term then adds to an accumulator already
            // holding the corrections of this k-step
            mma_f16(d_tmem, al + 2 * k, bh + 2 * k, idesc, (kin | k) != 0);
            mma_f16(d_tmem, ah + 2 * k, bl + 2 * k, idesc, 1);
            mma_f16(d_tmem, ah + 2 * k, bh + 2 * k, idesc, 1);
          }
          mma_commit(&empty[stage]);
          if (++stage == X3_STAGES) {
            stage = 0;
            phase ^= 1;
          }
          if (kin == p.kc - 1 || kb == w.kb1 - 1) {  // chunk complete
            mma_commit(&tfull[acc]);
            if (++acc == X3_SLOTS) {
              acc = 0;
              acc_phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;  // TMEM lane quadrant = tile rows [32q, 32q + 32)
    float* buf = reinterpret_cast<float*>(smem + X3_EPI_OFF + (warp - 4) * X3_EPI_WARP);
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool part = p.splits > 1;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      const X3Unit w = x3_unit(p, u);
      const int nchunks = (w.kb1 - w.kb0 + p.kc - 1) / p.kc;
      const int mt = w.mt, nt = w.nt;
      const int row0 = mt * X3_TM + q * 32;
      // partial sums (split-K) go to ws[ks] without bias / accumulate
      float* const out = part ? p.ws + (size_t)w.ks * p.M * p.N : p.C;
      const int ldo = part ? p.N : p.ldc;
      float sum[X3_TN];
#pragma unroll
      for (int j = 0; j < X3_TN; ++j) sum[j] = 0.0f;
      for (int ch = 0; ch < nchunks; ++ch) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * X3_TN;
#pragma unroll
        for (int c = 0; c < X3_TN / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tbase + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[c * 32 + j] += __uint_as_float(r[j]);
        }
        tc_fence_before();  // slot drained: hand it back to the MMA warp
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == X3_SLOTS) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      // undo the operand scaling: this thread's row scale now, the column's at the store
      const float srow = row0 + lane < p.M ? __ldg(p.sa + row0 + lane) : 0.0f;
#pragma unroll
      for (int c = 0; c < X3_TN / 32; ++c) {
#pragma unroll
        for (int j = 0; j < 32; ++j) buf[lane * 33 + j] = sum[c * 32 + j] * srow;
        __syncwarp();
        const int col = nt * X3_TN + c * 32 + lane;
        const bool cok = col < p.N;
        const float b = (!part && p.bias != nullptr && cok) ? __ldg(p.bias + col) : 0.0f;
        const float scol = cok ? __ldg(p.sb + col) : 0.0f;
        float* dst = out + (size_t)row0 * ldo + col;
        const int nrows = min(32, p.M - row0);
        if (p.accumulate && !part) {  // 16 loads of C in flight before the stores
#pragma unroll
          for (int h = 0; h < 32; h += 16) {
            float cv[16];
#pragma unroll
            for (int rr = 0; rr < 16; ++rr)
              cv[rr] = (cok && h + rr < nrows) ? dst[(size_t)(h + rr) * ldo] : 0.0f;
#pragma unroll
            for (int rr = 0; rr < 16; ++rr)
              if (cok && h + rr < nrows) dst[(size_t)(h + rr) * ldo] = buf[(h + rr) * 33 + lane] * scol + b + cv[rr];
          }
        } else {
#pragma unroll
          for (int rr = 0; rr < 32; ++rr)
            if (cok && rr < nrows) dst[(size_t)rr * ldo] = buf[rr * 33 + lane] * scol + b;
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, X3_SLOTS * X3_TN);
  }
}

// Row-scaled fp16 hi / lo split of X [M x K] (pitch ldx) into [M x ldo]
// (ldo even, >= K; columns [K, ldo) zero): one warp per row finds max |x|,
// picks 2^-e with max |x| 2^-e < 2^14 (e = 0 for an all-zero row), then
// writes hi = RN_fp16(y), lo = RN_fp16(y - hi) of y = x 2^-e and scale[r] = 2^e.
__global__ void split_x3_kernel(const float* __restrict__ X, int M, int K, int ldx, __half* __restrict__ hi,
                                __half* __restrict__ lo, int ldo, float* __restrict__ scale) {
  const int r = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (r >= M) return;
  const float* x = X + (size_t)r * ldx;
  float mx = 0.0f;
  for (int k = lane; k < K; k += 32) mx = fmaxf(mx, fabsf(x[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 14;  // all-zero row: scale 1
  if (mx > 0.0f) {
    frexpf(mx, &e);  // mx < 2^e
    e = max(e, -100);  // keeps 2^(14 - e) finite; such rows are ~0 anyway
  }
  const float inv = ldexpf(1.0f, 14 - e);
  if (lane == 0) scale[r] = ldexpf(1.0f, e - 14);
  __half2* h2 = reinterpret_cast<__half2*>(hi + (size_t)r * ldo);
  __half2* l2 = reinterpret_cast<__half2*>(lo + (size_t)r * ldo);
  for (int k = 2 * lane; k < ldo; k += 64) {
    const float y0 = k < K ? x[k] * inv : 0.0f, y1 = k + 1 < K ? x[k + 1] * inv : 0.0f;
    const __half2 h = __floats2half2_rn(y0, y1);
    const float2 f = __half22float2(h);
    h2[k >> 1] = h;
    l2[k >> 1] = __floats2half2_rn(y0 - f.x, y1 - f.y);
  }
}

// W [N x K] (pitch K) -> WT [K x N] (pitch N), 32 x 32 smem tiles.
__global__ void transpose_f32_kernel(const float* __restrict__ W, int N, int K, float* __restrict__ WT) {
  __shared__ float t[32][33];
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    t[i][threadIdx.x] = (n < N && k < K) ? W[(size_t)n * K + k] : 0.0f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    if (k < K && n < N) WT[(size_t)k * N + n] = t[threadIdx.x][i];
  }
}

// C = sum_ks ws[ks] + bias (+ C), partials added in ks order (deterministic).
// One thread per 4 consecutive columns (N % 4 == 0 and ldc % 4 == 0: float4
// accesses; the launcher checks alignment), else one per element.
template <bool V4>
__global__ void x3_splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N,
                                        const float* __restrict__ bias, float* C, int ldc, int accumulate) {
  constexpr int W = V4 ? 4 : 1;
  const int nq = N / W;
  const size_t n = (size_t)M * nq, plane = (size_t)M * N, stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int r = (int)(i / nq), c = (int)(i - (size_t)r * nq) * W;
    const size_t o = (size_t)r * N + c;
    float* dst = C + (size_t)r * ldc + c;
    if constexpr (V4) {
      float4 v = *reinterpret_cast<const float4*>(ws + o);
      for (int k = 1; k < splits; ++k) {
        const float4 w = *reinterpret_cast<const float4*>(ws + (size_t)k * plane + o);
        v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
      }
      if (bias != nullptr) {
        const float4 b = *reinterpret_cast<const float4*>(bias + c);
        v.x += b.x; v.y += b.y; v.z += b.z; v.w += b.w;
      }
      if (accumulate) {
        const float4 d = *reinterpret_cast<const float4*>(dst);
        v.x += d.x; v.y += d.y; v.z += d.z; v.w += d.w;
      }
      *reinterpret_cast<float4*>(dst) = v;
    } else {
      float v = ws[o];
      for (int k = 1; k < splits; ++k) v += ws[(size_t)k * plane + o];
      if (bias != nullptr) v += __ldg(bias + c);
      if (accumulate) v += *dst;
      *dst = v;
    }
  }
}

// Split count for the K loop: the wave makespan of 148 persistent CTAs, in
// k-block times, plus ~3 k-blocks of fill / drain per unit and the partial-sum
// traffic of the reduction (S + 2 passes over M x N fp32 at ~5 TB/s against
// ~0.75 us per k-block); at most `cap` partial buffers fit the workspace.
int pick_splits(int tiles, int k_blocks, size_t MN, int cap) {
  int best = 1;
  double best_cost = 1e30;
  for (int S = 1; S <= std::min(4, cap); ++S) {
    if (S > 1 && k_blocks / S < 4) break;
    const int kbps = (k_blocks + S - 1) / S;
    const int waves = (tiles * S + kNumSMs - 1) / kNumSMs;
    double cost = (double)waves * (kbps + 3);
    if (S > 1) cost += (double)(S + 2) * MN * 4 / 5e12 / 0.75e-6;
    if (cost < best_cost * 0.97) {
      best_cost = cost;
      best = S;
    }
  }
  return best;
}

}  // namespace

cudaError_t launch_gemm_x3(const __half* Ah, const __half* Al, const float* sa, int lda, const __half* Bh,
                           const __half* Bl, const float* sb, int ldb, int M, int N, int K, const float* bias, float* C,
                           int ldc, bool accumulate, cudaStream_t s, const char** err, int kc, float* ws,
                           size_t ws_floats) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (kc < 1) {
    *err = "gemm_x3: kc must be >= 1";
    return cudaErrorInvalidValue;
  }
  if ((lda & 7) || (ldb & 7) || K > lda || K > ldb) {
    *err = "gemm_x3: operand pitch must be a multiple of 8 halves and >= K";
    return cudaErrorInvalidValue;
  }
  // the maps cover the K-padded width (zeros), so K rounds up to whole k-blocks
  CUtensorMap ah, al, bh, bl;
  if (!make_operand_map(&ah, Ah, M, lda, 2, (size_t)lda * 2, 128, err) ||
      !make_operand_map(&al, Al, M, lda, 2, (size_t)lda * 2, 128, err) ||
      !make_operand_map(&bh, Bh, N, ldb, 2, (size_t)ldb * 2, 128, err) ||
      !make_operand_map(&bl, Bl, N, ldb, 2, (size_t)ldb * 2, 128, err))
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
  p.sa = sa;
  p.sb = sb;
  p.M = M;
  p.N = N;
  p.ldc = ldc;
  p.accumulate = accumulate ? 1 : 0;
  p.m_tiles = (M + X3_TM - 1) / X3_TM;
  p.n_tiles = (N + X3_TN - 1) / X3_TN;
  p.k_blocks = std::max(1, (K + X3_KE - 1) / X3_KE);
  p.kc = kc;
  const int tiles = p.m_tiles * p.n_tiles;
  const size_t MN = (size_t)M * N;
  const int cap = ws != nullptr ? (int)std::min<size_t>(4, ws_floats / MN) : 1;
  p.splits = pick_splits(tiles, p.k_blocks, MN, std::max(1, cap));
  p.kbps = (p.k_blocks + p.splits - 1) / p.splits;
  p.splits = (p.k_blocks + p.kbps - 1) / p.kbps;  // no empty split
  p.ws = ws;
  const int units = tiles * p.splits;
  gemm_x3_kernel<<<std::min(units, kNumSMs), X3_THREADS, X3_SMEM, s>>>(ah, al, bh, bl, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || p.splits == 1) return e;
  const bool v4 = (N % 4) == 0 && (ldc % 4) == 0 && ((reinterpret_cast<uintptr_t>(C) | reinterpret_cast<uintptr_t>(ws) |
                                                      reinterpret_cast<uintptr_t>(bias)) & 15) == 0;
  const size_t work = v4 ? MN / 4 : MN;
  const int blocks = (int)std::min<size_t>((work + 255) / 256, (size_t)kNumSMs * 8);
  if (v4) x3_splitk_reduce_kernel<true><<<blocks, 256, 0, s>>>(ws, p.splits, M, N, bias, C, ldc, accumulate ? 1 : 0);
  else x3_splitk_reduce_kernel<false><<<blocks, 256, 0, s>>>(ws, p.splits, M, N, bias, C, ldc, accumulate ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_split_x3(const float* X, int M, int K, int ldx, __half* hi, __half* lo, int ldo, float* scale,
                            cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  split_x3_kernel<<<(M + 7) / 8, 256, 0, s>>>(X, M, K, ldx, hi, lo, ldo, scale);
  return cudaGetLastError();
}

cudaError_t launch_transpose_f32(const float* W, int N, int K, float* WT, cudaStream_t s) {
  if (N <= 0 || K <= 0) return cudaSuccess;
  transpose_f32_kernel<<<dim3((N + 31) / 32, (K + 31) / 32), dim3(32, 8), 0, s>>>(W, N, K, WT);
  return cudaGetLastError();
}

}  // namespace ff
