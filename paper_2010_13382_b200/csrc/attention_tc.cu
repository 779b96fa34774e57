// attention_tc.cu -- fused masked-softmax attention on the 5th-gen tensor
// cores (tcgen05 + TMEM + TMA) for head_dim 64 and S <= 128: the shapes of the
// headline configs (P:135 multi-head attention node fusion;
// Q.K^T and P.V in floating point).
//
// One work item = (sequence b, head h < A'_l); 2 persistent CTAs per SM.
//   warp 0     TMA: Q, K, V head slices (128 rows x 64 fp16, 128B-swizzled)
//   warp 1     TMEM allocator + MMA issuer (one thread):
//                S[128 x 128] (TMEM, fp32) = Q . K^T        kind::f16, K-major A/B
//                O[128 x  64] (TMEM, fp32) = P . V          A = P (smem, K-major),
//                                                            B = V (smem, MN-major)
//   warps 2-5  softmax + epilogue, thread = query row (TMEM lane):
//                s = fp32(q.k) * fp32(1/sqrt(d)), masked keys -> -inf (R4)
//                p = exp(s - max) / sum  in fp32, P16 = R16(p)  (R9, normalized
//                before P.V), written to smem in the 128B-swizzled K-major
//                layout the MMA reads; ctx = R16(O) stored to HBM.
// Row max / sum are thread-local (one thread owns a whole score row), so the
// reduction order is a fixed sequential order.  Keys beyond S (S < 128) are
// masked; Q rows beyond S are computed and not stored.
#include "ff_kernels.h"
#include "ptx.cuh"

namespace ff {

namespace {

constexpr int kQ = 128;             // queries per item (TMEM lanes)
constexpr int kKeys = 128;          // keys (S <= 128)
constexpr int kD = 64;              // head_dim
constexpr int kTileBytes = 128 * 128;  // 128 rows x 128 B (64 fp16)
constexpr int kThreadsTC = 192;

struct SmemTC {
  static constexpr int Q = 0;
  static constexpr int K = Q + kTileBytes;
  static constexpr int V = K + kTileBytes;
  static constexpr int P = V + kTileBytes;          // 2 k-blocks of 64 keys, 128B-swizzled
  static constexpr int MASK = P + 2 * kTileBytes;   // kKeys floats
  static constexpr int BAR = MASK + kKeys * 4;
  static constexpr int TOTAL = BAR + 128 + 1024;    // barriers + alignment slack
};

// kind::f16, fp32 accumulate, M = 128; b_mn = 1 when B is MN-major.
__device__ __forceinline__ constexpr uint32_t idesc_f16(int N, int b_mn) {
  return (1u << 4) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// MN-major 128B-swizzled operand: atoms of 8 K-rows x 128 B, SBO = 1024 B
// between consecutive 8-row groups along K (one 64-element atom along N).
__device__ __forceinline__ uint64_t make_sw128_desc_mn(const void* smem_tile) {
  const uint64_t addr = smem_u32(smem_tile);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(kThreadsTC, 2)
    attention_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const int32_t* __restrict__ mask, int B, int S,
                        int A, float scale, __half* __restrict__ ctx, int ldc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SmemTC::BAR);
  uint64_t* kv_full = bar + 0;   // TMA -> MMA
  uint64_t* kv_empty = bar + 1;  // MMA (after P.V) -> TMA
  uint64_t* s_full = bar + 2;    // MMA1 -> softmax
  uint64_t* s_empty = bar + 3;   // softmax (S read) -> MMA1
  uint64_t* p_full = bar + 4;    // softmax (P written) -> MMA2
  uint64_t* o_full = bar + 5;    // MMA2 -> epilogue
  uint64_t* o_empty = bar + 6;   // epilogue (O read) -> MMA2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);
  float* sMask = reinterpret_cast<float*>(smem + SmemTC::MASK);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int D = A * kD;
  const int n_items = B * A;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(s_empty, 128);
    mbar_init(p_full, 128);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 128);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 256);  // S: columns [0,128), O: [128,192)
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // QKV / mask come from the previous kernel
  griddep_launch();

  if (warp == 0) {
    if (lane == 0) {
      uint32_t ph = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ph ^= 1) {
        const int b = item / A, h = item - b * A;
        mbar_wait(kv_empty, ph ^ 1);
        mbar_expect_tx(kv_full, 3 * kTileBytes);
        tma_load_2d(smem + SmemTC::Q, &tmQKV, kv_full, h * kD, b * S, kEvictFirst);
        tma_load_2d(smem + SmemTC::K, &tmQKV, kv_full, D + h * kD, b * S, kEvictFirst);
        tma_load_2d(smem + SmemTC::V, &tmQKV, kv_full, 2 * D + h * kD, b * S, kEvictFirst);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id1 = idesc_f16(kKeys, 0);  // S = Q K^T: N = 128 keys
      constexpr uint32_t id2 = idesc_f16(kD, 1);     // O = P V:   N = 64, V MN-major
      uint32_t ph = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ph ^= 1) {
        mbar_wait(kv_full, ph);
        mbar_wait(s_empty, ph ^ 1);
        tc_fence_after();
        const uint64_t qd = make_sw128_desc(smem + SmemTC::Q), kd = make_sw128_desc(smem + SmemTC::K);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) mma_f16(tmem, qd + 2 * k, kd + 2 * k, id1, k != 0);
        mma_commit(s_full);
        mbar_wait(p_full, ph);
        mbar_wait(o_empty, ph ^ 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k) {
          // A = P: k-block k/4 (64 keys), +32 B per 16 keys inside the 128B row
          const uint64_t pd = make_sw128_desc(smem + SmemTC::P + (k >> 2) * kTileBytes) + 2 * (k & 3);
          // B = V (MN-major): 16 keys = two 8-row groups = 2048 B
          const uint64_t vd = make_sw128_desc_mn(smem + SmemTC::V + k * 2048);
          mma_f16(tmem + 128, pd, vd, id2, k != 0);
        }
        mma_commit(o_full);
        mma_commit(kv_empty);  // Q/K/V (and P) smem free once these MMAs complete
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quadrant
    const int r = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    constexpr float kLog2e = 1.4426950408889634f;
    uint32_t ph = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ph ^= 1) {
      const int b = item / A, h = item - b * A;
      // key mask of this sequence (keys >= S masked); consumed after s_full
      const int tid = threadIdx.x - 64;
      // sMask is rewritten per item: the previous item's softmax (same threads)
      // finished reading it before p_full, so a named barrier suffices
      asm volatile("bar.sync 1, 128;" ::: "memory");
      sMask[tid] = (tid < S && __ldg(mask + (size_t)b * S + tid) != 0) ? 0.0f : -INFINITY;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      mbar_wait(s_full, ph);
      tc_fence_after();
      uint32_t raw[kKeys / 32][32];
#pragma unroll
      for (int c = 0; c < kKeys / 32; ++c) tmem_ld32(trow + c * 32, raw[c]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(s_empty);
      float s[kKeys];
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < kKeys; ++j) {
        s[j] = __fmul_rn(__uint_as_float(raw[j >> 5][j & 31]), scale) + sMask[j];
        mx = fmaxf(mx, s[j]);
      }
      float l = 0.0f;
#pragma unroll
      for (int j = 0; j < kKeys; ++j) {
        s[j] = ex2f((s[j] - mx) * kLog2e);
        l += s[j];
      }
      const float inv = __frcp_rn(l);
      // P16 = R16(p) into the K-major 128B-swizzled tile: k-block kb holds keys
      // [64kb, 64kb+64) of row r; 16B chunk c at (c ^ (r & 7)).
      uint8_t* prow = smem + SmemTC::P + r * 128;
#pragma unroll
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int j = kb * 64 + c * 8;
          uint4 v;
          v.x = pack_half2(s[j] * inv, s[j + 1] * inv);
          v.y = pack_half2(s[j + 2] * inv, s[j + 3] * inv);
          v.z = pack_half2(s[j + 4] * inv, s[j + 5] * inv);
          v.w = pack_half2(s[j + 6] * inv, s[j + 7] * inv);
          *reinterpret_cast<uint4*>(prow + kb * kTileBytes + ((c ^ (r & 7)) << 4)) = v;
        }
      fence_async_smem();
      mbar_arrive(p_full);
      // epilogue: ctx row = R16(O row)
      mbar_wait(o_full, ph);
      tc_fence_after();
      uint32_t o[64];
      tmem_ld32(trow + 128, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
      tmem_ld32(trow + 160, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
      tmem_wait_ld();  // (o[] is a plain register array: both loads land before use)
      tc_fence_before();
      mbar_arrive(o_empty);
      if (r < S) {
        __half* dst = ctx + ((size_t)b * S + r) * ldc + h * kD;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 v;
          v.x = pack_half2(__uint_as_float(o[c * 8 + 0]), __uint_as_float(o[c * 8 + 1]));
          v.y = pack_half2(__uint_as_float(o[c * 8 + 2]), __uint_as_float(o[c * 8 + 3]));
          v.z = pack_half2(__uint_as_float(o[c * 8 + 4]), __uint_as_float(o[c * 8 + 5]));
          v.w = pack_half2(__uint_as_float(o[c * 8 + 6]), __uint_as_float(o[c * 8 + 7]));
          *reinterpret_cast<uint4*>(dst + c * 8) = v;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

}  // namespace

bool attention_tc_supported(int S, int d, int ldqkv, int ldctx) {
  return d == kD && S >= 1 && S <= kKeys && (ldqkv % 8) == 0 && (ldctx % 8) == 0;
}

bool plan_attention_tc(CUtensorMap* map, const void* qkv, int M_rows, int ldqkv, const char** err) {
  // [M_rows x ldqkv] fp16, 64-column x 128-row boxes, 128B swizzle
  return make_operand_map(map, qkv, M_rows, ldqkv, 2, (size_t)ldqkv * 2, 128, err);
}

cudaError_t prepare_attention_tc_kernel() {
  return cudaFuncSetAttribute(attention_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemTC::TOTAL);
}

cudaError_t launch_attention_tc(const CUtensorMap& map, const int32_t* mask, int B, int S, int A, __half* ctx,
                                int ldctx, cudaStream_t s) {
  const int n_items = B * A;
  const int grid = n_items < 2 * kNumSMs ? n_items : 2 * kNumSMs;
  const float scale = (float)(1.0 / sqrt((double)kD));
  launch_ex(attention_tc_kernel, dim3(grid), dim3(kThreadsTC), SmemTC::TOTAL, s, 0, map, mask, B, S, A, scale, ctx,
            ldctx);
  return cudaGetLastError();
}

}  // namespace ff
