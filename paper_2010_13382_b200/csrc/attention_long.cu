// attention_long.cu -- fused masked-softmax attention on the tcgen05 tensor
// cores for 128 < S <= 512 and head_dim 64: the long-passage shapes of the
// SuperGLUE configs (C4 BERT-base at S 512, C5 at S 256; "ReCoRD's long
// passages"; SURVEY 8(a) a3, P:104 Q.K^T and P.V in floating point).
//
// Work unit = (sequence b, query block of 128 rows, head h); one persistent
// CTA per SM takes a contiguous range of units (heads fastest, so its units
// share the sequence's key mask and the K / V tiles of a head stay in L2
// across the query blocks).  Per unit, with KC =
// ceil(S / 128) key chunks:
//   warp 0     TMA: Q block, K_0..K_{KC-1}, V_0..V_{KC-1} (128 rows x 64 fp16,
//              128B swizzle) through a ring of 16 KB tile slots, running ahead
//              into the next units
//   warp 1     TMEM allocator + MMA issuer (one thread):
//                S_c = Q . K_c^T     (fp32, TMEM columns [128 c, 128 c + 128))
//                O  += P_c . V_c     (fp32; KC = 4: columns [0, 64), reusing
//                                    S_0 once it has been read; KC = 2: [256, 320))
//   warps 2-17 softmax + epilogue: four warps per TMEM lane quadrant (= 32
//              query rows), each owning one quarter (32 keys) of every chunk
//              (16 warps hide the MUFU / TMEM latencies of the serial passes):
//                pass 1: s = RN(raw * fp32(1/sqrt d)) (+ key mask -inf), row max
//                pass 2: e = exp(s - max) (ex2.approx of (s - max) log2 e), the
//                        row sum l; e written back over S in TMEM
//                pass 3: p = e / l (IEEE quotient, Markstein), P16 = R16(p)
//                        into a double-buffered 128B-swizzled K-major P tile
//                epilogue: ctx = R16(O) (fp16 rows)
// This is the oracle's order (DESIGN R9: max over all keys, then e, l, then
// normalise and round P to fp16 before P.V) -- no online rescaling -- and one
// exp per score.  TMEM reads are cheap (~900 B/clk/SM, tools/micro/tmem_bw.cu)
// so S is re-read per pass instead of being held in registers.
// int8 layers store fp16 ctx here; their Q8row requant runs as quant_rows.
#include "ff_kernels.h"
#include "ptx.cuh"
#include "quant.cuh"

namespace ff {

namespace {

constexpr int kLQ = 128;               // query rows per unit (TMEM lanes)
constexpr int kLD = 64;                // head_dim
constexpr int kLTile = 128 * 128;      // one 128-row x 64-column fp16 tile, 128B swizzle
constexpr int kLSlots = 8;             // ring of tile slots (Q, K_c, V_c of consecutive units)
constexpr int kLSoftWarps = 16;
constexpr int kLThreads = 64 + 32 * kLSoftWarps;
constexpr int kLMaxKeys = 512;

struct SmemL {
  static constexpr int RING = 0;                              // [kLSlots] tiles
  static constexpr int P = RING + kLSlots * kLTile;           // P[2]: 2 k-blocks of 64 keys each
  static constexpr int MASK = P + 2 * 2 * kLTile;             // kLMaxKeys floats
  static constexpr int RED = MASK + kLMaxKeys * 4;            // [2][4][128] floats: max, sum per quarter
  static constexpr int BAR = RED + 2 * 4 * kLQ * 4;
  static constexpr int TOTAL = BAR + 256 + 1024;
  static_assert(TOTAL <= 227 * 1024, "smem budget");
};

__device__ __forceinline__ constexpr uint32_t idesc_l(int N, int b_mn) {
  return (1u << 4) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ uint64_t sw128_desc_mn(const void* smem_tile) {
  const uint64_t addr = smem_u32(smem_tile);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ float ex2l(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Debug timeline (ff_debug_set_trace which = 4): %globaltimer of event e for
// the CTA's unit k at trace[(cta * 32 + k) * 8 + e]: 0 Q load issued, 1 MMA saw
// t_free, 2 S committed, 3 softmax saw s_full, 4 pass 1 done, 5 pass 2 done,
// 6 last P chunk published, 7 O read (epilogue).
__device__ __forceinline__ void ltrace(unsigned long long* tr, uint32_t k, int e) {
  if (tr != nullptr && k < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    tr[((size_t)blockIdx.x * 32 + k) * 8 + e] = t;
  }
}

struct Unit {
  int b, qb, h;
};
__device__ __forceinline__ Unit unit_of(int u, int nqb, int A) {
  Unit x;
  x.h = u % A;
  const int t = u / A;
  x.qb = t % nqb;
  x.b = t / nqb;
  return x;
}

template <int KC>
__global__ void __launch_bounds__(kLThreads, 1)
    attention_long_kernel(const __grid_constant__ CUtensorMap tmQKV, const int32_t* __restrict__ mask, int B, int S,
                          int A, int hm_rows, float scale, __half* __restrict__ ctx, int ldc,
                          unsigned long long* __restrict__ trace) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SmemL::BAR);
  uint64_t* full = bar;                    // [kLSlots] TMA -> MMA
  uint64_t* empty = bar + kLSlots;         // [kLSlots] MMA -> TMA
  uint64_t* s_full = bar + 2 * kLSlots;    // MMA (all S chunks) -> softmax
  uint64_t* p_full = s_full + 1;           // [2] softmax (P chunk written) -> MMA
  uint64_t* p_empty = p_full + 2;          // [2] MMA (P chunk consumed) -> softmax
  uint64_t* o_full = p_empty + 2;          // MMA (last P.V) -> epilogue
  uint64_t* t_free = o_full + 1;           // epilogue (O read, all of S consumed) -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_free + 1);
  float* sMask = reinterpret_cast<float*>(smem + SmemL::MASK);
  float* sRed = reinterpret_cast<float*>(smem + SmemL::RED);
  constexpr uint32_t kO = KC == 4 ? 0u : (uint32_t)(KC * 128);  // O columns
  constexpr int kSoft = 32 * kLSoftWarps;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int D = A * kLD;
  const int nqb = (S + kLQ - 1) / kLQ;
  const int n_units = B * nqb * A;
  const int per = (n_units + gridDim.x - 1) / gridDim.x;  // contiguous units of this CTA
  const int u_begin = min(n_units, (int)blockIdx.x * per), u_end = min(n_units, u_begin + per);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    for (int i = 0; i < kLSlots; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    mbar_init(s_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(p_full + i, kSoft);
      mbar_init(p_empty + i, 1);
    }
    mbar_init(o_full, 1);
    mbar_init(t_free, kSoft);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
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
      uint32_t cnt = 0;
      auto load = [&](int col, int row) {
        const int slot = cnt % kLSlots;
        mbar_wait(empty + slot, ((cnt / kLSlots) & 1) ^ 1);
        mbar_expect_tx(full + slot, kLTile);
        tma_load_2d(smem + SmemL::RING + slot * kLTile, &tmQKV, full + slot, col, row, kEvictFirst);
        ++cnt;
      };
      for (int u = u_begin; u < u_end; ++u) {
        const Unit x = unit_of(u, nqb, A);
        const int row0 = x.b * S;
        ltrace(trace, (uint32_t)(u - u_begin), 0);
        if (hm_rows > 0) {  // head-major QKV: contiguous 128 x 64 blocks
          load(0, x.h * hm_rows + row0 + x.qb * kLQ);
          for (int c = 0; c < KC; ++c) load(0, (A + x.h) * hm_rows + row0 + c * 128);
          for (int c = 0; c < KC; ++c) load(0, (2 * A + x.h) * hm_rows + row0 + c * 128);
        } else {
          load(x.h * kLD, row0 + x.qb * kLQ);
          for (int c = 0; c < KC; ++c) load(D + x.h * kLD, row0 + c * 128);
          for (int c = 0; c < KC; ++c) load(2 * D + x.h * kLD, row0 + c * 128);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id1 = idesc_l(128, 0);   // S_c = Q K_c^T: N = 128 keys
      constexpr uint32_t id2 = idesc_l(kLD, 1);   // O += P_c V_c: N = 64, V MN-major
      uint32_t cnt = 0, g = 0, n = 0;
      for (int u = u_begin; u < u_end; ++u, ++n) {
        // TMEM (S chunks, O) free once the previous unit's epilogue read O
        mbar_wait(t_free, (n & 1) ^ 1);
        ltrace(trace, n, 1);
        tc_fence_after();
        const int qslot = cnt % kLSlots;
        mbar_wait(full + qslot, (cnt / kLSlots) & 1);
        ++cnt;
        const uint64_t qd = make_sw128_desc(smem + SmemL::RING + qslot * kLTile);
        for (int c = 0; c < KC; ++c) {
          const int ks = cnt % kLSlots;
          mbar_wait(full + ks, (cnt / kLSlots) & 1);
          ++cnt;
          tc_fence_after();
          const uint64_t kd = make_sw128_desc(smem + SmemL::RING + ks * kLTile);
#pragma unroll
          for (int k = 0; k < kLD / 16; ++k) mma_f16(tmem + c * 128, qd + 2 * k, kd + 2 * k, id1, k != 0);
          mma_commit(empty + ks);
        }
        mma_commit(empty + qslot);
        mma_commit(s_full);
        ltrace(trace, n, 2);
        for (int c = 0; c < KC; ++c, ++g) {
          const int vs = cnt % kLSlots;
          mbar_wait(full + vs, (cnt / kLSlots) & 1);
          ++cnt;
          mbar_wait(p_full + (g & 1), (g >> 1) & 1);
          tc_fence_after();
          uint8_t* P = smem + SmemL::P + (g & 1) * 2 * kLTile;
          uint8_t* V = smem + SmemL::RING + vs * kLTile;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t pd = make_sw128_desc(P + (k >> 2) * kLTile) + 2 * (k & 3);
            const uint64_t vd = sw128_desc_mn(V + k * 2048);
            mma_f16(tmem + kO, pd, vd, id2, (c | k) != 0);
          }
          mma_commit(empty + vs);
          mma_commit(p_empty + (g & 1));
        }
        mma_commit(o_full);
      }
    }
  } else {
    const int q = warp & 3;              // TMEM lane quadrant
    const int qt = (warp - 2) >> 2;      // keys [32 qt, +32) of every chunk; O columns [16 qt, +16)
    const int r = q * 32 + lane;
    const int tid = threadIdx.x - 64;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    float* redMax = sRed;
    float* redSum = sRed + 4 * kLQ;
    const int quad_bar = 2 + q;  // the four warps sharing TMEM lane quadrant q
    auto quad_sync = [quad_bar]() { asm volatile("bar.sync %0, 128;" ::"r"(quad_bar) : "memory"); };
    auto soft_sync = []() { asm volatile("bar.sync 1, %0;" ::"n"(kSoft) : "memory"); };
    const float2 cd2 = make_float2(scale, scale);
    const float2 l2e = make_float2(1.4426950408889634f, 1.4426950408889634f);
    uint32_t g = 0, n = 0;
    int prev_b = -1;
    for (int u = u_begin; u < u_end; ++u, ++n) {
      const Unit x = unit_of(u, nqb, A);
      if (x.b != prev_b) {  // key mask bias of the sequence (0 / -inf; keys >= S masked)
        soft_sync();        // every thread finished reading the previous mask
        for (int j = tid; j < KC * 128; j += kSoft)
          sMask[j] = (j < S && __ldg(mask + (size_t)x.b * S + j) != 0) ? 0.0f : -INFINITY;
        soft_sync();
        prev_b = x.b;
      }
      mbar_wait(s_full, n & 1);
      if (threadIdx.x == 64) ltrace(trace, n, 3);
      tc_fence_after();
      // The three passes walk this quarter's keys in 16-column slices; the
      // TMEM load of slice i + 1 is issued right after the wait for slice i,
      // so it lands while slice i is processed (tcgen05.wait::ld waits for all
      // outstanding loads, hence two alternating register buffers).
      constexpr int NSL = 2 * KC;
      auto col_of = [&](int sl) { return (uint32_t)((sl >> 1) * 128 + qt * 32 + (sl & 1) * 16); };
      // pass 1: row max of s = RN(raw * cd) + mask bias
      float mx = -INFINITY;
      {
        uint32_t buf[2][16];
        tmem_ld16(trow + col_of(0), buf[0]);
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) {
          tmem_wait_ld();
          if (sl + 1 < NSL) tmem_ld16(trow + col_of(sl + 1), buf[(sl + 1) & 1]);
          const float2* mk = reinterpret_cast<const float2*>(sMask + col_of(sl));
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float2 sv = fma2(make_float2(__uint_as_float(buf[sl & 1][2 * j]), __uint_as_float(buf[sl & 1][2 * j + 1])),
                                   cd2, mk[j]);
            mx = fmaxf(mx, fmaxf(sv.x, sv.y));
          }
        }
      }
      if (threadIdx.x == 64) ltrace(trace, n, 4);
      redMax[qt * kLQ + r] = mx;
      quad_sync();
      mx = fmaxf(fmaxf(redMax[r], redMax[kLQ + r]), fmaxf(redMax[2 * kLQ + r], redMax[3 * kLQ + r]));
      const float2 mxv = make_float2(mx, mx);
      // pass 2: e = exp(s - max) in fp32, written back over S; row sum
      float2 la = make_float2(0.0f, 0.0f), lb = make_float2(0.0f, 0.0f);
      {
        uint32_t buf[2][16];
        tmem_ld16(trow + col_of(0), buf[0]);
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) {
          tmem_wait_ld();
          if (sl + 1 < NSL) tmem_ld16(trow + col_of(sl + 1), buf[(sl + 1) & 1]);
          const float2* mk = reinterpret_cast<const float2*>(sMask + col_of(sl));
          uint32_t* v = buf[sl & 1];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float2 sv = fma2(make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])), cd2, mk[j]);
            const float2 t = mul2(sub2(sv, mxv), l2e);
            const float2 e = make_float2(ex2l(t.x), ex2l(t.y));
            if (j & 1) lb = add2(lb, e);
            else la = add2(la, e);
            v[2 * j] = __float_as_uint(e.x);
            v[2 * j + 1] = __float_as_uint(e.y);
          }
          tmem_st16(trow + col_of(sl), *reinterpret_cast<uint32_t(*)[16]>(v));
        }
      }
      tmem_wait_st();
      if (threadIdx.x == 64) ltrace(trace, n, 5);
      const float2 l2 = add2(la, lb);
      redSum[qt * kLQ + r] = l2.x + l2.y;
      quad_sync();
      const float l = (redSum[r] + redSum[kLQ + r]) + (redSum[2 * kLQ + r] + redSum[3 * kLQ + r]);  // fixed order
      quad_sync();  // every quarter read redMax / redSum before the next unit's writes
      const float rl = __frcp_rn(l);
      const float2 lv = make_float2(l, l), rlv = make_float2(rl, rl);
      // pass 3: P16 = R16(e / l) chunk by chunk into P[g & 1] (K-major, 128B
      // swizzle: 16-byte chunk cc of row r at (cc ^ (r & 7)); this quarter's
      // 32 keys = chunks 4 (qt & 1) .. + 3 of k-block qt >> 1)
      {
        uint32_t buf[2][16];
        tmem_ld16(trow + col_of(0), buf[0]);
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) {
          tmem_wait_ld();
          if (sl + 1 < NSL) tmem_ld16(trow + col_of(sl + 1), buf[(sl + 1) & 1]);
          const uint32_t gg = g + (sl >> 1);  // P buffer of chunk sl / 2
          if ((sl & 1) == 0) mbar_wait(p_empty + (gg & 1), ((gg >> 1) & 1) ^ 1);  // P.V of chunk gg - 2 done
          uint8_t* prow = smem + SmemL::P + (gg & 1) * 2 * kLTile + (qt >> 1) * kLTile + r * 128;
          const uint32_t* v = buf[sl & 1];
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int j = cc * 4 + i;
              const float2 pv = div2_cr(make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])), lv, rlv);
              w[i] = pack_half2(pv.x, pv.y);
            }
            const int pc = (qt & 1) * 4 + (sl & 1) * 2 + cc;
            *reinterpret_cast<uint4*>(prow + ((pc ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
          if (sl & 1) {
            tc_fence_before();
            fence_async_smem();
            mbar_arrive(p_full + (gg & 1));
          }
        }
        g += KC;
      }
      if (threadIdx.x == 64) ltrace(trace, n, 6);
      // epilogue: ctx = R16(O), fp16 rows; then TMEM is free for the next unit
      mbar_wait(o_full, n & 1);
      tc_fence_after();
      uint32_t o[16];
      tmem_ld16(trow + kO + qt * 16, o);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(t_free);
      if (threadIdx.x == 64) ltrace(trace, n, 7);
      const int qrow = x.qb * kLQ + r;
      if (qrow < S) {
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) pk[i] = pack_half2(__uint_as_float(o[2 * i]), __uint_as_float(o[2 * i + 1]));
        uint4* dst = reinterpret_cast<uint4*>(ctx + ((size_t)x.b * S + qrow) * ldc + x.h * kLD + qt * 16);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}


// ---------------------------------------------------------------------------
// KC = 2 (128 < S <= 256, C5): two units in flight.  The 16 softmax warps form
// two groups of 8 (two warps per TMEM lane quadrant, each owning the key half
// [64 hf, 64 hf + 64) of both chunks) that take alternate units; group G owns
// TMEM columns [256 G, 256 G + 256): S_0, S_1, and O over S_0's first 64
// columns once the group's pass 3 has consumed S_0.  The MMA thread issues
// S(n) as soon as group n & 1 has read O(n - 2), then P(n - 1) . V(n - 1) of
// the other group, so one group's passes overlap the other's MMAs, P.V and
// epilogue.  Same arithmetic order per row as attention_long_kernel except
// that the row sum is combined from two halves (half 0 + half 1) instead of
// four quarters.
constexpr int kL2Threads = 64 + 32 * 16;
struct SmemL2 {
  static constexpr int RING = 0;                              // [kLSlots] tiles
  static constexpr int P = RING + kLSlots * kLTile;           // [2 groups] 2 k-blocks of 64 keys (one chunk)
  static constexpr int MASK = P + 2 * 2 * kLTile;             // [2 groups][256] floats
  static constexpr int XCH = MASK + 2 * 256 * 4;              // [max|sum][2 G][2 half][128] floats
  static constexpr int BAR = XCH + 8 * kLQ * 4;
  static constexpr int TOTAL = BAR + 256 + 1024;
  static_assert(TOTAL <= 227 * 1024, "smem budget");
};

__global__ void __launch_bounds__(kL2Threads, 1)
    attention_long2_kernel(const __grid_constant__ CUtensorMap tmQKV, const int32_t* __restrict__ mask, int B, int S,
                           int A, int hm_rows, float scale, __half* __restrict__ ctx, int ldc) {
  constexpr int KC = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SmemL2::BAR);
  uint64_t* full = bar;                    // [kLSlots]
  uint64_t* empty = bar + kLSlots;         // [kLSlots]
  uint64_t* s_full = bar + 2 * kLSlots;    // [2] MMA -> group G (S of its unit)
  uint64_t* p_full = s_full + 2;           // [2] group G (P chunk written) -> MMA
  uint64_t* p_empty = p_full + 2;          // [2] MMA (P.V of the chunk done) -> group G
  uint64_t* o_full = p_empty + 2;          // [2] MMA (O complete) -> group G
  uint64_t* t_free = o_full + 2;           // [2] group G (O read) -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_free + 2);
  float* sMask = reinterpret_cast<float*>(smem + SmemL2::MASK);
  float* sXch = reinterpret_cast<float*>(smem + SmemL2::XCH);
  constexpr int kGroup = 256;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int D = A * kLD;
  const int nqb = (S + kLQ - 1) / kLQ;
  const int n_units = B * nqb * A;
  const int per = (n_units + gridDim.x - 1) / gridDim.x;
  const int u_begin = min(n_units, (int)blockIdx.x * per), u_end = min(n_units, u_begin + per);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    for (int i = 0; i < kLSlots; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(s_full + g, 1);
      mbar_init(p_full + g, kGroup);
      mbar_init(p_empty + g, 1);
      mbar_init(o_full + g, 1);
      mbar_init(t_free + g, kGroup);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();
  griddep_launch();

  if (warp == 0) {
    if (lane == 0) {
      uint32_t cnt = 0;
      auto load = [&](int col, int row) {
        const int slot = cnt % kLSlots;
        mbar_wait(empty + slot, ((cnt / kLSlots) & 1) ^ 1);
        mbar_expect_tx(full + slot, kLTile);
        tma_load_2d(smem + SmemL2::RING + slot * kLTile, &tmQKV, full + slot, col, row, kEvictFirst);
        ++cnt;
      };
      for (int u = u_begin; u < u_end; ++u) {  // ring position of unit n's tiles: 5 n + {Q, K0, K1, V0, V1}
        const Unit x = unit_of(u, nqb, A);
        const int row0 = x.b * S;
        if (hm_rows > 0) {
          load(0, x.h * hm_rows + row0 + x.qb * kLQ);
          for (int c = 0; c < KC; ++c) load(0, (A + x.h) * hm_rows + row0 + c * 128);
          for (int c = 0; c < KC; ++c) load(0, (2 * A + x.h) * hm_rows + row0 + c * 128);
        } else {
          load(x.h * kLD, row0 + x.qb * kLQ);
          for (int c = 0; c < KC; ++c) load(D + x.h * kLD, row0 + c * 128);
          for (int c = 0; c < KC; ++c) load(2 * D + x.h * kLD, row0 + c * 128);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id1 = idesc_l(128, 0);
      constexpr uint32_t id2 = idesc_l(kLD, 1);
      auto slot_of = [](uint32_t pos) { return (int)(pos % kLSlots); };
      auto par_of = [](uint32_t pos) { return (pos / kLSlots) & 1; };
      uint32_t pchunk[2] = {0, 0};  // P chunks consumed per group (p_full / p_empty phases)
      auto issue_pv = [&](uint32_t m) {
        const int g = m & 1;
        const uint32_t base = 5 * m;
        for (int c = 0; c < KC; ++c) {
          const uint32_t vpos = base + 3 + c;
          mbar_wait(full + slot_of(vpos), par_of(vpos));
          mbar_wait(p_full + g, pchunk[g] & 1);
          tc_fence_after();
          uint8_t* P = smem + SmemL2::P + g * 2 * kLTile;
          uint8_t* V = smem + SmemL2::RING + slot_of(vpos) * kLTile;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t pd = make_sw128_desc(P + (k >> 2) * kLTile) + 2 * (k & 3);
            const uint64_t vd = sw128_desc_mn(V + k * 2048);
            mma_f16(tmem + g * 256, pd, vd, id2, (c | k) != 0);
          }
          mma_commit(empty + slot_of(vpos));
          mma_commit(p_empty + g);
          ++pchunk[g];
        }
        mma_commit(o_full + g);
      };
      uint32_t n = 0;
      for (int u = u_begin; u < u_end; ++u, ++n) {
        const int g = n & 1;
        mbar_wait(t_free + g, ((n >> 1) & 1) ^ 1);  // O(n - 2) read: group g's columns are free
        tc_fence_after();
        const uint32_t base = 5 * n;
        mbar_wait(full + slot_of(base), par_of(base));
        const uint64_t qd = make_sw128_desc(smem + SmemL2::RING + slot_of(base) * kLTile);
        for (int c = 0; c < KC; ++c) {
          const uint32_t kpos = base + 1 + c;
          mbar_wait(full + slot_of(kpos), par_of(kpos));
          tc_fence_after();
          const uint64_t kd = make_sw128_desc(smem + SmemL2::RING + slot_of(kpos) * kLTile);
#pragma unroll
          for (int k = 0; k < kLD / 16; ++k) mma_f16(tmem + g * 256 + c * 128, qd + 2 * k, kd + 2 * k, id1, k != 0);
          mma_commit(empty + slot_of(kpos));
        }
        mma_commit(empty + slot_of(base));
        mma_commit(s_full + g);
        if (n > 0) issue_pv(n - 1);
      }
      if (n > 0) issue_pv(n - 1);
    }
  } else {
    const int G = (warp - 2) >> 3;
    const int hf = ((warp - 2) >> 2) & 1;
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int gtid = threadIdx.x - 64 - kGroup * G;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + G * 256;
    float* gMask = sMask + G * 256;
    float* xmax = sXch + ((0 * 2 + G) * 2) * kLQ;  // [half][kLQ]
    float* xsum = sXch + ((1 * 2 + G) * 2) * kLQ;
    auto group_sync = [G]() { asm volatile("bar.sync %0, 256;" ::"r"(2 + G) : "memory"); };
    auto pair_sync = [G, q]() { asm volatile("bar.sync %0, 64;" ::"r"(4 + 4 * G + q) : "memory"); };
    const float2 cd2 = make_float2(scale, scale);
    const float2 l2e = make_float2(1.4426950408889634f, 1.4426950408889634f);
    constexpr int NSL = 2 * KC * 2;  // 16-column slices of this thread's 2 x 64 keys
    auto col_of = [&](int sl) { return (uint32_t)((sl >> 2) * 128 + hf * 64 + (sl & 3) * 16); };
    uint32_t n = 0, k = 0, pc = 0;
    int prev_b = -1;
    for (int u = u_begin; u < u_end; ++u, ++n) {
      if ((int)(n & 1) != G) continue;
      const Unit x = unit_of(u, nqb, A);
      if (x.b != prev_b) {
        group_sync();
        for (int j = gtid; j < KC * 128; j += kGroup)
          gMask[j] = (j < S && __ldg(mask + (size_t)x.b * S + j) != 0) ? 0.0f : -INFINITY;
        group_sync();
        prev_b = x.b;
      }
      mbar_wait(s_full + G, k & 1);
      tc_fence_after();
      // pass 1: row max of s = RN(raw * cd) + mask bias over this thread's keys
      float mx = -INFINITY;
      {
        uint32_t buf[2][16];
        tmem_ld16(trow + col_of(0), buf[0]);
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) {
          tmem_wait_ld();
          if (sl + 1 < NSL) tmem_ld16(trow + col_of(sl + 1), buf[(sl + 1) & 1]);
          const float2* mk = reinterpret_cast<const float2*>(gMask + col_of(sl));
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float2 sv = fma2(make_float2(__uint_as_float(buf[sl & 1][2 * j]), __uint_as_float(buf[sl & 1][2 * j + 1])),
                                   cd2, mk[j]);
            mx = fmaxf(mx, fmaxf(sv.x, sv.y));
          }
        }
      }
      xmax[hf * kLQ + r] = mx;
      pair_sync();
      mx = fmaxf(mx, xmax[(hf ^ 1) * kLQ + r]);
      const float2 mxv = make_float2(mx, mx);
      // pass 2: e = exp(s - max), written back over S; row sum
      float2 la = make_float2(0.0f, 0.0f), lb = make_float2(0.0f, 0.0f);
      {
        uint32_t buf[2][16];
        tmem_ld16(trow + col_of(0), buf[0]);
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) {
          tmem_wait_ld();
          if (sl + 1 < NSL) tmem_ld16(trow + col_of(sl + 1), buf[(sl + 1) & 1]);
          const float2* mk = reinterpret_cast<const float2*>(gMask + col_of(sl));
          uint32_t* v = buf[sl & 1];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float2 sv = fma2(make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])), cd2, mk[j]);
            const float2 t = mul2(sub2(sv, mxv), l2e);
            const float2 e = make_float2(ex2l(t.x), ex2l(t.y));
            if (j & 1) lb = add2(lb, e);
            else la = add2(la, e);
            v[2 * j] = __float_as_uint(e.x);
            v[2 * j + 1] = __float_as_uint(e.y);
          }
          tmem_st16(trow + col_of(sl), *reinterpret_cast<uint32_t(*)[16]>(v));
        }
      }
      tmem_wait_st();
      const float2 l2 = add2(la, lb);
      const float lh = l2.x + l2.y;
      xsum[hf * kLQ + r] = lh;
      pair_sync();
      const float l = lh + xsum[(hf ^ 1) * kLQ + r];  // half 0 + half 1 (commutative: same on both)
      const float rl = __frcp_rn(l);
      const float2 lv = make_float2(l, l), rlv = make_float2(rl, rl);
      // pass 3: P16 = R16(e / l) chunk by chunk into the group's P buffer
      // (this thread's 64 keys = k-block hf of the chunk), P.V by the MMA
      {
        uint32_t buf[2][16];
        tmem_ld16(trow + col_of(0), buf[0]);
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) {
          tmem_wait_ld();
          if (sl + 1 < NSL) tmem_ld16(trow + col_of(sl + 1), buf[(sl + 1) & 1]);
          if ((sl & 3) == 0) {
            mbar_wait(p_empty + G, (pc & 1) ^ 1);  // the previous P.V of this group's buffer is done
            tc_fence_after();
          }
          uint8_t* prow = smem + SmemL2::P + G * 2 * kLTile + hf * kLTile + r * 128;
          const uint32_t* v = buf[sl & 1];
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int j = cc * 4 + i;
              const float2 pv = div2_cr(make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])), lv, rlv);
              w[i] = pack_half2(pv.x, pv.y);
            }
            const int pcol = (sl & 3) * 2 + cc;  // 16-byte chunk within the 128-byte k-block row
            *reinterpret_cast<uint4*>(prow + ((pcol ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
          if ((sl & 3) == 3) {
            tc_fence_before();
            fence_async_smem();
            mbar_arrive(p_full + G);
            ++pc;
          }
        }
      }
      // epilogue: ctx = R16(O) (this thread's half of the 64 O columns)
      mbar_wait(o_full + G, k & 1);
      tc_fence_after();
      uint32_t o[32];
      tmem_ld32(trow + hf * 32, o);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(t_free + G);
      const int qrow = x.qb * kLQ + r;
      if (qrow < S) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = pack_half2(__uint_as_float(o[2 * i]), __uint_as_float(o[2 * i + 1]));
        uint4* dst = reinterpret_cast<uint4*>(ctx + ((size_t)x.b * S + qrow) * ldc + x.h * kLD + hf * 32);
#pragma unroll
        for (int c = 0; c < 4; ++c) dst[c] = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      }
      ++k;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

bool attention_long_supported(int S, int d, int ldqkv, int ldctx) {
  return d == kLD && S > 128 && S <= kLMaxKeys && (ldqkv % 8) == 0 && (ldctx % 8) == 0;
}

cudaError_t prepare_attention_long_kernel() {
  cudaError_t e = cudaFuncSetAttribute(attention_long_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SmemL::TOTAL);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(attention_long2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemL2::TOTAL);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(attention_long_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemL::TOTAL);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(attention_long_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemL::TOTAL);
}

cudaError_t launch_attention_long(const AttnTCPlan& plan, const int32_t* mask, int B, int S, int A, __half* ctx,
                                  int ldctx, cudaStream_t s, unsigned long long* trace) {
  if (S <= 128 || S > kLMaxKeys) return cudaErrorInvalidValue;
  const float scale = (float)(1.0 / sqrt((double)kLD));  // fp32(1/sqrt(d)) (R10)
  const int n_units = B * ((S + kLQ - 1) / kLQ) * A;
  const int grid = n_units < kNumSMs ? n_units : kNumSMs;
  const int kc = (S + 127) / 128;
  // KC = 2: two units in flight (attention_long2_kernel; C5 launch 76 -> 65 us);
  // the debug timeline (trace) is only recorded by the one-unit kernel
  if (kc == 2 && trace == nullptr)
    launch_ex(attention_long2_kernel, dim3(grid), dim3(kL2Threads), SmemL2::TOTAL, s, 0, plan.map, mask, B, S, A,
              plan.hm_rows, scale, ctx, ldctx);
  else if (kc == 2)
    launch_ex(attention_long_kernel<2>, dim3(grid), dim3(kLThreads), SmemL::TOTAL, s, 0, plan.map, mask, B, S, A,
              plan.hm_rows, scale, ctx, ldctx, trace);
  else if (kc == 3)
    launch_ex(attention_long_kernel<3>, dim3(grid), dim3(kLThreads), SmemL::TOTAL, s, 0, plan.map, mask, B, S, A,
              plan.hm_rows, scale, ctx, ldctx, trace);
  else
    launch_ex(attention_long_kernel<4>, dim3(grid), dim3(kLThreads), SmemL::TOTAL, s, 0, plan.map, mask, B, S, A,
              plan.hm_rows, scale, ctx, ldctx, trace);
  return cudaGetLastError();
}

}  // namespace ff
