// attention_tc.cu -- fused masked-softmax attention on the 5th-gen tensor
// cores (tcgen05 + TMEM + TMA) for head_dim 64 and S <= 128: the shapes of the
// headline configs (P:135 multi-head attention node fusion;
// Q.K^T and P.V in floating point).
//
// One work item = (sequence b, group of <= 8 heads); one persistent CTA per SM
// walks the heads of its items with Q/K/V triple-buffered across heads.
//   warp 0     TMA: Q, K, V head slices (128 rows x 64 fp16, 128B-swizzled)
//   warp 1     TMEM allocator + MMA issuer (one thread):
//                S[128 x 128] (TMEM, fp32) = Q . K^T        kind::f16, K-major A/B
//                O[128 x  64] (TMEM, fp32) = P . V          A = P (smem, K-major),
//                                                            B = V (smem, MN-major)
//   warps 2-9  softmax + epilogue: TMEM lane quadrant = query rows, two warps
//              per quadrant split the keys (and O's columns) in halves:
//                s = fp32(q.k) * fp32(1/sqrt(d)), masked keys -> -inf (R4)
//                p = exp(s - max) / sum  in fp32, P16 = R16(p)  (R9, normalized
//                before P.V), written to smem in the 128B-swizzled K-major
//                layout the MMA reads; ctx = R16(O).
// int8 layers (A <= 8): the R16 ctx of all heads of the row is parked in TMEM
// (packed fp16 pairs, columns [256, 256 + 32 A)); after the item's last head
// the row scale (Q8row, R6-R8) is known, and head j of the item is quantized
// and stored by the epilogue of head j of the CTA's next item (the last item
// after the loop), so ctx goes to HBM once, as s8 rows + scale (SURVEY 8(a)
// a3+a4 fused) without a per-item requant stall.  Otherwise ctx is stored as
// fp16 rows.
// Row max / sum are combined across the two half-row threads through smem in
// a fixed order.  Keys beyond S (S < 128) are masked; Q rows beyond S are
// computed and not stored.
#include "ff_kernels.h"
#include "ptx.cuh"
#include "quant.cuh"

namespace ff {

namespace {

constexpr int kQ = 128;             // queries per item (TMEM lanes)
constexpr int kKeys = 128;          // keys (S <= 128)
// DP = head_dim padded to the MMA granularity: 64 (d in (32, 64]) or 32
// (d <= 32, e.g. the TinyBERT shape's d = 26, DESIGN R18); an item holds up
// to 512 / DP heads (their packed fp16 ctx fills the 256 parking columns).
template <int DP>
struct HeadCfg {
  static constexpr int kMaxHeads = 512 / DP;
  static constexpr int kPark = DP / 2;         // parking columns per head (packed fp16 pairs)
};
constexpr int kTileBytes = 128 * 128;  // 128 rows x 128 B (64 fp16)
// Q/K/V ring depth: P(n) is written over the dead Q and K tiles of head n's
// own slot (S(n) has consumed them), so no separate P buffers are needed and a
// 4th head fits in flight (192 KB of loads in flight per SM instead of 144 KB)
constexpr int kKVStages = 4;
constexpr int kSoftmaxWarps = 16;  // 2 groups x 4 quadrants x 2 key halves
constexpr int kThreadsTC = 64 + 32 * kSoftmaxWarps;
constexpr uint32_t kTmemCtx = 256;  // packed ctx [256, 256 + 32 * heads)

struct SmemTC {
  static constexpr int SLOT = 3 * kTileBytes;                // Q, K, V of one head (P(n) over Q, K)
  static constexpr int MASK = kKVStages * SLOT;              // [2][kKeys] floats (per group)
  static constexpr int RED = MASK + 2 * kKeys * 4;           // [2 G][2 half][128] floats: row amax partials
  static constexpr int XCH = RED + 4 * kQ * 4;               // [2 max|sum][2 G][2 half][128] floats
  static constexpr int BAR = XCH + 8 * kQ * 4;
  static constexpr int TOTAL = BAR + 256 + 1024;             // barriers + alignment slack
  static_assert(TOTAL <= 227 * 1024, "smem budget");
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
// Debug timeline (ff_debug_attention_q8 with a trace buffer): globaltimer of
// event e for head n of CTA c at trace[(c * kTraceHeads + n) * 8 + e].
constexpr int kTraceHeads = 32;
__device__ __forceinline__ void trace_ev(unsigned long long* trace, uint32_t n, int e) {
  if (trace != nullptr && n < kTraceHeads) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    trace[((size_t)blockIdx.x * kTraceHeads + n) * 8 + e] = t;
  }
}

// Walk of the heads one CTA processes: items blockIdx.x, +gridDim.x, ...;
// each item = (sequence b, heads [h0, h0 + nh)).
struct HeadIter {
  int item, hl, b, h0, nh;
  int n_items, n_groups, A, stride, mh, rev;
  __device__ HeadIter(int first, int n_items_, int n_groups_, int A_, int stride_, int mh_, int rev_)
      : item(first), hl(0), n_items(n_items_), n_groups(n_groups_), A(A_), stride(stride_), mh(mh_), rev(rev_) {
    set();
  }
  __device__ void set() {
    if (item < n_items) {
      // rev: items walked from the last sequence to the first, so that the
      // rows the QKV GEMM wrote last (most likely still in L2) are read first
      const int ri = rev ? n_items - 1 - item : item;
      b = ri / n_groups;
      h0 = (ri - b * n_groups) * mh;
      nh = min(A, h0 + mh) - h0;
    }
  }
  __device__ bool valid() const { return item < n_items; }
  __device__ void next() {
    if (++hl == nh) {
      hl = 0;
      item += stride;
      set();
    }
  }
};

// Per-head schedule (n = this CTA's head counter; every role walks the same
// sequence).  The 8 softmax warps form two groups of 4 (one warp per TMEM lane
// quadrant, a thread owns a whole query row) that take alternate heads:
// group G = n & 1 owns TMEM columns [128 G, 128 G + 128), where the MMA
// computes S(n) and later, once the group has turned S into P, O(n) = P V
// (first DP columns).  The MMA thread issues S(n) as soon as group G has read
// O(n - 2), then O(n - 1) of the other group, so one group's softmax overlaps
// the other's exp / P-store / epilogue and the MMAs:
//   MMA:      .. S(n) | O(n-1) | S(n+1) | O(n) ..
//   group G:  .. softmax(n) -> P[G] | epilogue(n) (O(n) from its S columns) ..
// Buffers: Q/K/V x4 stages (smem; P(n) is written over head n's Q and K
// tiles), S/O x2 (TMEM, one per group), parked int8 ctx [256, 512).
template <int DP>
__global__ void __launch_bounds__(kThreadsTC, 1)  // a thread holds half an S row
    attention_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const int32_t* __restrict__ mask, int B, int S,
                        int A, int d, int hs, int mh, int hm_rows, float scale, __half* __restrict__ ctx, int ldc,
                        int8_t* __restrict__ ctxq, int ldq, float* __restrict__ ctxs,
                        const uint8_t* __restrict__ qkv_rows, int row_bytes, unsigned long long* __restrict__ trace,
                        int rev) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SmemTC::BAR);
  uint64_t* kv_full = bar + 0;                 // [kKVStages] TMA -> MMA
  uint64_t* kv_empty = bar + kKVStages;        // [kKVStages] MMA (after P.V) -> TMA
  uint64_t* s_full = bar + 2 * kKVStages;      // [2] MMA (S in group G's columns) -> group G
  uint64_t* p_full = s_full + 2;               // [2] group G (P written, S consumed) -> MMA
  uint64_t* o_full = p_full + 2;               // [2] MMA (O in group G's columns) -> group G
  uint64_t* t_free = o_full + 2;               // [2] group G (O read) -> MMA: columns free for S(n + 2)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_free + 2);
  float* sMask = reinterpret_cast<float*>(smem + SmemTC::MASK);  // [2][kKeys]: per group
  float* sRed = reinterpret_cast<float*>(smem + SmemTC::RED);    // [2 G][2 half][kQ]: row amax partials
  float* sXch = reinterpret_cast<float*>(smem + SmemTC::XCH);    // [max|sum][G][half][kQ]: half-row stats

  using HC = HeadCfg<DP>;
  using Iter = HeadIter;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int D = A * hs;  // QKV section width (head stride hs >= d; hs > d: zero-padded heads)
  const int n_groups = (A + mh - 1) / mh;  // items per sequence (mh heads each, mh <= 512 / DP)
  const int n_items = B * n_groups;
  const int it_first = (int)blockIdx.x;
  const int it_stride = (int)gridDim.x;
  constexpr int kGroupThreads = 256;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    for (int i = 0; i < kKVStages; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(s_full + g, 1);
      mbar_init(p_full + g, kGroupThreads);
      mbar_init(o_full + g, 1);
      mbar_init(t_free + g, kGroupThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);  // S/O of group 0 [0,128), group 1 [128,256), packed ctx [256, 512)
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
      // (An L2 bulk prefetch of each item's QKV rows, meant to open each DRAM
      // page once per item, measured 5.5 us slower per C3 launch: the QKV
      // buffer was just written by the projection GEMM and is largely still
      // in L2, and the prefetch queued ahead of the first head's loads.)
      (void)qkv_rows;
      (void)row_bytes;
      uint32_t n = 0;
      for (Iter it(it_first, n_items, n_groups, A, it_stride, mh, rev); it.valid(); it.next(), ++n) {
        const int slot = n % kKVStages;
        const int h = it.h0 + it.hl;
        uint8_t* base = smem + slot * SmemTC::SLOT;
        mbar_wait(kv_empty + slot, ((n / kKVStages) & 1) ^ 1);
        trace_ev(trace, n, 0);
        mbar_expect_tx(kv_full + slot, 3 * kTileBytes);
        if (hm_rows > 0) {  // head-major QKV: each slice is a contiguous 128 x 64 block
          tma_load_2d(base, &tmQKV, kv_full + slot, 0, h * hm_rows + it.b * S, kEvictFirst);
          tma_load_2d(base + kTileBytes, &tmQKV, kv_full + slot, 0, (A + h) * hm_rows + it.b * S, kEvictFirst);
          tma_load_2d(base + 2 * kTileBytes, &tmQKV, kv_full + slot, 0, (2 * A + h) * hm_rows + it.b * S,
                      kEvictFirst);
        } else {
          tma_load_2d(base, &tmQKV, kv_full + slot, h * hs, it.b * S, kEvictFirst);
          tma_load_2d(base + kTileBytes, &tmQKV, kv_full + slot, D + h * hs, it.b * S, kEvictFirst);
          tma_load_2d(base + 2 * kTileBytes, &tmQKV, kv_full + slot, 2 * D + h * hs, it.b * S, kEvictFirst);
        }
      }
    }
  } else if (warp == 1) {
    // all 32 lanes walk the schedule (they zero Q's padding columns when
    // hs < DP); lane 0 issues the MMAs and commits
    const bool issuer = lane == 0;
    constexpr uint32_t id1 = idesc_f16(kKeys, 0);  // S = Q K^T: N = 128 keys
    constexpr uint32_t id2 = idesc_f16(DP, 1);     // O = P V:   N = DP, V MN-major
    auto issue_pv = [&](uint32_t m) {
      const int g = m & 1;
      const int slot = m % kKVStages;
      mbar_wait(p_full + g, (m >> 1) & 1);  // group g has written P(m) and read all of S(m)
      if (issuer) {
        trace_ev(trace, m, 5);
        tc_fence_after();
        uint8_t* P = smem + slot * SmemTC::SLOT;  // P(m) over the Q, K tiles of m's slot
        uint8_t* V = smem + slot * SmemTC::SLOT + 2 * kTileBytes;
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k) {
          // A = P: k-block k/4 (64 keys), +32 B per 16 keys inside the 128B row
          const uint64_t pd = make_sw128_desc(P + (k >> 2) * kTileBytes) + 2 * (k & 3);
          // B = V (MN-major): 16 keys = two 8-row groups = 2048 B
          const uint64_t vd = make_sw128_desc_mn(V + k * 2048);
          mma_f16(tmem + g * 128, pd, vd, id2, k != 0);
        }
        mma_commit(o_full + g);
        mma_commit(kv_empty + slot);  // Q/K/V of head m free once these MMAs complete
      }
      __syncwarp();
    };
    uint32_t n = 0;
    for (Iter it(it_first, n_items, n_groups, A, it_stride, mh, rev); it.valid(); it.next(), ++n) {
      const int slot = n % kKVStages;
      const int g = n & 1;
      uint8_t* base = smem + slot * SmemTC::SLOT;
      mbar_wait(kv_full + slot, (n / kKVStages) & 1);
      if (issuer) trace_ev(trace, n, 1);
      if (hs < DP) {
        // head stride below the MMA granularity (d = 16 unpadded): the box
        // also holds the next head's first columns; zero Q's columns
        // [hs, DP) so they add nothing to Q.K^T (V's extra columns only
        // reach O columns that are never stored).  Padded heads (hs = DP >
        // d, e.g. d = 26) carry exact zeros in [d, hs) from the QKV GEMM.
        for (int rr = lane; rr < 128; rr += 32)
          for (int c = hs; c < DP; ++c)
            *reinterpret_cast<__half*>(base + rr * 128 + (((c >> 3) ^ (rr & 7)) << 4) + (c & 7) * 2) =
                __float2half_rn(0.0f);
        fence_async_smem();
        __syncwarp();
      }
      mbar_wait(t_free + g, ((n >> 1) & 1) ^ 1);  // group g has read O(n - 2) out of its columns
      if (issuer) {
        trace_ev(trace, n, 2);
        tc_fence_after();
        const uint64_t qd = make_sw128_desc(base), kd = make_sw128_desc(base + kTileBytes);
#pragma unroll
        for (int k = 0; k < DP / 16; ++k) mma_f16(tmem + g * 128, qd + 2 * k, kd + 2 * k, id1, k != 0);
        mma_commit(s_full + g);
      }
      __syncwarp();
      if (n > 0) issue_pv(n - 1);
    }
    if (n > 0) issue_pv(n - 1);
  } else {
    const int G = (warp - 2) >> 3;        // ping-pong group: heads n with n & 1 == G
    const int hf = ((warp - 2) >> 2) & 1;  // key half [64 hf, 64 hf + 64) of S, O columns half hf
    const int q = warp & 3;               // TMEM lane quadrant = rows [32 q, 32 q + 32)
    const int r = q * 32 + lane;
    const int gtid = threadIdx.x - 64 - kGroupThreads * G;  // 0..255 within the group
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t treg = trow + G * 128;  // this group's S / O columns
    float* gMask = sMask + G * kKeys;
    const bool fuse_q = ctxq != nullptr;
    auto both_sync = []() { asm volatile("bar.sync 2, 512;" ::: "memory"); };  // both groups (item end)
    auto group_sync = [G]() { asm volatile("bar.sync %0, 256;" ::"r"(3 + G) : "memory"); };
    // the two half-row warps of (group, quadrant): row max / sum exchange
    auto pair_sync = [G, q]() { asm volatile("bar.sync %0, 64;" ::"r"(5 + 4 * G + q) : "memory"); };
    float* xmax = sXch + ((0 * 2 + G) * 2) * kQ;  // [half][kQ]
    float* xsum = sXch + ((1 * 2 + G) * 2) * kQ;
    const float2 cd2 = make_float2(scale, scale);
    const float2 l2e = make_float2(1.4426950408889634f, 1.4426950408889634f);
    constexpr int HW = DP / 2;  // packed fp16 words of one head's row
    __half2 amax2 = __float2half2_rn(0.0f);  // |ctx| max of the row over this group's heads of the item

    // Q8row of a finished item (R6-R8): its packed fp16 ctx stays parked in
    // TMEM; head j of it is quantized and stored by whichever group runs head
    // j of the CTA's NEXT item, right before that head parks its own ctx in the
    // same columns (fused items hold all A heads); the last item is flushed
    // after the loop.  Both groups derive the same scale at the item end.
    bool qpend = false;
    int qb = 0, qhbase = 0, qnh = 0;
    float qsc = 1.0f, qrs = 1.0f;
    constexpr int HH = HW / 2;       // packed words of this thread's half of a head row
    const int c0 = hf * (DP / 2);    // first head column of this thread's half
    auto flush_head = [&](int j) {  // quantize + store this thread's half of parked head j of the pending item
      uint32_t v[HH];
      if constexpr (HH == 16) tmem_ld16(trow + kTmemCtx + j * HC::kPark + hf * HH, v);
      else tmem_ld8(trow + kTmemCtx + j * HC::kPark + hf * HH, v);
      tmem_wait_ld();
      uint32_t w[HH / 2];
#pragma unroll
      for (int i = 0; i < HH / 2; ++i) {
        const float2 a0 = __half22float2(*reinterpret_cast<const __half2*>(&v[2 * i]));
        const float2 a1 = __half22float2(*reinterpret_cast<const __half2*>(&v[2 * i + 1]));
        w[i] = q8_quant4(a0, a1, qsc, qrs);
      }
      if (r < S) {
        int8_t* row_q = ctxq + ((size_t)qb * S + r) * ldq + (qhbase + j) * d + c0;
        if (DP == 64 && d == 64) {  // the half row's 32 s8 values: one 32-byte sector
          uint4* dst = reinterpret_cast<uint4*>(row_q);
#pragma unroll
          for (int c = 0; c < 2; ++c) dst[c] = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
        } else {  // d even: 2-byte aligned pieces of the valid values
#pragma unroll
          for (int i = 0; i < HH; ++i)
            if (c0 + 2 * i < d) *reinterpret_cast<uint16_t*>(row_q + 2 * i) = (uint16_t)(w[i >> 1] >> ((i & 1) * 16));
        }
      }
    };

    uint32_t n = 0;
    int mask_item = -1;
    // key mask words of the next item, loaded one item ahead (thread gtid < kKeys
    // holds key gtid) so the load latency is not exposed at the item switch
    auto load_mask = [&](int item) -> int {
      if (gtid >= kKeys || gtid >= S || item >= n_items) return 0;
      return __ldg(mask + (size_t)((rev ? n_items - 1 - item : item) / n_groups) * S + gtid);
    };
    int mask_next = load_mask(it_first);
    for (Iter it(it_first, n_items, n_groups, A, it_stride, mh, rev); it.valid(); it.next(), ++n) {
      const bool mine = (int)(n & 1) == G;
      const bool item_last = it.hl == it.nh - 1;
      if (mine) {
        const uint32_t k = n >> 1;  // this group's head counter
        const int h = it.h0 + it.hl;
        if (it.item != mask_item) {  // key mask of the item's sequence (keys >= S masked)
          group_sync();              // every group thread finished reading the previous mask
          if (gtid < kKeys) gMask[gtid] = (gtid < S && mask_next != 0) ? 0.0f : -INFINITY;
          mask_next = load_mask(it.item + it_stride);
          group_sync();
          mask_item = it.item;
        }
        mbar_wait(s_full + G, k & 1);
        if (threadIdx.x == 64) trace_ev(trace, n, 3);
        tc_fence_after();
        // half an S row in registers (keys [64 hf, 64 hf + 64); 2 loads, one
        // wait): s = RN(raw * fp32(1/sqrt d)) + mask bias (0 / -inf) in one
        // FFMA2 per pair (R10), the row max (the two halves combined through
        // smem), e = exp2((s - max) log2 e) (R9) and the row sum in place
        uint32_t v[64];
#pragma unroll
        for (int c = 0; c < 2; ++c) tmem_ld32(treg + hf * 64 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
        tmem_wait_ld();
        tc_fence_before();  // (S is read; the MMA overwrites these columns with O after p_full)
        const float2* mk = reinterpret_cast<const float2*>(gMask + hf * 64);
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 sv = fma2(make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])), cd2, mk[j]);
          v[2 * j] = __float_as_uint(sv.x);
          v[2 * j + 1] = __float_as_uint(sv.y);
          m4[j & 1] = fmaxf(m4[j & 1], sv.x);
          m4[2 + (j & 1)] = fmaxf(m4[2 + (j & 1)], sv.y);
        }
        float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        xmax[hf * kQ + r] = mx;
        pair_sync();
        mx = fmaxf(mx, xmax[(hf ^ 1) * kQ + r]);
        const float2 mxv = make_float2(mx, mx);
        float2 la = make_float2(0.0f, 0.0f), lb = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 t = mul2(sub2(make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])), mxv), l2e);
          const float2 e = make_float2(ex2f(t.x), ex2f(t.y));
          if (j & 1) lb = add2(lb, e);
          else la = add2(la, e);
          v[2 * j] = __float_as_uint(e.x);
          v[2 * j + 1] = __float_as_uint(e.y);
        }
        const float2 l2 = add2(la, lb);
        const float lh = l2.x + l2.y;
        xsum[hf * kQ + r] = lh;
        pair_sync();
        const float l = lh + xsum[(hf ^ 1) * kQ + r];  // half 0 + half 1 (commutative: same on both)
        const float rl = __frcp_rn(l);
        const float2 lv = make_float2(l, l), rlv = make_float2(rl, rl);
        // P16 = R16(e / l) (IEEE quotient, R9) into a K-major 128B-swizzled
        // P tile over this head's Q / K tiles: keys [32 c, 32 c + 32) = 16-byte chunks
        // 4 (c & 1) .. + 3 of k-block c >> 1, chunk cc of row r at (cc ^ (r & 7))
        // (over the Q and K tiles of this head's slot: S(n) has consumed them)
        // (this thread's half: keys [64 hf, +64) = k-block hf)
        uint8_t* prow = smem + (n % kKVStages) * SmemTC::SLOT + r * 128 + hf * kTileBytes;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int j = c * 16 + cc * 4 + i;
              const float2 pv =
                  div2_cr(make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])), lv, rlv);
              w[i] = pack_half2(pv.x, pv.y);
            }
            const int pc = c * 4 + cc;
            *reinterpret_cast<uint4*>(prow + ((pc ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        tc_fence_before();
        fence_async_smem();
        mbar_arrive(p_full + G);
        if (threadIdx.x == 64) trace_ev(trace, n, 4);
        // epilogue of this head: ctx = R16(O), O in the group's first DP columns
        mbar_wait(o_full + G, k & 1);
        if (threadIdx.x == 64) trace_ev(trace, n, 6);
        tc_fence_after();
        // this thread's half of O: columns [c0, c0 + DP / 2)
        uint32_t o[DP / 2];
        if constexpr (DP == 64) tmem_ld32(treg + c0, *reinterpret_cast<uint32_t(*)[32]>(o));
        else tmem_ld16(treg + c0, *reinterpret_cast<uint32_t(*)[16]>(o));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(t_free + G);
        uint32_t pk[HH];
#pragma unroll
        for (int i = 0; i < HH; ++i) {
          // O columns >= d (padded or neighbouring head columns): zero
          pk[i] = c0 + 2 * i < d ? pack_half2(__uint_as_float(o[2 * i]), __uint_as_float(o[2 * i + 1])) : 0u;
          amax2 = __hmax2(amax2, __habs2(*reinterpret_cast<const __half2*>(&pk[i])));
        }
        if (ctx != nullptr && r < S) {
          __half* row_c = ctx + ((size_t)it.b * S + r) * ldc + h * d + c0;
          if (DP == 64 && d == 64) {
            uint4* dst = reinterpret_cast<uint4*>(row_c);
#pragma unroll
            for (int c = 0; c < 4; ++c) dst[c] = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
          } else {  // d even: 4-byte aligned pairs
#pragma unroll
            for (int i = 0; i < HH; ++i)
              if (c0 + 2 * i < d) *reinterpret_cast<uint32_t*>(row_c + 2 * i) = pk[i];
          }
        }
        if (fuse_q) {
          if (qpend && it.hl < qnh) flush_head(it.hl);  // frees parking slot hl (its load completed)
          if constexpr (HH == 16)
            tmem_st16(trow + kTmemCtx + it.hl * HC::kPark + hf * HH, *reinterpret_cast<uint32_t(*)[16]>(pk));
          else
            tmem_st8(trow + kTmemCtx + it.hl * HC::kPark + hf * HH, *reinterpret_cast<uint32_t(*)[8]>(pk));
          tmem_wait_st();
        }
        if (threadIdx.x == 64) trace_ev(trace, n, 7);
      }
      if (fuse_q && item_last) {
        // both groups: the row amax over all heads of the item -> its scale;
        // the previous item's parked heads this group did not flush (the item
        // had more heads than this one's flushing heads covered) are flushed
        // first, so the parking columns are free for the next item
        if (qpend) {
          for (int j = it.nh; j < qnh; ++j)
            if ((j & 1) == G) flush_head(j);
        }
        sRed[(2 * G + hf) * kQ + r] = fmaxf(__low2float(amax2), __high2float(amax2));
        tc_fence_before();  // parked TMEM stores ordered before the other group's later reads
        both_sync();
        tc_fence_after();
        const float am = fmaxf(fmaxf(sRed[r], sRed[kQ + r]), fmaxf(sRed[2 * kQ + r], sRed[3 * kQ + r]));
        both_sync();  // both groups read sRed before the next item's writes
        amax2 = __float2half2_rn(0.0f);
        qb = it.b;
        qhbase = it.h0;
        qnh = it.nh;
        qpend = true;
        qsc = q8_scale(am);
        qrs = __frcp_rn(qsc);
        if (G == 0 && hf == 0 && r < S) ctxs[(size_t)it.b * S + r] = qsc;
      }
    }
    if (fuse_q && qpend)
      for (int j = 0; j < qnh; ++j)
        if ((j & 1) == G) flush_head(j);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

// TMA addresses a head slice only when it starts on a 16-byte boundary
// (2 hs % 16 == 0).  TinyBERT's d = 26 is therefore stored with head stride
// hs = 32 (the QKV GEMM writes zero-padded heads, ff_api.cu); unpadded, it
// would start at byte 52 h (a 4-byte cp.async producer for that layout
// measured 99 us per C2 launch, 2.4x the mma.sync kernel).
bool attention_tc_supported(int S, int d, int hs, int ldqkv, int ldctx) {
  const bool shape = (d == 64 && hs == 64) || (d >= 2 && d % 2 == 0 && d <= hs && hs <= 32 && (2 * hs) % 16 == 0);
  return shape && S >= 1 && S <= kKeys && (ldqkv % 8) == 0 && (ldctx % 2) == 0;
}

bool attention_tc_fuses_quant(int A, int d) { return A >= 1 && A <= (d <= 32 ? 16 : 8); }

bool plan_attention_tc(AttnTCPlan* plan, const void* qkv, int M_rows, int ldqkv, const char** err) {
  // [M_rows x ldqkv] fp16, 64-column x 128-row boxes, 128B swizzle
  plan->qkv = qkv;
  plan->ldqkv = ldqkv;
  plan->hm_rows = 0;
  return make_operand_map(&plan->map, qkv, M_rows, ldqkv, 2, (size_t)ldqkv * 2, 128, err);
}

bool plan_attention_tc_hm(AttnTCPlan* plan, const void* qkv, int n_blocks, int hm_rows, const char** err) {
  // [n_blocks * hm_rows x 64] fp16 (128-byte rows), 128-row boxes, 128B swizzle
  plan->qkv = qkv;
  plan->ldqkv = 64;
  plan->hm_rows = hm_rows;
  return make_operand_map(&plan->map, qkv, n_blocks * hm_rows, 64, 2, 128, 128, err);
}

cudaError_t prepare_attention_tc_kernel() {
  cudaError_t e = cudaFuncSetAttribute(attention_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SmemTC::TOTAL);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(attention_tc_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemTC::TOTAL);
}

// Heads per work item: the whole row (A heads) when the ctx requant is fused
// (its row amax needs every head); otherwise the item size that minimises the
// heads on the busiest CTA (ties: larger items, fewer item switches), so small
// batches still spread over all SMs (C2: 64 sequences x 12 heads).
static int heads_per_item(int B, int A, int max_heads, bool fused) {
  if (fused) return A;
  int best = max_heads < A ? max_heads : A;
  long long best_cost = -1;
  for (int mh = best; mh >= 1; --mh) {
    const long long items = (long long)B * ((A + mh - 1) / mh);
    const long long cost = ((items + kNumSMs - 1) / kNumSMs) * mh;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = mh;
    }
  }
  return best;
}

cudaError_t launch_attention_tc(const AttnTCPlan& plan, const int32_t* mask, int B, int S, int A, int d, int hs,
                                __half* ctx, int ldctx, int8_t* ctxq, int ldq, float* ctxs, cudaStream_t s,
                                unsigned long long* trace, int rev) {
  if (ctxq != nullptr && !attention_tc_fuses_quant(A, d)) return cudaErrorInvalidValue;
  const float scale = (float)(1.0 / sqrt((double)d));  // fp32(1/sqrt(d)) (R10)
  const int max_heads = d <= 32 ? HeadCfg<32>::kMaxHeads : HeadCfg<64>::kMaxHeads;
  const int mh = heads_per_item(B, A, max_heads, ctxq != nullptr);
  const int n_items = B * ((A + mh - 1) / mh);
  const int grid = n_items < kNumSMs ? n_items : kNumSMs;
  if (d <= 32)
    launch_ex(attention_tc_kernel<32>, dim3(grid), dim3(kThreadsTC), SmemTC::TOTAL, s, 0, plan.map, mask, B, S, A, d,
              hs, mh, plan.hm_rows, scale, ctx, ldctx, ctxq, ldq, ctxs, static_cast<const uint8_t*>(plan.qkv),
              plan.ldqkv * 2, trace, rev);
  else
    launch_ex(attention_tc_kernel<64>, dim3(grid), dim3(kThreadsTC), SmemTC::TOTAL, s, 0, plan.map, mask, B, S, A, d,
              hs, mh, plan.hm_rows, scale, ctx, ldctx, ctxq, ldq, ctxs, static_cast<const uint8_t*>(plan.qkv),
              plan.ldqkv * 2, trace, rev);
  return cudaGetLastError();
}

}  // namespace ff
