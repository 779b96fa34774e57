// gemm_tc.cu -- the four constant-weight GEMMs of every encoder layer
// (fused QKV, out-proj, FFN1, FFN2) on the 5th-gen
// tensor cores.
//
//   C[M,N] = A[M,K] * W[N,K]^T  (both operands K-major, PyTorch [out,in] W)
//   fp16 layers: tcgen05.mma kind::f16, fp32 accumulate
//   int8 layers: tcgen05.mma kind::i8,  s32 accumulate (exact)
//
// Persistent, warp-specialised kernel, one CTA (or CTA pair) per SM, 640 threads:
//   warp 0      TMA producer: 128x128B A tile + (BN or BN/2)x128B W tile per
//               k-block into a STAGES-deep ring of 128B-swizzled smem tiles
//               (mbarrier full/empty); CTA pairs (cta_group::2) split W
//   warp 1      MMA issuer: one thread issues 4 x tcgen05.mma (K = 32 bytes each)
//               per k-block into a double-buffered TMEM accumulator (2 x BN cols)
//   warp 2      TMEM allocator
//   warps 4-19  epilogue: warp w drains TMEM lane quadrant w%4, column quarter
//               (w-4)/4, with tcgen05.ld 32x32b.x16 (thread = output row) in
//               32-column chunks, applies the fused epilogue on packed fp32
//               pairs, writes fp16 into a 64B-swizzled smem staging block and
//               issues a TMA bulk-tensor store per 32x32 block; bias / column
//               scales are staged in smem per tile; the accumulator is released
//               as soon as its last TMEM load completed, so the next tile's
//               mainloop overlaps this epilogue.
// Epilogue (out_mode 1):
//   fp16: y = acc + b[n]
//   int8: y = fma(float(acc), sx[m]*sw[n], b[n])          (DESIGN R13, bit-exact)
//         per-tensor u8 variant (PT): acc - zp * colsum[n] first (R22)
//   then optional activation (GELU-erf / ReLU / GELU-tanh) in fp32 and
//   RNE to fp16.  out_mode 0 stores the raw 32-bit accumulators (tests only).
#include <cstdio>
#include "ff_kernels.h"
#include "ptx.cuh"
#include "quant.cuh"

namespace ff {

constexpr int BM = 128;
constexpr int BK_BYTES = 128;  // one 128-byte swizzle row of K per k-block
// gemm_tc_kernel: 16 epilogue warps (4 per TMEM lane quadrant, each owning a
// quarter of the tile's columns), 32-column chunks, 32x32 fp16 staging blocks
// stored with 64B swizzle.  <= 96 registers per thread at 640 threads.
constexpr int kEpiWarps = 16;
constexpr int kThreads = 128 + 32 * kEpiWarps;
constexpr int kEpiCols = 32;                     // columns per epilogue chunk (two 16-column TMEM loads)
constexpr int kStageTile = 32 * kEpiCols * 2;  // 2 KB: 32 rows x 64 B, 64-byte swizzle
constexpr int kStageBufs = 1;                  // staging buffers per epilogue warp
// gemm_rr_kernel: 16 epilogue warps (4 per quadrant, 64 columns each),
// 32-column chunks, 32x32 fp16 staging blocks with 64B swizzle.
constexpr int kRREpiWarps = 16;
constexpr int kRRThreads = 128 + 32 * kRREpiWarps;
constexpr int kRRStageTile = 32 * 64;  // 2 KB

// PAIR = CTA pair (cta_group::2): a 256-row tile per pair, each CTA loads its
// 128 rows of A and its BN/2 rows of W, the leader issues M=256 MMAs.
template <int BN, bool PAIR>
struct GemmCfg {
  static constexpr int TM = PAIR ? 256 : 128;  // rows per (pair-)tile
  static constexpr int A_BYTES = BM * BK_BYTES;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (PAIR || BN == 128) ? 5 : 3;
  static constexpr int EPI_OFF = STAGES * STAGE_BYTES;
  // [acc][bias | col scale | weight column sums (int)][BN]
  static constexpr int PAR_OFF = EPI_OFF + kEpiWarps * kStageBufs * kStageTile;
  static constexpr int BAR_OFF = PAR_OFF + 2 * 3 * BN * 4;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;  // barriers + 1 KB alignment slack
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static_assert(SMEM <= 227 * 1024, "smem budget");
};

// Instruction descriptor (kind::f16 / kind::i8), both operands K-major:
// c_format [4,6) (1 = f32, 2 = s32), a_format [7,10), b_format [10,13)
// (f16 = 0; s8 = 1), N>>3 at [17,23), M>>4 at [24,29).
template <bool I8, int TM, int BN>
__device__ __forceinline__ constexpr uint32_t make_idesc() {
  return (I8 ? (2u << 4) : (1u << 4)) | (I8 ? (1u << 7) : 0u) | (I8 ? (1u << 10) : 0u) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}

// GELU(y) = y/2 (1 + erf(y / sqrt 2)) for the FFN1 epilogue.
// With s = |y| and e = erfc(s / sqrt 2) = 2^(-s * P(s)):  GELU(y) = y/2 * (2 - e)
// for y >= 0 and y/2 * e for y < 0 -- no cancellation on the negative side.
// P is a Chebyshev-weighted fit of -log2(erfc(s / sqrt 2)) / s:
//   P7  on [0, 2.5] (relative error of e <= 1.6e-8): the fast path;
//   P11 on [0, 6.5] (<= 1.2e-8; s clamped to 6.5, beyond which GELU(y) rounds
//       to y, resp. to 0 in fp16): used for elements with s > 2.5 only.
// The choice is per ELEMENT (s <= 2.5 -> P7), so an output depends on its own
// input alone (batch / padding invariance stay bit-exact); the warp only
// evaluates P11 when one of its 32 x 32 chunk values has s > 2.5 (rare: the
// FFN1 pre-activations are ~N(0, 0.55) on the synthetic C3 weights).
// Measured on the GPU (tools/micro/exp_accuracy.cu, 2^28 points): 0.0066% of
// outputs whose fp16 rounding differs from RN16(RN32(exact GELU)) -- the
// oracle's rounding point (DESIGN R2) -- against 0.21% for the round-1
// degree-6 fit.  Replaces erff, whose divergent branches made the FFN1
// epilogue the GEMM's bottleneck.
// Coefficients, highest degree first (Horner).
#define FF_GELU_P7(X)                                                                                         \
  X(3.84035457e-06f) X(-4.82531614e-05f) X(2.16719927e-04f) X(8.50132710e-05f) X(-7.01780897e-03f)          \
  X(5.24765067e-02f) X(4.59211707e-01f) X(1.15110505e+00f)
#define FF_GELU_P11(X)                                                                                        \
  X(1.91209187e-10f) X(-8.90500740e-09f) X(1.86934614e-07f) X(-2.33101059e-06f) X(1.90286646e-05f)           \
  X(-1.03522529e-04f) X(3.35359509e-04f) X(-6.75584961e-05f) X(-6.90312125e-03f) X(5.24297878e-02f)          \
  X(4.59220439e-01f) X(1.15110457e+00f)
constexpr float kGeluFast = 2.5f;
constexpr float kGeluClamp = 6.5f;

// s * P(s) for one value: P7 when s <= 2.5, else P11 of min(s, 6.5).
__device__ __forceinline__ float gelu_expo(float s) {
  // (Horner starts from the leading coefficient: fma(0, s, c) is not folded
  // by the compiler -- 0 * inf -- and would cost an instruction per value)
  float p7 = 0.0f, p11 = 0.0f;
  bool f7 = true, f11 = true;
  const float sc = fminf(s, kGeluClamp);
#define FF_H7(c) p7 = f7 ? (c) : __fmaf_rn(p7, s, c); f7 = false;
#define FF_H11(c) p11 = f11 ? (c) : __fmaf_rn(p11, sc, c); f11 = false;
  FF_GELU_P7(FF_H7)
  FF_GELU_P11(FF_H11)
#undef FF_H7
#undef FF_H11
  return s <= kGeluFast ? s * p7 : sc * p11;
}

// GELU(y) = y/2 (2 - e) for y >= 0, y/2 e for y < 0, written without a
// select as 0.5 * fma(-|y|, e, y + |y|) (y + |y| is 2y or 0, exact; one
// rounding for y >= 0, the same value as (0.5 y) e for y < 0).
__device__ __forceinline__ float gelu_from_expo(float y, float a) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-a));
  const float s = fabsf(y);
  return 0.5f * __fmaf_rn(-s, e, y + s);
}

template <int ACT>
__device__ __forceinline__ float act_fn(float y) {
  if (ACT == ACT_GELU) return gelu_from_expo(y, gelu_expo(fabsf(y)));
  if (ACT == ACT_RELU) return fmaxf(y, 0.0f);
  if (ACT == ACT_GELU_TANH) {
    const float u = 0.7978845608028654f * (y + 0.044715f * y * y * y);
    return 0.5f * y * (1.0f + tanhf(u));
  }
  return y;
}

// GELU of 16 pairs on packed fp32 (FFMA2 / FMUL2): the fast P7 path for the
// whole warp unless some element has s > 2.5; then every element takes the
// per-element choice of gelu_expo (identical results for s <= 2.5).
__device__ __forceinline__ void gelu16x2(float2 (&v)[16]) {
  float m = 0.0f;
#pragma unroll
  for (int e = 0; e < 16; ++e) m = fmaxf(m, fmaxf(fabsf(v[e].x), fabsf(v[e].y)));
  if (__any_sync(0xffffffffu, m > kGeluFast)) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      v[e].x = gelu_from_expo(v[e].x, gelu_expo(fabsf(v[e].x)));
      v[e].y = gelu_from_expo(v[e].y, gelu_expo(fabsf(v[e].y)));
    }
    return;
  }
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const float2 s = make_float2(fabsf(v[e].x), fabsf(v[e].y));
    float2 p = make_float2(0.0f, 0.0f);
    bool first = true;  // Horner from the leading coefficient (see gelu_expo)
#define FF_H2(c) p = first ? make_float2(c, c) : fma2(p, s, make_float2(c, c)); first = false;
    FF_GELU_P7(FF_H2)
#undef FF_H2
    const float2 a = mul2(s, p);
    float2 ex;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex.x) : "f"(-a.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex.y) : "f"(-a.y));
    // select-free tail (gelu_from_expo): 0.5 * fma(-s, e, y + s)
    const float2 h = add2(v[e], s);
    v[e] = mul2(fma2(make_float2(-s.x, -s.y), ex, h), make_float2(0.5f, 0.5f));
  }
}

// 32 columns of this thread's row (r[0]: columns 0-15, r[1]: 16-31), bias /
// column scales read from smem (bs / ss, broadcast LDS.64 per pair):
// dequant / bias / activation, RNE to fp16, packed as 16 half2 words.
// PT (per-tensor u8 activations, DESIGN R22): acc - zp * colsum[n] (exact
// in int32, cs = column sums) replaces acc; PT = false: per-row s8 scheme.
template <bool I8, int ACT, bool PT = false>
__device__ __forceinline__ void epi32(const uint32_t (&r)[2][16], const float* bs, const float* ss, float sx,
                                      uint32_t (&h)[16], const int* cs = nullptr, int zp = 0) {
  float2 v[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int j = 2 * e;
    uint32_t r0 = r[j >> 4][j & 15], r1 = r[j >> 4][(j & 15) + 1];
    if (I8 && PT) {
      const int2 c2 = *reinterpret_cast<const int2*>(cs + j);
      r0 = (uint32_t)((int)r0 - zp * c2.x);
      r1 = (uint32_t)((int)r1 - zp * c2.y);
    }
    const float2 b = *reinterpret_cast<const float2*>(bs + j);
    if (I8) {
      const float2 sw2 = *reinterpret_cast<const float2*>(ss + j);
      const float2 a = make_float2(__int2float_rn(static_cast<int>(r0)), __int2float_rn(static_cast<int>(r1)));
      v[e] = fma2(a, mul2(make_float2(sx, sx), sw2), b);
    } else {
      v[e] = add2(make_float2(__uint_as_float(r0), __uint_as_float(r1)), b);
    }
  }
  if (ACT == ACT_GELU) {
    gelu16x2(v);
  } else if (ACT != ACT_NONE) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      v[e].x = act_fn<ACT>(v[e].x);
      v[e].y = act_fn<ACT>(v[e].y);
    }
  }
#pragma unroll
  for (int e = 0; e < 16; ++e) h[e] = pack_half2(v[e].x, v[e].y);
}


// tcgen05.ld of 16 columns (32x32b.x16): thread t gets row (lane base + t).

// Debug timeline: globaltimer of event e for local tile t of CTA c at
// trace[(c * kTraceTiles + t) * 24 + e] (events: 0 acc free seen by MMA, 1
// first operands seen, 2 accumulator committed, 3 tfull seen by epilogue
// warp 0, 4 accumulator released, 5 epilogue done, 6 first load issued;
// epilogue warp 0, chunk i < 4: 8+3i TMEM load landed, 9+3i staging buffer
// free, 10+3i store issued).
constexpr int kTraceTiles = 64;
__device__ __forceinline__ void gemm_trace(unsigned long long* trace, int t, int e) {
  if (trace != nullptr && t < kTraceTiles) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    trace[((size_t)blockIdx.x * kTraceTiles + t) * 24 + e] = v;
  }
}

// PT: per-tensor u8 activations with a zero point (DESIGN R22; I8 only), a
// separate instantiation so the per-row kernel's registers are unaffected.
// (Measured and removed: W multicast across clusters of two CTA pairs, and
// splitting the last partial wave of pair tiles into half-width tiles; DESIGN
// section 6.)
template <int BN, bool I8, bool PAIR, bool PT = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, GemmParams p) {
  using Cfg = GemmCfg<BN, PAIR>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int TM = Cfg::TM;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sEpi = smem + Cfg::EPI_OFF;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;  // 0 = leader of the pair
  const int unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int nunits = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (p.out_mode == 1) tma_prefetch(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], (PAIR ? 2 : 1) * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if (PAIR) {
      tmem_alloc2(tmem_slot, Cfg::TMEM_COLS);
      tmem_relinquish2();
    } else {
      tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // peer barriers initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // A operand / scales come from the previous kernel
  griddep_launch();

  const int num_tiles = p.m_tiles * p.n_tiles;
  constexpr int KE = I8 ? 128 : 64;  // elements per k-block

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int lt = 0;
      for (int tile = unit; tile < num_tiles; tile += nunits, ++lt) {
        const int mt0 = tile / p.n_tiles, nt = tile - mt0 * p.n_tiles;
        const int mt = p.rev ? p.m_tiles - 1 - mt0 : mt0;
        const int arow = mt * TM + (int)rank * BM;
        const int brow = nt * BN + (PAIR ? (int)rank * (BN / 2) : 0);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (kb == 0) gemm_trace(p.trace, lt, 6);
          if (p.dbg_noload) {  // MMA-rate probe: operands left as they are in smem
            if (rank == 0) mbar_arrive(&full[stage]);
          } else if (PAIR) {
            // the leader's full barrier counts the bytes of both CTAs' loads
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
            const uint32_t bar = mapa_shared(smem_u32(&full[stage]), 0);
            tma_load_2d_pair(sA + stage * Cfg::A_BYTES, &tmA, bar, kb * KE, arow, kEvictNormal);
            tma_load_2d_pair(sB + stage * Cfg::B_BYTES, &tmB, bar, kb * KE, brow, kEvictLast);
          } else {
            mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
            tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * KE, arow, kEvictNormal);
            tma_load_2d(sB + stage * Cfg::B_BYTES, &tmB, &full[stage], kb * KE, brow, kEvictLast);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // per-tensor u8 activations (DESIGN R22): a_format u8 (bit 7 clear)
      constexpr uint32_t idesc = make_idesc<I8, TM, BN>() & (PT ? ~(1u << 7) : ~0u);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int lt = 0;
      for (int tile = unit; tile < num_tiles; tile += nunits, ++lt) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        gemm_trace(p.trace, lt, 0);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          if (kb == 0) gemm_trace(p.trace, lt, 1);
          tc_fence_after();
          const uint64_t adesc = make_sw128_desc(sA + stage * Cfg::A_BYTES);
          const uint64_t bdesc = make_sw128_desc(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 4 x 32 bytes of K; +2 = +32 B in the >>4 address field
            const uint32_t accum = (kb | k) != 0;
            if (PAIR) {
              if (I8) mma_i8_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, accum);
              else mma_f16_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, accum);
            } else {
              if (I8) mma_i8(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, accum);
              else mma_f16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, accum);
            }
          }
          // frees the smem slot (of both CTAs) when these MMAs finish
          if (PAIR) mma_commit_pair(&empty[stage], 0x3);
          else mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        // accumulator ready for the epilogue warps (of both CTAs)
        if (PAIR) mma_commit_pair(&tfull[acc], 0x3);
        else mma_commit(&tfull[acc]);
        gemm_trace(p.trace, lt, 2);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int q = warp & 3;                         // TMEM lane quadrant this warp may access
    constexpr int WCOLS = BN / (kEpiWarps / 4);     // columns per warp (64 or 32)
    uint8_t* stage_buf = sEpi + ew * kStageBufs * kStageTile;
    const uint32_t tempty_leader0 = PAIR ? mapa_shared(smem_u32(&tempty[0]), 0) : 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int nbuf = 0;
    int lt = 0;
    const bool tr0 = ew == 0 && lane == 0;
    float* sPar = reinterpret_cast<float*>(smem + Cfg::PAR_OFF);
    const int et = ew * 32 + lane;  // 0 .. 511
    for (int tile = unit; tile < num_tiles; tile += nunits, ++lt) {
      const int mt0 = tile / p.n_tiles, nt = tile - mt0 * p.n_tiles;
        const int mt = p.rev ? p.m_tiles - 1 - mt0 : mt0;
      const int nb = nt * BN;  // first output column of this tile
      constexpr int wcols = WCOLS;
      const int c_lo = (ew >> 2) * wcols;  // this warp's column group of the tile
      const int row0 = mt * TM + (int)rank * BM + q * 32;
      const int row = row0 + lane;
      float sx = 0.0f;
      if (I8 && p.out_mode == 1 && row < p.M) sx = PT ? p.tensor_qp[0] : p.row_scale[(size_t)row * p.rs_stride];
      const int zp = (PT && p.out_mode == 1) ? (int)p.tensor_qp[1] : 0;
      // this tile's bias / column scales -> smem (double-buffered by acc; the
      // barrier of tile t+1 orders every warp's reads of tile t before the
      // writes of tile t+2), read by the chunks with low-latency LDS
      float* par = sPar + acc * 3 * BN;
      if (p.out_mode == 1) {
        const int npar = PT ? 3 * BN : 2 * BN;
        for (int i = et; i < npar; i += 32 * kEpiWarps) {
          const int col = nb + (i % BN);
          if (i < 2 * BN) {
            const float* src = i < BN ? p.bias : p.col_scale;
            par[i] = (src != nullptr && col < p.N) ? __ldg(src + col) : 0.0f;
          } else {
            reinterpret_cast<int*>(par)[i] = (p.colsum != nullptr && col < p.N) ? __ldg(p.colsum + col) : 0;
          }
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
      mbar_wait(&tfull[acc], acc_phase);
      if (tr0) gemm_trace(p.trace, lt, 3);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      // Release the accumulator to the MMA warp as soon as this warp's last
      // TMEM load has completed (before its math and stores).
      auto release_acc = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) mbar_arrive_remote(tempty_leader0 + acc * 8);  // the leader's barrier
          else mbar_arrive(&tempty[acc]);
        }
        if (tr0) gemm_trace(p.trace, lt, 4);
      };
      if (p.out_mode == 0) {  // raw accumulators (tests only)
#pragma unroll 1
        for (int c = c_lo; c < c_lo + wcols; c += kEpiCols) {
          uint32_t r[kEpiCols];
          tmem_ld32(tbase + c, r);
          tmem_wait_ld();
          const int n0 = nb + c;
          if (row < p.M && n0 < p.N) {
            uint32_t* o = reinterpret_cast<uint32_t*>(p.out) + (size_t)row * p.ldo + n0;
#pragma unroll
            for (int j = 0; j < kEpiCols; ++j)
              if (n0 + j < p.N) o[j] = r[j];
          }
        }
        release_acc();
      } else {
        // software pipeline: the TMEM loads of chunk c+1 overlap the stores of chunk c
        uint32_t r[2][16];
        tmem_ld16(tbase + c_lo, r[0]);
        tmem_ld16(tbase + c_lo + 16, r[1]);
#pragma unroll 1
        for (int c = c_lo; c < c_lo + wcols; c += kEpiCols) {
          const int n0 = nb + c;
          const bool last = c + kEpiCols >= c_lo + wcols;
          tmem_wait_ld();
          const int ci = (c - c_lo) / kEpiCols;
          if (tr0 && ci < 4) gemm_trace(p.trace, lt, 8 + 3 * ci);
          if (last) release_acc();
          uint32_t h[16];
          if (PT) {  // per-tensor u8 activations
            const int* cs = reinterpret_cast<const int*>(par + 2 * BN + c);
            switch (p.act) {
              case ACT_GELU: epi32<I8, ACT_GELU, true>(r, par + c, par + BN + c, sx, h, cs, zp); break;
              case ACT_RELU: epi32<I8, ACT_RELU, true>(r, par + c, par + BN + c, sx, h, cs, zp); break;
              case ACT_GELU_TANH: epi32<I8, ACT_GELU_TANH, true>(r, par + c, par + BN + c, sx, h, cs, zp); break;
              default: epi32<I8, ACT_NONE, true>(r, par + c, par + BN + c, sx, h, cs, zp); break;
            }
          } else {
            switch (p.act) {
              case ACT_GELU: epi32<I8, ACT_GELU>(r, par + c, par + BN + c, sx, h); break;
              case ACT_RELU: epi32<I8, ACT_RELU>(r, par + c, par + BN + c, sx, h); break;
              case ACT_GELU_TANH: epi32<I8, ACT_GELU_TANH>(r, par + c, par + BN + c, sx, h); break;
              default: epi32<I8, ACT_NONE>(r, par + c, par + BN + c, sx, h); break;
            }
          }
          if (!last) {
            tmem_ld16(tbase + c + kEpiCols, r[0]);
            tmem_ld16(tbase + c + kEpiCols + 16, r[1]);
          }
          if (tr0 && ci < 4) gemm_trace(p.trace, lt, 20 + ci);
          if (n0 < p.N && row0 < p.M) {  // warp-uniform; TMA clips the N tail of the chunk
            uint8_t* buf = stage_buf + (nbuf % kStageBufs) * kStageTile;
            if (lane == 0) bulk_wait_read<kStageBufs - 1>();  // the store that last used `buf` has read it
            __syncwarp();
            if (tr0 && ci < 4) gemm_trace(p.trace, lt, 9 + 3 * ci);
            uint8_t* srow = buf + lane * 64;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {  // SWIZZLE_64B: 16B chunk cc of 64B row `lane`
              const int pc = cc ^ ((lane >> 1) & 3);
              *reinterpret_cast<uint4*>(srow + pc * 16) =
                  make_uint4(h[4 * cc], h[4 * cc + 1], h[4 * cc + 2], h[4 * cc + 3]);
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (p.hm_rows > 0) tma_store_2d(&tmC, buf, n0 & 63, (n0 >> 6) * p.hm_rows + row0);
              else tma_store_2d(&tmC, buf, n0, row0);
              bulk_commit();
            }
            if (tr0 && ci < 4) gemm_trace(p.trace, lt, 10 + 3 * ci);
            ++nbuf;
          }
        }
      }
      if (tr0) gemm_trace(p.trace, lt, 5);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // no CTA leaves while its peer may still signal it
  if (warp == 2) {
    tc_fence_after();
    if (PAIR) tmem_dealloc2(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ========================================================================
// Row-reduction GEMM: C tile rows span a cluster of CN CTAs along N (one
// 128x256 tile per CTA; CTA `rank` always owns columns [256 rank, +256), so
// its bias / column scales / LN gamma, beta are staged in smem once).
// Same producer / MMA roles as gemm_tc_kernel (single-CTA MMA, 3 smem
// stages, double-buffered TMEM accumulator).  The 16 epilogue warps form TWO
// groups of 8 that ping-pong: group G drains accumulator buffer G, i.e. every
// other tile, so one group's cluster exchanges, barriers and store waits
// overlap the other group's arithmetic (the epilogue is FMA-pipe and
// latency bound, not TMEM bound: tcgen05.ld reads ~900 B/clk/SM,
// tools/micro/tmem_bw.cu).  In a group, warp (q, hc) owns rows [32q, +32) x
// columns [128hc, +128) of the tile, in 4 chunks of 32; intermediates stay in
// the group's own accumulator columns (x as fp32, then the packed fp16
// results), which are released to the MMA warp after the last pass.  Row
// statistics: the 2 column-half partials of a row are combined inside the
// CTA (smem, 64-thread named barrier per quadrant), the CTA partial is
// bulk-copied into every CTA of the cluster (cp.async.bulk.shared::cluster,
// completion on an mbarrier armed with the expected bytes), and every CTA
// combines the CN partials in the same fixed order, so all derive
// bit-identical statistics.  Exchange buffers are per group (x2 in flight).
//   RR_LN:    x = R16(dequant(acc) + bias) + residual (R11); LN over the row
//             (per-thread two-pass mean / M2, Chan combination); y16 = R16(LN)
//             -> fp16 rows (TMA) [+ Q8row s8 rows + scale]
//   RR_QUANT: y16 = R16(act(dequant(acc) + bias)) [-> fp16 rows]; Q8row s8
//             rows + scale (the FFN-intermediate requant)
// ========================================================================
constexpr int kRRStages = 3;
#ifndef FF_RR_SLEEP_NS
#define FF_RR_SLEEP_NS 128
#endif
constexpr uint32_t kRRSleepNs = FF_RR_SLEEP_NS;  // epilogue group's probe interval while its accumulator is computed
constexpr int kRRBN = 256;
// PARK (RR_LN): the LN output row is parked in registers instead of TMEM, so
// the accumulator returns to the MMA warp before the amax exchange and the
// requant; warpgroup 0 hands registers to the epilogue (setmaxnreg).
constexpr uint32_t kRRRegsCtl = 40;
constexpr uint32_t kRRRegsEpi = 104;  // 128 x 40 + 512 x 104 <= 640 x 96
static_assert(128 * kRRRegsCtl + 32 * kRREpiWarps * kRRRegsEpi <= kRRThreads * 96, "register pool");
constexpr int kRRParkKBlocks = 8;
constexpr int kRRMaxCN = 8;
constexpr int kRRGroupWarps = kRREpiWarps / 2;  // 8 warps per ping-pong group
struct RRCfg {
  static constexpr int A_BYTES = BM * BK_BYTES;
  static constexpr int B_BYTES = kRRBN * BK_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_OFF = kRRStages * STAGE_BYTES;                 // staging [warp] 2 KB
  static constexpr int PAR_OFF = EPI_OFF + kRREpiWarps * kRRStageTile;    // [bias|sw|gamma|beta][256] fp32
  static constexpr int LOC_OFF = PAR_OFF + 4 * kRRBN * 4;                 // [G 2][par 2][hc 2][q 4][v 2][32] fp32
  static constexpr int RED_OFF = LOC_OFF + 2 * 2 * 2 * 4 * 2 * 32 * 4;    // [b 4][rank 8][q 4][v 2][32] fp32
  static constexpr int BAR_OFF = RED_OFF + 4 * kRRMaxCN * 4 * 2 * 32 * 4;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;
  static_assert(SMEM <= 227 * 1024, "smem budget");
};

template <bool I8, int MODE, bool PARK = false>
__global__ void __launch_bounds__(kRRThreads, 1)
    gemm_rr_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmR,
                   const __grid_constant__ CUtensorMap tmQ, RRParams p) {
  constexpr int STAGES = kRRStages;
  constexpr int BN = kRRBN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * RRCfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RRCfg::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* redbar = tempty + 2;  // [4] = [group][exchange parity]
  uint64_t* resbar = redbar + 4;  // [kRREpiWarps] per-warp residual TMA loads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(resbar + kRREpiWarps);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int CN = (int)cluster_nctarank();
  const int unit = (int)blockIdx.x / CN;
  const int nunits = (int)gridDim.x / CN;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (p.store16) tma_prefetch(&tmC);
    if (MODE == RR_LN) tma_prefetch(&tmR);
    if (p.outq) tma_prefetch(&tmQ);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kRRGroupWarps);  // the 8 warps of the group draining buffer a
    }
    for (int b = 0; b < 4; ++b) mbar_init(&redbar[b], 1);
    for (int w = 0; w < kRREpiWarps; ++w) mbar_init(&resbar[w], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 2 * BN);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // every CTA's reduction barriers exist before any remote copy
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // A operand / scales / residual come from the previous kernel
  griddep_launch();
  constexpr int KE = I8 ? 128 : 64;

  if (warp < 4) {
    if constexpr (PARK) regs_dec<kRRRegsCtl>();
    if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int mt = unit; mt < p.m_tiles; mt += nunits) {
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], RRCfg::STAGE_BYTES);
          tma_load_2d(sA + stage * RRCfg::A_BYTES, &tmA, &full[stage], kb * KE, (p.rev ? p.m_tiles - 1 - mt : mt) * BM, kEvictNormal);
          tma_load_2d(sB + stage * RRCfg::B_BYTES, &tmB, &full[stage], kb * KE, (int)rank * BN, kEvictLast);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc<I8, BM, BN>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int lt = 0;
      for (int mt = unit; mt < p.m_tiles; mt += nunits, ++lt) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        gemm_trace(p.trace, lt, 0);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          if (kb == 0) gemm_trace(p.trace, lt, 1);
          tc_fence_after();
          const uint64_t adesc = make_sw128_desc(sA + stage * RRCfg::A_BYTES);
          const uint64_t bdesc = make_sw128_desc(sB + stage * RRCfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (I8) mma_i8(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            else mma_f16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
        gemm_trace(p.trace, lt, 2);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    }
  } else {
    if constexpr (PARK) regs_inc<kRRRegsEpi>();
    const int ew = warp - 4;
    const int G = ew / kRRGroupWarps;          // ping-pong group: accumulator buffer G, local tiles lt % 2 == G
    const int q = warp & 3;                    // TMEM lane quadrant: rows [32q, 32q+32)
    const int hc = (ew % kRRGroupWarps) >> 2;  // column half: [128hc, 128hc+128) of the CTA's 256
    const int c_lo = hc * 128;
    const int ncol0 = (int)rank * BN;
    float* par = reinterpret_cast<float*>(smem + RRCfg::PAR_OFF);
    float* loc = reinterpret_cast<float*>(smem + RRCfg::LOC_OFF);
    float* red = reinterpret_cast<float*>(smem + RRCfg::RED_OFF);
    uint8_t* stage_buf = smem + RRCfg::EPI_OFF + ew * kRRStageTile;
    // this CTA's column parameters, once: bias, column scale, gamma, beta
    for (int i = ew * 32 + lane; i < 4 * BN; i += 32 * kRREpiWarps) {
      const int kind = i / BN, col = ncol0 + (i % BN);
      const float* src = kind == 0 ? p.bias : kind == 1 ? p.col_scale : kind == 2 ? p.gamma : p.beta;
      par[i] = (src != nullptr && col < p.N) ? __ldg(src + col) : 0.0f;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kRREpiWarps) : "memory");
    const float* pbias = par + c_lo;
    const float* psw = par + BN + c_lo;
    const float* pgam = par + 2 * BN + c_lo;
    const float* pbet = par + 3 * BN + c_lo;
    const int qbar = 2 + G * 4 + q;  // named barrier of the group's two warps on quadrant q

    int step = 0;  // this group's exchange counter (buffer 2G + (step & 1), phase (step >> 1) & 1)
    // Row combine of per-thread values: in-CTA over the 2 column halves, then
    // across the cluster.  STATS: (mean, M2) of 128 values each -> (mean, M2)
    // of the full row; MAX: max.  Every thread returns the row result.
    auto exchange = [&](float v0, float v1, bool stats, float& o0, float& o1) {
      const int nv = stats ? 2 : 1;
      const int b = 2 * G + (step & 1);
      const uint32_t ph = (uint32_t)(step >> 1) & 1u;
      // in-CTA partials, double-buffered by exchange parity so that the next
      // exchange's writes never alias the combining warp's reads
      float* lg = loc + (2 * G + (step & 1)) * (2 * 4 * 2 * 32);
      lg[((hc * 4 + q) * 2 + 0) * 32 + lane] = v0;
      if (stats) lg[((hc * 4 + q) * 2 + 1) * 32 + lane] = v1;
      asm volatile("bar.sync %0, 64;" ::"r"(qbar) : "memory");
      if (hc == 0) {
        float r0, r1 = 0.0f;
        const float a0 = lg[((0 * 4 + q) * 2) * 32 + lane], a1 = lg[((1 * 4 + q) * 2) * 32 + lane];
        if (stats) {
          r0 = (a0 + a1) * 0.5f;
          const float d0 = a0 - r0, d1 = a1 - r0;
          const float m0 = lg[((0 * 4 + q) * 2 + 1) * 32 + lane], m1 = lg[((1 * 4 + q) * 2 + 1) * 32 + lane];
          r1 = (m0 + m1) + 128.0f * (d0 * d0 + d1 * d1);
        } else {
          r0 = fmaxf(a0, a1);
        }
        if (CN == 1) {  // a one-CTA cluster: the CTA partial is the row result
          float* slot = red + (((b * kRRMaxCN) * 4 + q) * 2) * 32;
          slot[lane] = r0;
          if (stats) slot[32 + lane] = r1;
        } else {
          // every lane stores its row's partial into slot `rank` of every
          // CTA of the cluster (st.async: remote smem stores counted on the
          // destination's mbarrier; no trip through the bulk-copy engine,
          // which queues behind the mainloop's operand loads)
          if (lane == 0 && q == 0) mbar_expect_tx(&redbar[b], (uint32_t)(CN * 4 * nv * 128));
          const uint32_t dst = smem_u32(red + (((b * kRRMaxCN + (int)rank) * 4 + q) * 2) * 32 + lane);
          const uint32_t bl = smem_u32(&redbar[b]);
          for (int c = 0; c < CN; ++c) {
            const uint32_t rb = mapa_shared(bl, c), rd = mapa_shared(dst, c);
            st_async_f32(rd, r0, rb);
            if (stats) st_async_f32(rd + 128, r1, rb);
          }
        }
      }
      if (CN == 1) asm volatile("bar.sync %0, 64;" ::"r"(qbar) : "memory");
      else mbar_wait(&redbar[b], ph);
      ++step;
      if (stats) {
        float msum = 0.0f;
        for (int c = 0; c < CN; ++c) msum += red[(((b * kRRMaxCN + c) * 4 + q) * 2) * 32 + lane];
        const float mean = msum / (float)CN;
        float m2 = 0.0f, dd = 0.0f;
        for (int c = 0; c < CN; ++c) {
          const float* rc = red + (((b * kRRMaxCN + c) * 4 + q) * 2) * 32;
          const float dm = rc[lane] - mean;
          m2 += rc[32 + lane];
          dd = __fmaf_rn(dm, dm, dd);
        }
        o0 = mean;
        o1 = m2 + (float)BN * dd;
      } else {
        float mx = 0.0f;
        for (int c = 0; c < CN; ++c) mx = fmaxf(mx, red[(((b * kRRMaxCN + c) * 4 + q) * 2) * 32 + lane]);
        o0 = mx;
        o1 = 0.0f;
      }
    };
    // fp16 staging + TMA store of a 32-row x 32-column block (64B swizzle)
    auto store16 = [&](const uint32_t (&h)[16], int n0, int row0) {
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
      uint8_t* srow = stage_buf + lane * 64;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int pc = cc ^ ((lane >> 1) & 3);
        *reinterpret_cast<uint4*>(srow + pc * 16) = make_uint4(h[4 * cc], h[4 * cc + 1], h[4 * cc + 2], h[4 * cc + 3]);
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&tmC, stage_buf, n0, row0);
        bulk_commit();
      }
    };

    const int acc = G;
    uint32_t acc_phase = 0;
    uint32_t rphase = 0;  // resbar[ew] phase
    const bool tr0 = ew == 0 && lane == 0;
    int lt = G;
    for (int mt = unit + G * nunits; mt < p.m_tiles; mt += 2 * nunits, lt += 2) {
      const int row0 = (p.rev ? p.m_tiles - 1 - mt : mt) * BM + q * 32;
      const int row = row0 + lane;
      const bool row_ok = row < p.M;
      const float sx = (I8 && row_ok) ? p.row_scale[(size_t)row * p.rs_stride] : 0.0f;
      const float2 sx2 = make_float2(sx, sx);
      if (MODE == RR_LN) {
        // residual of this group's NEXT tile -> L2 (its TMA loads then hit
        // L2, not HBM): this thread's 256 bytes of its row
        const int nrow = p.rev ? row - 2 * nunits * BM : row + 2 * nunits * BM;
        if (nrow >= 0 && nrow < p.M) {
          prefetch_l2(p.residual + (size_t)nrow * p.ldr + ncol0 + c_lo);
          prefetch_l2(p.residual + (size_t)nrow * p.ldr + ncol0 + c_lo + 64);
        }
        if (lt < 2 && row_ok) {
          prefetch_l2(p.residual + (size_t)row * p.ldr + ncol0 + c_lo);
          prefetch_l2(p.residual + (size_t)row * p.ldr + ncol0 + c_lo + 64);
        }
        // residual block of chunk 0 -> the warp's staging buffer, in flight
        // while the accumulator is still being computed
        if (lane == 0) {
          bulk_wait_read<0>();  // the staging buffer's previous store has been read
          mbar_expect_tx(&resbar[ew], 32 * 64);
          tma_load_2d(stage_buf, &tmR, &resbar[ew], ncol0 + c_lo, row0, kEvictFirst);
        }
      }
      mbar_wait_sleep(&tfull[acc], acc_phase, kRRSleepNs);
      if (tr0) gemm_trace(p.trace, lt, 3);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c_lo;
      __half2 amax2 = __float2half2_rn(0.0f);

      // The packed fp16 results of chunk ch are parked in the group's own
      // accumulator columns [16 ch, 16 ch + 16) of the warp's range, which
      // chunk 0 has already been read from.
      uint32_t hp[PARK ? 4 : 1][16];  // PARK: the LN output row (fp16 pairs)
      if (MODE == RR_LN) {
        // pass 1: x = R16(dequant + bias) + residual (written back over the
        // accumulator); shifted sums (shift = the thread's first x) for the
        // local mean / M2.  The residual block (32 rows x 32 columns fp16)
        // arrives by TMA in the warp's staging buffer (64B swizzle).
        float2 sd = make_float2(0.0f, 0.0f), sq = make_float2(0.0f, 0.0f);
        float2 shift = make_float2(0.0f, 0.0f);
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t r[32];
          tmem_ld32(tbase + ch * 32, r);
          mbar_wait(&resbar[ew], (uint32_t)(rphase & 1));
          ++rphase;
          uint4 rv[4];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            rv[cc] = *reinterpret_cast<const uint4*>(stage_buf + lane * 64 + ((cc ^ ((lane >> 1) & 3)) << 4));
          __syncwarp();  // every lane has read the block before it is reused
          if (ch < 3 && lane == 0) {  // the next chunk's residual block, overlapping this chunk's math
            mbar_expect_tx(&resbar[ew], 32 * 64);
            tma_load_2d(stage_buf, &tmR, &resbar[ew], ncol0 + c_lo + 32 * (ch + 1), row0, kEvictFirst);
          }
          tmem_wait_ld();
          const __half2* rh = reinterpret_cast<const __half2*>(rv);
          const float* pb = pbias + ch * 32;
          const float* ps = psw + ch * 32;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 bb = *reinterpret_cast<const float2*>(pb + 2 * e);
            float2 y;
            if (I8) {
              const float2 a = make_float2(__int2float_rn(static_cast<int>(r[2 * e])),
                                           __int2float_rn(static_cast<int>(r[2 * e + 1])));
              y = fma2(a, mul2(sx2, *reinterpret_cast<const float2*>(ps + 2 * e)), bb);
            } else {
              y = add2(make_float2(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1])), bb);
            }
            // x = R16(y) + residual: the fp16-rounded y added as fp16 (FHADD)
            const float2 x = add_h2f(pack_half2(y.x, y.y), __half22float2(rh[e]));
            if (ch == 0 && e == 0) shift = make_float2(x.x, x.x);
            const float2 d = sub2(x, shift);
            sd = add2(sd, d);
            sq = fma2(d, d, sq);
            r[2 * e] = __float_as_uint(x.x);
            r[2 * e + 1] = __float_as_uint(x.y);
          }
          tmem_st32(tbase + ch * 32, r);  // x replaces the accumulator columns
        }
        tmem_wait_st();
        const float sdt = sd.x + sd.y;
        const float mean_t = shift.x + sdt * (1.0f / 128.0f);
        const float m2_t = fmaxf((sq.x + sq.y) - sdt * sdt * (1.0f / 128.0f), 0.0f);
        float mean, m2;
        if (tr0) gemm_trace(p.trace, lt, 8);
        exchange(mean_t, m2_t, true, mean, m2);
        if (tr0) gemm_trace(p.trace, lt, 9);
        const float var = __fdiv_rn(m2, (float)p.N);
        const float rstd = 1.0f / sqrtf(var + p.eps);
        const float2 mean2 = make_float2(mean, mean), rstd2 = make_float2(rstd, rstd);
        // pass 2: y16 = R16((x - mean) * rstd * gamma + beta) -> fp16 store, amax, park
        if constexpr (PARK) {
#pragma unroll
          for (int hh = 0; hh < 8; ++hh) {  // 16-column pieces (register budget)
            uint32_t r[16];
            tmem_ld16(tbase + hh * 16, r);
            tmem_wait_ld();
            const float* pg = pgam + hh * 16;
            const float* pt = pbet + hh * 16;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float2 d = sub2(make_float2(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1])), mean2);
              const float2 y = fma2(mul2(d, rstd2), *reinterpret_cast<const float2*>(pg + 2 * e),
                                    *reinterpret_cast<const float2*>(pt + 2 * e));
              const __half2 hh2 = __floats2half2_rn(y.x, y.y);
              amax2 = __hmax2(amax2, __habs2(hh2));
              hp[hh >> 1][(hh & 1) * 8 + e] = *reinterpret_cast<const uint32_t*>(&hh2);
            }
            if ((hh & 1) && p.store16) store16(hp[hh >> 1], ncol0 + c_lo + (hh >> 1) * 32, row0);
          }
          // every TMEM read of this tile is complete: release the accumulator
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        } else {
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t r[32];
          tmem_ld32(tbase + ch * 32, r);
          tmem_wait_ld();
          uint32_t h[16];
          const float* pg = pgam + ch * 32;
          const float* pt = pbet + ch * 32;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 d = sub2(make_float2(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1])), mean2);
            const float2 y = fma2(mul2(d, rstd2), *reinterpret_cast<const float2*>(pg + 2 * e),
                                  *reinterpret_cast<const float2*>(pt + 2 * e));
            const __half2 hh = __floats2half2_rn(y.x, y.y);
            amax2 = __hmax2(amax2, __habs2(hh));
            h[e] = *reinterpret_cast<const uint32_t*>(&hh);
          }
          if (p.outq) tmem_st16(tbase + ch * 16, h);
          if (p.store16) store16(h, ncol0 + c_lo + ch * 32, row0);
        }
        }
      } else {  // RR_QUANT: y16 = R16(act(dequant + bias)); amax; park
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t r[2][16];
          tmem_ld16(tbase + ch * 32, r[0]);
          tmem_ld16(tbase + ch * 32 + 16, r[1]);
          tmem_wait_ld();
          uint32_t h[16];
          switch (p.act) {
            case ACT_GELU: epi32<I8, ACT_GELU>(r, pbias + ch * 32, psw + ch * 32, sx, h); break;
            case ACT_RELU: epi32<I8, ACT_RELU>(r, pbias + ch * 32, psw + ch * 32, sx, h); break;
            case ACT_GELU_TANH: epi32<I8, ACT_GELU_TANH>(r, pbias + ch * 32, psw + ch * 32, sx, h); break;
            default: epi32<I8, ACT_NONE>(r, pbias + ch * 32, psw + ch * 32, sx, h); break;
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) amax2 = __hmax2(amax2, __habs2(*reinterpret_cast<const __half2*>(&h[e])));
          if (p.outq) tmem_st16(tbase + ch * 16, h);
          if (p.store16) store16(h, ncol0 + c_lo + ch * 32, row0);
        }
      }
      (void)sx2;

      if (tr0) gemm_trace(p.trace, lt, 10);
      if (p.outq) {
        if constexpr (!PARK) tmem_wait_st();
        // the parked values of chunk 0 are read while the row amax is exchanged
        // (they do not depend on it); chunk ch + 1 is read during chunk ch
        uint32_t hv[2][16];
        if constexpr (!PARK) tmem_ld16(tbase, hv[0]);
        // Q8row over the whole row (R6-R8, R12) from the fp16-rounded values
        float rmax, unused;
        exchange(fmaxf(__low2float(amax2), __high2float(amax2)), 0.0f, false, rmax, unused);
        if (tr0) gemm_trace(p.trace, lt, 11);
        const float sc = q8_scale(rmax);
        const float rs = __frcp_rn(sc);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          if constexpr (PARK) {
#pragma unroll
            for (int e = 0; e < 16; ++e) hv[ch & 1][e] = hp[ch][e];
          } else {
            tmem_wait_ld();
            if (ch < 3) tmem_ld16(tbase + (ch + 1) * 16, hv[(ch + 1) & 1]);
            if (ch == 3) {  // the group's accumulator buffer has been read for the last time
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty[acc]);
            }
          }
          uint32_t o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            o[e] = q8_quant4(__half22float2(*reinterpret_cast<const __half2*>(&hv[ch & 1][2 * e])),
                             __half22float2(*reinterpret_cast<const __half2*>(&hv[ch & 1][2 * e + 1])), sc, rs);
          // s8 block 32 rows x 32 B (1 KB, 32B swizzle) + TMA store, double
          // buffered in the two halves of the warp's staging buffer: chunk ch
          // only waits for the store that last read its half (ch 0: for every
          // earlier store, which may have used the whole buffer)
          uint8_t* qbuf = stage_buf + (ch & 1) * 1024;
          if (lane == 0) {
            if (ch == 0) bulk_wait_read<0>();
            else bulk_wait_read<1>();
          }
          __syncwarp();
#pragma unroll
          for (int cc = 0; cc < 2; ++cc)
            *reinterpret_cast<uint4*>(qbuf + lane * 32 + ((cc ^ ((lane >> 2) & 1)) << 4)) =
                make_uint4(o[4 * cc], o[4 * cc + 1], o[4 * cc + 2], o[4 * cc + 3]);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmQ, qbuf, ncol0 + c_lo + ch * 32, row0);
            bulk_commit();
          }
          if (tr0 && ch < 2) gemm_trace(p.trace, lt, 12 + ch);
        }
        if (rank == 0 && hc == 0 && row_ok) p.out_scale[row] = sc;
      } else if (!PARK || MODE != RR_LN) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
      if (tr0) gemm_trace(p.trace, lt, 5);
      acc_phase ^= 1;
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while a peer may still copy into it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * BN);
  }
}

// ------------------------------------------------------------------- host
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(ptr);
  }
  return fn;
}

static bool encode_2d(CUtensorMap* map, const void* base, int rows, int cols, CUtensorMapDataType dt, int elem_bytes,
                      size_t pitch_bytes, int box_cols, int box_rows, CUtensorMapSwizzle sw, const char** err) {
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  if ((pitch_bytes & 15) || (reinterpret_cast<uintptr_t>(base) & 15)) {
    *err = "TMA tensor needs a 16-byte aligned base and row pitch";
    return false;
  }
  (void)elem_bytes;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed";
    return false;
  }
  return true;
}

bool make_operand_map(CUtensorMap* map, const void* base, int rows, int cols, int elem_bytes, size_t pitch_bytes,
                      int box_rows, const char** err) {
  return encode_2d(map, base, rows, cols,
                   elem_bytes == 4   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                   : elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                     : CU_TENSOR_MAP_DATA_TYPE_UINT8,
                   elem_bytes,
                   pitch_bytes, 128 / elem_bytes, box_rows, CU_TENSOR_MAP_SWIZZLE_128B, err);
}

static int pick_bn(int N) {
  // (measured: 128-column tiles for the N = 768 / 1536 GEMMs of C3 are 6-15% slower)
  // Fewer wasted columns wins; ties prefer the wider tile (less A re-reading).
  const int w256 = ((N + 255) / 256) * 256 - N;
  const int w128 = ((N + 127) / 128) * 128 - N;
  return (w256 <= w128) ? 256 : 128;
}

bool plan_gemm(GemmPlan* g, bool i8, const void* A, int M_rows, int lda, const void* W, int ldw, int N, int K,
               const char** err) {
  const int eb = i8 ? 1 : 2;
  g->i8 = i8 ? 1 : 0;
  g->bn = pick_bn(N);
  g->M_rows = M_rows;
  g->has_out_map = false;
  g->force_pair = -1;
  if (!make_operand_map(&g->tmA, A, M_rows, K, eb, (size_t)lda * eb, BM, err)) return false;
  // W boxes cover BN rows (single CTA) or BN/2 rows (each CTA of a pair), BN
  // 256 or 128 chosen per M (plan_gemm_set_m): 256-, 128- and 64-row maps.
  if (!make_operand_map(&g->tmB, W, N, K, eb, (size_t)ldw * eb, 256, err)) return false;
  if (!make_operand_map(&g->tmB2, W, N, K, eb, (size_t)ldw * eb, 128, err)) return false;
  if (!make_operand_map(&g->tmB3, W, N, K, eb, (size_t)ldw * eb, 64, err)) return false;
  g->p.N = N;
  g->p.K = K;
  g->p.n_tiles = (N + g->bn - 1) / g->bn;
  g->p.k_blocks = (K * eb + BK_BYTES - 1) / BK_BYTES;
  g->p.out = nullptr;
  g->p.ldo = 0;
  g->p.out_mode = 1;
  g->p.bias = g->p.row_scale = g->p.col_scale = nullptr;
  g->p.act = ACT_NONE;
  g->p.trace = nullptr;
  g->p.tensor_qp = nullptr;
  g->p.colsum = nullptr;
  g->p.hm_rows = 0;
  g->p.rev = 0;
  g->p.rs_stride = 1;
  plan_gemm_set_m(g, M_rows);
  return true;
}

bool plan_gemm_output_hm(GemmPlan* g, void* out, int hm_rows, const char** err) {
  if (hm_rows % 256 != 0 || hm_rows < g->M_rows || g->p.N % 64 != 0) {
    *err = "head-major output needs N % 64 == 0 and hm_rows a multiple of 256 >= M_rows";
    return false;
  }
  g->p.out = out;
  g->p.ldo = 64;
  g->p.hm_rows = hm_rows;
  g->has_out_map = true;
  return encode_2d(&g->tmC, out, (g->p.N / 64) * hm_rows, 64, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, 128, kEpiCols, 32,
                   CU_TENSOR_MAP_SWIZZLE_64B, err);
}

bool plan_gemm_output(GemmPlan* g, void* out, int ldo, const char** err) {
  g->p.out = out;
  g->p.ldo = ldo;
  g->p.hm_rows = 0;
  g->p.rev = 0;
  g->p.rs_stride = 1;
  g->has_out_map = true;
  return encode_2d(&g->tmC, out, g->M_rows, g->p.N, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (size_t)ldo * 2, kEpiCols,
                   32, CU_TENSOR_MAP_SWIZZLE_64B, err);
}

// Pair decision for a tile width: CTA pairs (256-row tiles) when there are
// enough of them to fill the GPU.
static bool use_pairs(const GemmPlan* g, int M, int bn) {
  const int pair_tiles = ((M + 255) / 256) * ((g->p.N + bn - 1) / bn);
  return g->force_pair == 1 || (g->force_pair < 0 && pair_tiles >= kNumSMs / 2);
}

void plan_gemm_set_m(GemmPlan* g, int M) {
  g->p.M = M;
  // Tile width: the fewer wasted columns (pick_bn), unless 128-column tiles
  // give a shorter makespan for this M: rounds of the tile grid over the
  // persistent CTAs (or pairs) x tile width, 128-column tiles charged 10% extra (their
  // per-column cost measured 6-15% higher on C3).  Small batches (C2: M = 8192,
  // N = 1200: 3 rounds of 256-column pair tiles vs 5 of 128) take the
  // narrower tiles; the large shapes keep 256.
  int bn = pick_bn(g->p.N);
  if (bn == 256 && g->p.hm_rows == 0) {
    auto cost = [&](int w) {
      const bool pr = use_pairs(g, M, w);
      const long tiles = (long)((M + (pr ? 255 : 127)) / (pr ? 256 : 128)) * ((g->p.N + w - 1) / w);
      const long units = pr ? kNumSMs / 2 : kNumSMs;
      return (double)((tiles + units - 1) / units) * w * (w == 128 ? 1.1 : 1.0);  // per-SM work per round: 128 x w
    };
    if (cost(128) < cost(256)) bn = 128;
  }
  g->bn = bn;
  g->p.n_tiles = (g->p.N + bn - 1) / bn;
  g->pair = use_pairs(g, M, bn);
  const int tm = g->pair ? 256 : BM;
  g->p.m_tiles = (M + tm - 1) / tm;
  const int tiles = g->p.m_tiles * g->p.n_tiles;
  g->p.dbg_noload = 0;
  if (g->pair) {
    const int pairs = tiles < kNumSMs / 2 ? tiles : kNumSMs / 2;
    g->grid = 2 * pairs;
  } else {
    g->grid = tiles < kNumSMs ? tiles : kNumSMs;
  }
}

template <int BN, bool I8, bool PAIR>
static cudaError_t set_attr() {
  cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN, I8, PAIR, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<BN, PAIR>::SMEM);
  if (e != cudaSuccess) return e;
  if (!I8) return e;
  return cudaFuncSetAttribute(gemm_tc_kernel<BN, I8, PAIR, I8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              GemmCfg<BN, PAIR>::SMEM);
}

cudaError_t prepare_gemm_kernels() {
  cudaError_t e;
  if ((e = set_attr<256, true, false>()) != cudaSuccess) return e;
  if ((e = set_attr<128, true, false>()) != cudaSuccess) return e;
  if ((e = set_attr<256, false, false>()) != cudaSuccess) return e;
  if ((e = set_attr<128, false, false>()) != cudaSuccess) return e;
  if ((e = set_attr<256, true, true>()) != cudaSuccess) return e;
  if ((e = set_attr<128, true, true>()) != cudaSuccess) return e;
  if ((e = set_attr<256, false, true>()) != cudaSuccess) return e;
  return set_attr<128, false, true>();
}

// W map whose box is the rows one CTA loads per k-block: BN, or BN / 2 in a pair
template <int BN, bool PAIR>
static const CUtensorMap& wmap(const GemmPlan& g) {
  constexpr int rows = PAIR ? BN / 2 : BN;
  return rows == 256 ? g.tmB : rows == 128 ? g.tmB2 : g.tmB3;
}

template <int BN, bool I8, bool PAIR>
static cudaError_t launch_t(const GemmPlan& g, cudaStream_t s) {
  if (g.grid <= 0) return cudaSuccess;
  if (I8 && g.p.tensor_qp != nullptr)
    return launch_ex(gemm_tc_kernel<BN, I8, PAIR, I8>, dim3(g.grid), dim3(kThreads), GemmCfg<BN, PAIR>::SMEM, s,
                     PAIR ? 2 : 0, g.tmA, wmap<BN, PAIR>(g), g.tmC, g.p);
  return launch_ex(gemm_tc_kernel<BN, I8, PAIR, false>, dim3(g.grid), dim3(kThreads), GemmCfg<BN, PAIR>::SMEM, s,
                   PAIR ? 2 : 0, g.tmA, wmap<BN, PAIR>(g), g.tmC, g.p);
}

cudaError_t launch_gemm(const GemmPlan& g, cudaStream_t s) {
  if (g.p.out_mode == 1 && !g.has_out_map) return cudaErrorInvalidValue;
  if (g.pair) {
    if (g.i8) return g.bn == 256 ? launch_t<256, true, true>(g, s) : launch_t<128, true, true>(g, s);
    return g.bn == 256 ? launch_t<256, false, true>(g, s) : launch_t<128, false, true>(g, s);
  }
  if (g.i8) return g.bn == 256 ? launch_t<256, true, false>(g, s) : launch_t<128, true, false>(g, s);
  return g.bn == 256 ? launch_t<256, false, false>(g, s) : launch_t<128, false, false>(g, s);
}

// ------------------------------------------------- row-reduction GEMM host
bool rr_supported(int N) { return N % kRRBN == 0 && N / kRRBN >= 1 && N / kRRBN <= 8; }

bool plan_rr(RRPlan* g, bool i8, const void* A, int M_rows, int lda, const void* W, int ldw, int N, int K,
             void* out16, int ldo, const char** err) {
  if (!rr_supported(N)) {
    *err = "row-reduction GEMM needs N = 256 * (1..8)";
    return false;
  }
  const int eb = i8 ? 1 : 2;
  g->i8 = i8 ? 1 : 0;
  g->cn = N / kRRBN;
  g->M_rows = M_rows;
  if (!make_operand_map(&g->tmA, A, M_rows, K, eb, (size_t)lda * eb, BM, err)) return false;
  if (!make_operand_map(&g->tmB, W, N, K, eb, (size_t)ldw * eb, kRRBN, err)) return false;
  if (out16 != nullptr &&
      !encode_2d(&g->tmC, out16, M_rows, N, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (size_t)ldo * 2, 32, 32,
                 CU_TENSOR_MAP_SWIZZLE_64B, err))
    return false;
  RRParams& p = g->p;
  p = RRParams{};
  p.rs_stride = 1;
  p.N = N;
  p.K = K;
  p.k_blocks = (K * eb + BK_BYTES - 1) / BK_BYTES;
  p.act = ACT_NONE;
  plan_rr_set_m(g, M_rows);
  return true;
}

bool rebind_gemm_rows(GemmPlan* g, const void* A, int lda, int M_rows, const char** err) {
  const int eb = g->i8 ? 1 : 2;
  if (!make_operand_map(&g->tmA, A, M_rows, g->p.K, eb, (size_t)lda * eb, BM, err)) return false;
  g->M_rows = M_rows;
  return true;
}

bool rebind_rr_rows(RRPlan* g, const void* A, int lda, const void* residual, int ldr, int M_rows, const char** err) {
  const int eb = g->i8 ? 1 : 2;
  if (!make_operand_map(&g->tmA, A, M_rows, g->p.K, eb, (size_t)lda * eb, BM, err)) return false;
  if (residual != nullptr &&
      !encode_2d(&g->tmR, const_cast<void*>(residual), M_rows, g->p.N, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                 (size_t)ldr * 2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B, err))
    return false;
  g->M_rows = M_rows;
  return true;
}

bool plan_rr_io(RRPlan* g, const void* residual, int ldr, void* outq, int ldq, const char** err) {
  if (residual != nullptr &&
      !encode_2d(&g->tmR, const_cast<void*>(residual), g->M_rows, g->p.N, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                 (size_t)ldr * 2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B, err))
    return false;
  if (outq != nullptr &&
      !encode_2d(&g->tmQ, outq, g->M_rows, g->p.N, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (size_t)ldq, 32, 32,
                 CU_TENSOR_MAP_SWIZZLE_32B, err))
    return false;
  return true;
}

template <bool I8, int MODE>
static int rr_max_clusters_t(int cn) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cn * (kNumSMs / cn));
  cfg.blockDim = dim3(kRRThreads);
  cfg.dynamicSmemBytes = RRCfg::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cn;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_rr_kernel<I8, MODE>, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = kNumSMs / cn;
  }
  return n;
}

// Clusters that can be co-resident (GPC packing of CN-CTA clusters), cached.
static int rr_max_clusters(bool i8, int mode, int cn) {
  static int cache[2][3][9] = {};
  int& c = cache[i8 ? 1 : 0][mode][cn];
  if (c == 0) {
    if (mode == RR_LN) c = i8 ? rr_max_clusters_t<true, RR_LN>(cn) : rr_max_clusters_t<false, RR_LN>(cn);
    else c = i8 ? rr_max_clusters_t<true, RR_QUANT>(cn) : rr_max_clusters_t<false, RR_QUANT>(cn);
  }
  return c;
}

void plan_rr_set_m(RRPlan* g, int M) {
  g->p.M = M;
  g->p.m_tiles = (M + BM - 1) / BM;
  const int max_clusters =
      (g->p.mode == RR_LN || g->p.mode == RR_QUANT) ? rr_max_clusters(g->i8, g->p.mode, g->cn) : kNumSMs / g->cn;
  const int nc = g->p.m_tiles < max_clusters ? g->p.m_tiles : max_clusters;
  g->grid = nc * g->cn;
}

template <bool I8, int MODE, bool PARK = false>
static cudaError_t launch_rr_t(const RRPlan& g, cudaStream_t s) {
  // LN-mode row-reduction GEMMs launch without PDL unless FF_OPT_PDL_RR (measured)
  const bool pdl = tl_launch.pdl && (MODE != RR_LN || tl_launch.pdl_rr);
  return launch_ex_pdl(pdl, gemm_rr_kernel<I8, MODE, PARK>, dim3(g.grid), dim3(kRRThreads), RRCfg::SMEM, s, g.cn,
                       g.tmA, g.tmB, g.tmC, g.tmR, g.tmQ, g.p);
}

template <bool I8, int MODE, bool PARK = false>
static cudaError_t set_rr_attr() {
  return cudaFuncSetAttribute(gemm_rr_kernel<I8, MODE, PARK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              RRCfg::SMEM);
}

cudaError_t prepare_rr_kernels() {
  cudaError_t e;
  if ((e = set_rr_attr<true, RR_LN>()) != cudaSuccess) return e;
  if ((e = set_rr_attr<false, RR_LN>()) != cudaSuccess) return e;
  if ((e = set_rr_attr<true, RR_LN, true>()) != cudaSuccess) return e;
  if ((e = set_rr_attr<false, RR_LN, true>()) != cudaSuccess) return e;
  if ((e = set_rr_attr<true, RR_QUANT>()) != cudaSuccess) return e;
  return set_rr_attr<false, RR_QUANT>();
}

cudaError_t launch_rr(const RRPlan& g, cudaStream_t s) {
  if (g.grid <= 0) return cudaSuccess;
  // LN launches with long K rows (>= kRRParkKBlocks k-blocks: FFN2) take the
  // register-parked variant -- their MMA would otherwise wait for the whole
  // epilogue of the tile holding its accumulator; the short-K out-projection
  // is bound by epilogue throughput and keeps TMEM parking (same-box A/B:
  // FFN2 parked +0.9% on the C3 step, out-proj parked -1.2%)
  if (g.p.mode == RR_LN) {
    if (g.p.k_blocks >= kRRParkKBlocks)
      return g.i8 ? launch_rr_t<true, RR_LN, true>(g, s) : launch_rr_t<false, RR_LN, true>(g, s);
    return g.i8 ? launch_rr_t<true, RR_LN>(g, s) : launch_rr_t<false, RR_LN>(g, s);
  }
  return g.i8 ? launch_rr_t<true, RR_QUANT>(g, s) : launch_rr_t<false, RR_QUANT>(g, s);
}

}  // namespace ff
