// ff_kernels.h -- internal launcher interface between the host plan (ff_api.cu)
// and the sm_100a kernels.  Not part of the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ff {

constexpr int kNumSMs = 148;

// Launch policy of the forward being enqueued: the model's FF_OPT_PDL /
// FF_OPT_PDL_RR settings, installed for the duration of one run_forward on the
// calling thread (LaunchScope).  Thread-local, so models driven from several
// host threads never see each other's settings; outside a forward (weight
// packing) launches carry no PDL attribute.
struct LaunchPolicy {
  bool pdl = false;     // programmatic dependent launch between forward kernels
  bool pdl_rr = false;  // ... also on the LN-mode row-reduction GEMMs (measured slower)
};
extern thread_local LaunchPolicy tl_launch;
struct LaunchScope {
  LaunchPolicy saved;
  explicit LaunchScope(const LaunchPolicy& p) : saved(tl_launch) { tl_launch = p; }
  ~LaunchScope() { tl_launch = saved; }
};
// Launch with the programmatic-dependent-launch attribute (when the policy
// enables it) and an optional 1-D cluster (cluster = 0: no cluster
// attribute).  All forward-pass kernels go through this.
template <typename... KArgs, typename... Args>
cudaError_t launch_ex_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          int cluster, Args... args);
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster,
                      Args... args) {
  return launch_ex_pdl(tl_launch.pdl, kern, grid, block, smem, s, cluster, args...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_ex_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster >= 1) {  // 0 = plain launch; >= 1 = cluster launch (kernels using cluster PTX need it even for 1)
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

enum Act { ACT_NONE = -1, ACT_GELU = 0, ACT_RELU = 1, ACT_GELU_TANH = 2 };

// ---------------------------------------------------------------- GEMM
// C[M,N] = A[M,K] * W[N,K]^T on tcgen05 (kind::f16 or kind::i8), TMA-fed.
struct GemmParams {
  int M, N, K;
  int m_tiles, n_tiles, k_blocks;
  void* out;               // fp16 [M, ldo] (out_mode 1) or 32-bit raw [M, ldo] (out_mode 0)
  int ldo;                 // elements
  int out_mode;            // 0 raw accumulators, 1 production epilogue
  const float* bias;       // [N] or null
  const float* row_scale;  // sx [M] (i8)
  const float* col_scale;  // sw [N] (i8)
  int act;                 // Act
  unsigned long long* trace;  // debug timeline (ff_debug_set_trace), null in production
  // per-tensor u8 activations (DESIGN R22; null = per-row s8): A is u8, the
  // epilogue uses tensor_qp[0] (scale), tensor_qp[1] (zero point) and
  // colsum[n] = sum_k wq[n][k]
  const float* tensor_qp;
  const int* colsum;
  int dbg_noload;  // debug MMA-rate probe: skip the operand loads (ff_debug_gemm bit 6; 0 in production)
  // head-major output (the fused QKV projection, hs = 64): output column n goes
  // to row (n / 64) * hm_rows + m, column n % 64 of a [heads * hm_rows, 64]
  // buffer, so every (section, head) slice is one contiguous block; 0 = row-major
  int hm_rows;
  // 1: walk the row tiles from the last to the first (the launch order
  // alternates so a kernel first reads the rows its producer wrote last,
  // i.e. the ones most likely still in L2)
  int rev;
  int rs_stride;  // row_scale[m * rs_stride] (1; S when A holds every S-th token row)
};

struct GemmPlan {
  CUtensorMap tmA, tmB, tmB2, tmB3, tmC;  // A, W (256 / 128 / 64-row boxes, 128B swizzle); fp16 output
  GemmParams p;
  int bn;       // N tile (128 or 256)
  int i8;       // 1 = kind::i8
  int grid;
  int M_rows;   // row capacity of A / the output buffer
  bool has_out_map;
  int force_pair;   // -1 auto (pairs when >= 74 pair-tiles), 0 never, 1 always
  bool pair;        // chosen for the current M
};

// Encode a 2-D K-major tensor map for a GEMM operand: rows x cols elements of
// `elem_bytes` (4 fp32 / 2 fp16 / 1 int8), row pitch in bytes, box = box_rows x 128 B,
// 128-byte swizzle, zero fill out of bounds.
bool make_operand_map(CUtensorMap* map, const void* base, int rows, int cols, int elem_bytes, size_t pitch_bytes,
                      int box_rows, const char** err);
// Fill a GemmPlan (tile choice, maps, grid) for A [M_rows x K] (pitch lda
// elements) and W [N x K] (pitch ldw); M_rows >= M is the buffer capacity.
bool plan_gemm(GemmPlan* g, bool i8, const void* A, int M_rows, int lda, const void* W, int ldw, int N, int K,
               const char** err);
// Bind the fp16 output buffer [M_rows x N] (pitch ldo elements) of a plan.
bool plan_gemm_output(GemmPlan* g, void* out, int ldo, const char** err);
// Bind a head-major fp16 output (see GemmParams::hm_rows): N / 64 blocks of
// hm_rows x 64 (hm_rows >= M_rows, a multiple of 256 so no tile straddles two heads).
bool plan_gemm_output_hm(GemmPlan* g, void* out, int hm_rows, const char** err);
// Update the per-call fields (M) of a plan.
void plan_gemm_set_m(GemmPlan* g, int M);
cudaError_t launch_gemm(const GemmPlan& g, cudaStream_t s);

// -------------------------------------------- row-reduction GEMM epilogues
// GEMM whose epilogue needs whole output rows: a cluster of CN = N/256 CTAs
// spans the row (one 128x256 tile each) and exchanges per-row partials through
// DSMEM (st.async + mbarrier).
//   RR_LN:    y = LN(R16(acc-epilogue) + residual) -> fp16 [+ s8 rows + scale]
//             (post-LN residual + LayerNorm fused into out-proj / FFN2)
//   RR_QUANT: y = R16(act(acc-epilogue)) -> s8 rows + scale [+ fp16 copy]
//             (FFN-intermediate requant fused into FFN1)
enum RRMode { RR_LN = 1, RR_QUANT = 2 };
struct RRParams {
  int M, N, K, m_tiles, k_blocks;
  int mode;
  const float* bias;       // [N]
  const float* row_scale;  // sx [M] (int8 A)
  const float* col_scale;  // sw [N] (int8 W)
  int act;                 // RR_QUANT
  const __half* residual;  // RR_LN: [M, ldr]
  int ldr;
  const float* gamma;      // RR_LN
  const float* beta;
  float eps;
  int store16;             // write the fp16 result through tmC
  int8_t* outq;            // s8 rows [M, ldq] or null
  int ldq;
  float* out_scale;        // [M] or null
  unsigned long long* trace;  // debug timeline (ff_debug_set_trace), null in production
  int rev;                    // 1: row tiles walked last to first (see GemmParams::rev)
  int rs_stride;              // row_scale[m * rs_stride]
};
struct RRPlan {
  CUtensorMap tmA, tmB, tmC;
  CUtensorMap tmR;  // residual fp16 [M_rows x N], 32 x 32 boxes (RR_LN)
  CUtensorMap tmQ;  // s8 output [M_rows x N], 32 x 32 boxes (when outq is used)
  RRParams p;
  int i8, cn, grid, M_rows;
};
bool rr_supported(int N);
bool plan_rr(RRPlan* g, bool i8, const void* A, int M_rows, int lda, const void* W, int ldw, int N, int K,
             void* out16, int ldo, const char** err);
void plan_rr_set_m(RRPlan* g, int M);
// Bind the residual (RR_LN) and s8 output buffers (either may be null) of a plan.
bool plan_rr_io(RRPlan* g, const void* residual, int ldr, void* outq, int ldq, const char** err);
// Re-encode the row-indexed input maps of a plan for M_rows rows at pitch lda
// (elements) -- e.g. the first token of each sequence (lda = S x the row
// pitch); the residual map of an RR_LN plan too when residual != null.
bool rebind_gemm_rows(GemmPlan* g, const void* A, int lda, int M_rows, const char** err);
bool rebind_rr_rows(RRPlan* g, const void* A, int lda, const void* residual, int ldr, int M_rows, const char** err);
cudaError_t launch_rr(const RRPlan& g, cudaStream_t s);
cudaError_t prepare_rr_kernels();

// ------------------------------------------------------------ row kernels
// X = LN(E_tok[id] + Ppos'[t]) -> x16 [M, ldx] (+ optional s8 xq [M, ldq], xs [M]).
// Validates ids / mask into *err_flag (sticky bits).
cudaError_t launch_embed_ln(const int32_t* ids, const int32_t* mask, int B, int S, int H, int V,
                            const float* tok, const float* pos, const float* g, const float* b, float eps,
                            __half* x16, int ldx, int8_t* xq, int ldq, float* xs, int* err_flag, cudaStream_t s);
// y = LN(a + r) -> y16 (+ optional s8 yq, ys).
cudaError_t launch_add_ln(const __half* a, int lda, const __half* r, int ldr, int M, int H, const float* g,
                          const float* b, float eps, __half* y16, int ldy, int8_t* yq, int ldq, float* ys,
                          cudaStream_t s);
// Per-tensor u8 quantization with zero point (DESIGN R22) of fp16 rows
// [M, K] (K % 8 == 0): mm = 2 uint scratch (reset here), q = u8 [M, ldq],
// qp[0] = scale, qp[1] = zero point.
cudaError_t launch_quant_tensor(const __half* x, int ldx, int M, int K, unsigned* mm, uint8_t* q, int ldq, float* qp,
                                cudaStream_t s);
// colsum[n] = sum_k wq[n][k] of packed s8 weights.
cudaError_t launch_weight_colsum(const int8_t* wq, int ldw, int N, int K, int* colsum, cudaStream_t s);
// Per-row symmetric int8 quantization of fp16 rows.
cudaError_t launch_quant_rows(const __half* x, int ldx, int M, int K, int8_t* q, int ldq, float* scale,
                              cudaStream_t s);
// pooled = tanh(Wp x0 + bp); logits = Wc pooled + bc, x0 = row b*S of x16.
// part: fp32 scratch of at least B x S x H floats (split-K partials).
cudaError_t launch_head(const __half* x16, int ldx, int B, int S, int H, int C, const float* Wp, const float* bp,
                        const float* Wc, const float* bc, float* part, float* logits, cudaStream_t s,
                        int seq_stride = -1);

// ------------------------------------------------------------- attention
size_t attention_smem_bytes(int S, int d);
// mma.sync attention: QKV sections of A heads at head stride hs >= d (hs > d:
// zero-padded head columns), ctx rows unpadded [B*S, ldctx] (head h at h * d).
cudaError_t launch_attention(const __half* qkv, int ldqkv, const int32_t* mask, int B, int S, int A, int d, int hs,
                             int hm_rows, __half* ctx, int ldctx, cudaStream_t s);

// tcgen05 attention (head_dim 64 or <= 32 even -- padded to 32 --, S <= 128); the tensor map covers the QKV
// buffer [M_rows x ldqkv] fp16 with 64-column x 128-row boxes.  Writes the
// fp16 ctx rows when ctx != null and, when ctxq != null (requires
// attention_tc_fuses_quant(A, d)), the Q8row s8 ctx rows + per-row scales.
// hs: head stride of the QKV buffer (>= d; TMA needs 2 hs % 16 == 0).
bool attention_tc_supported(int S, int d, int hs, int ldqkv, int ldctx);
bool attention_tc_fuses_quant(int A, int d);
struct AttnTCPlan {
  CUtensorMap map;
  const void* qkv;  // QKV rows (contiguous: ldqkv fp16 per row)
  int ldqkv;
  // 0: row-major [tokens, ldqkv] QKV; > 0: head-major [3 A heads x hm_rows, 64]
  // (the map then has 64 columns and the head slice (t, h) of token r is row
  // (t A + h) hm_rows + r)
  int hm_rows;
};
bool plan_attention_tc(AttnTCPlan* plan, const void* qkv, int M_rows, int ldqkv, const char** err);
// Head-major QKV buffer of n_blocks = 3 * Amax blocks of hm_rows x 64 fp16.
bool plan_attention_tc_hm(AttnTCPlan* plan, const void* qkv, int n_blocks, int hm_rows, const char** err);
cudaError_t launch_attention_tc(const AttnTCPlan& plan, const int32_t* mask, int B, int S, int A, int d, int hs,
                                __half* ctx,
                                int ldctx, int8_t* ctxq, int ldq, float* ctxs, cudaStream_t s,
                                unsigned long long* trace = nullptr, int rev = 1);
cudaError_t prepare_attention_tc_kernel();

// tcgen05 attention for 128 < S <= 512, head_dim 64 (attention_long.cu): fp16
// ctx rows [B*S, ldctx]; the same QKV tensor map as attention_tc.
bool attention_long_supported(int S, int d, int ldqkv, int ldctx);
cudaError_t launch_attention_long(const AttnTCPlan& plan, const int32_t* mask, int B, int S, int A, __half* ctx,
                                  int ldctx, cudaStream_t s, unsigned long long* trace = nullptr);
cudaError_t prepare_attention_long_kernel();

// ------------------------------------------------------- weight packing
cudaError_t launch_cast_f16(const float* src, int N, int K, __half* dst, int ldd, cudaStream_t s);
cudaError_t launch_quant_weight(const float* src, int N, int K, int8_t* dst, int ldd, float* scale,
                                cudaStream_t s);
cudaError_t launch_add_row(const float* src, int N, int K, const float* row, float* dst, cudaStream_t s);

// One-time cudaFuncSetAttribute calls (outside any stream capture).
cudaError_t prepare_gemm_kernels();
cudaError_t prepare_attention_kernels();
cudaError_t prepare_row_kernels();

// ---- importance scorer: 3xFP16 tcgen05 GEMM (gemm_x3.cu)
// C[M x N] (+)= A[M x K] B[N x K]^T (+ bias[N]) with A row m = sa[m] (Ah + Al)
// and B row n = sb[n] (Bh + Bl) given as row-scaled fp16 hi / lo splits (row
// pitch lda / ldb halves, multiples of 8, zero-padded beyond K); C has row
// pitch ldc.  kc = k-blocks (64 of K) per TMEM accumulation chunk (chunks are
// summed with IEEE fp32 adds).  ws (optional, ws_floats floats): split-K
// partial sums for shapes with too few tiles to fill the SMs (up to 4 x M x N).
// *err set on a setup failure.
cudaError_t launch_gemm_x3(const __half* Ah, const __half* Al, const float* sa, int lda, const __half* Bh,
                           const __half* Bl, const float* sb, int ldb, int M, int N, int K, const float* bias, float* C,
                           int ldc, bool accumulate, cudaStream_t s, const char** err, int kc = 2,
                           float* ws = nullptr, size_t ws_floats = 0);
// Row-scaled hi / lo fp16 split of X [M x K] (pitch ldx) into [M x ldo]
// buffers (ldo % 8 == 0, >= K; zero-padded) and the row scales scale[M] (2^e).
cudaError_t launch_split_x3(const float* X, int M, int K, int ldx, __half* hi, __half* lo, int ldo, float* scale,
                            cudaStream_t s);
// WT [K x N] = W^T for W [N x K] (fp32, dense).
cudaError_t launch_transpose_f32(const float* W, int N, int K, float* WT, cudaStream_t s);

}  // namespace ff
