/* include/fastformers.h -- C ABI of the B200-native FastFormers encoder forward.
 *
 * FastFormers (arXiv 2010.13382) = knowledge distillation + structured pruning
 * + 8-bit / 16-bit numerics + runtime fusion for Transformer NLU inference.
 * This library is the data-parallel hot path of that recipe: the batched
 * forward pass of a distilled, structurally pruned post-LN BERT/RoBERTa
 * encoder classifier (PAPER.md "P:n" lines cited below; DESIGN.md "R<k>" =
 * reading k of the paper).  Each layer l keeps its own number of attention
 * heads A'_l and FFN width F'_l ("re-group and reconnect the remaining
 * heads and hidden states"), and runs its four constant-weight GEMMs either in
 * fp16 ("all the model parameters are converted into 16-bit floating
 * point") or as dynamically quantized int8 ("8-bit quantized matrix
 * multiplication ... dynamic quantization", per-row activation / per-output
 * channel weight scales, R6-R8).  Q.K^T and P.V always stay in floating point
 * ("we do not use 8-bit matrix product for the Q, K inner product").
 *
 * No C++ or torch types cross this boundary: plain pointers and sizes only.
 * Device pointers are marked d_, host pointers h_.  All device work is
 * enqueued on the caller's CUDA stream (cudaStream_t passed as void*; NULL =
 * legacy default stream).  Every call returns ff_status and sets a
 * thread-local message readable with ff_last_error(); no exception crosses
 * the ABI.  Compute runs only in the sm_100a kernels of this library; there
 * is no CPU fallback (a missing GPU / wrong arch is FF_E_CUDA).
 *
 * Call order (anything else returns FF_E_STATE):
 *   ff_model_create -> ff_model_memory -> (caller allocates two device
 *   buffers) -> ff_bind_memory -> ff_load_weights x N -> ff_finalize ->
 *   ff_encode* / ff_encode_host* (+ ff_check) -> ff_model_destroy.
 *
 * Ownership: the CALLER owns every device buffer (weight arena, workspace,
 * ids, mask, logits).  The library owns host metadata, TMA tensor maps and
 * CUDA-graph executables only; ff_model_destroy frees those.  Weights are
 * immutable after ff_finalize.  Concurrent ff_encode calls on one model race
 * on its workspace: use one model (one binding) per concurrent stream.
 */
#ifndef FASTFORMERS_H_
#define FASTFORMERS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FF_ABI_VERSION 1

#if defined(__GNUC__)
#define FF_API __attribute__((visibility("default")))
#else
#define FF_API
#endif

typedef struct ff_model ff_model; /* opaque */

typedef enum {
  FF_OK = 0,
  FF_E_INVALID = 1,     /* bad argument / config value                         */
  FF_E_SHAPE = 2,       /* unknown tensor name, wrong shape, size over capacity */
  FF_E_STATE = 3,       /* call out of order                                    */
  FF_E_CUDA = 4,        /* CUDA runtime / driver error (message has details)    */
  FF_E_INPUT = 5,       /* data-dependent input error seen on the device        */
  FF_E_UNSUPPORTED = 6, /* valid but unsupported geometry                       */
  FF_E_NOMEM = 7        /* caller-provided buffer too small                     */
} ff_status;

typedef enum { FF_F16 = 0, FF_I8 = 1 } ff_dtype;

/* Activation of the FFN ("We replace GELU with ReLU"; R2): GELU with
 * erf (HF "gelu", default), ReLU, or the tanh approximation. */
typedef enum { FF_ACT_GELU = 0, FF_ACT_RELU = 1, FF_ACT_GELU_TANH = 2 } ff_act;

typedef struct {
  int32_t abi_version;   /* must be FF_ABI_VERSION                                      */
  int32_t num_layers;    /* L >= 1                                                       */
  int32_t hidden;        /* H, multiple of 8, <= 1024                                    */
  int32_t head_dim;      /* d, even, 2..128 (same in every layer)                       */
  int32_t vocab_size;    /* V                                                            */
  int32_t max_positions; /* P: max sequence length S (position table rows)              */
  int32_t num_classes;   /* C >= 1                                                       */
  float ln_eps;          /* LayerNorm epsilon: 1e-12 BERT, 1e-5 RoBERTa (R3)            */
  int32_t act;           /* ff_act                                                       */
  const int32_t *heads;  /* [num_layers] surviving heads A'_l >= 1 (copied at create)   */
  const int32_t *ffn_dim;/* [num_layers] surviving FFN width F'_l >= 1 (copied)         */
  const int32_t *dtype;  /* [num_layers] ff_dtype of the layer's GEMMs (copied)         */
  int32_t max_tokens;    /* capacity: largest B*S passed to ff_encode (workspace size)  */
} ff_config;

FF_API int32_t ff_abi_version(void);
FF_API const char *ff_last_error(void);

/* Validate cfg and build the host-side plan for CUDA device `cuda_device`
 * (must be sm_100).  *out receives the model.  Errors: FF_E_INVALID,
 * FF_E_UNSUPPORTED (geometry the kernels do not cover), FF_E_CUDA. */
FF_API ff_status ff_model_create(const ff_config *cfg, int32_t cuda_device, ff_model **out);

/* Bytes the caller must allocate on the device: the packed weight arena and
 * the activation workspace (one layer's worth, reused across layers). */
FF_API ff_status ff_model_memory(const ff_model *m, size_t *weight_bytes, size_t *workspace_bytes);

/* Hand the library the two caller-owned device buffers (256-B aligned).  The
 * weight arena is zero-filled here (on `stream`).  FF_E_NOMEM if too small. */
FF_API ff_status ff_bind_memory(ff_model *m, void *d_weights, size_t weight_bytes, void *d_workspace,
                         size_t workspace_bytes, void *stream);

/* Load one fp32 host tensor by its HuggingFace state_dict name (optional
 * "bert."/"roberta." prefix; RoBERTa head aliases classifier.dense.* ->
 * pooler.dense.*, classifier.out_proj.* -> classifier.*).  Layout is PyTorch
 * [out, in] row-major.  Weight packing happens here once, on the GPU (P:104
 * "the result of the packing operation needs to be properly cached"): GEMM
 * weights of fp16 layers are cast to fp16, those of int8 layers quantized per
 * output channel (scale = amax/127, RNE, R7-R8); Q|K|V are concatenated
 * (fused QKV).  The host buffer may be reused when the call returns (it
 * synchronizes `stream`).  Errors: FF_E_SHAPE (unknown name / wrong shape),
 * FF_E_STATE (before ff_bind_memory or after ff_finalize), FF_E_CUDA. */
FF_API ff_status ff_load_weights(ff_model *m, const char *name, const float *h_data, const int64_t *shape,
                          int32_t rank, void *stream);

/* All tensors present -> fold the token-type-0 row into the position table
 * (R16), build TMA tensor maps, mark READY.  FF_E_STATE lists what is missing. */
FF_API ff_status ff_finalize(ff_model *m, void *stream);

/* The hot path: logits[B, C] (fp32) = classifier(pooler(encoder(ids, mask))).
 * d_token_ids, d_mask: [batch, seq] int32 row-major on the device; mask is
 * 1 for real tokens, 0 for padding; keys with mask 0 are excluded from the
 * softmax (R4) and mask[b, 0] must be 1 (R5).  d_logits: [batch, C] fp32.
 * Asynchronous on `stream`.  Host-checkable errors return at once: seq >
 * max_positions or batch*seq > max_tokens -> FF_E_SHAPE.  Ids outside [0, V),
 * a mask value not in {0,1} or mask[b,0] != 1 set a sticky device flag that
 * ff_check reports as FF_E_INPUT (the bad row's logits are unspecified).
 * With graphs enabled (default) the launch sequence is captured once per
 * (batch, seq, buffer addresses) and replayed. */
FF_API ff_status ff_encode(ff_model *m, const int32_t *d_token_ids, const int32_t *d_mask, int32_t batch,
                    int32_t seq, float *d_logits, void *stream);

/* End-to-end form of ff_encode on HOST buffers: copies ids/mask host->device
 * into the workspace, runs ff_encode, copies logits device->host and
 * synchronizes `stream` (pinned host memory gives full copy bandwidth). */
FF_API ff_status ff_encode_host(ff_model *m, const int32_t *h_token_ids, const int32_t *h_mask, int32_t batch,
                         int32_t seq, float *h_logits, void *stream);

/* Pipelined form of ff_encode_host: enqueued WITHOUT the final
 * synchronization, so a serving loop can enqueue batch k+1 while batch k
 * runs.  The ids / mask copies run on a library-owned copy stream into one of
 * two workspace input sets (alternating per call, each reused only after the
 * forward that last read it), so the next batch's upload overlaps the current
 * forward; the forward and the logits copy run on `stream`.  h_token_ids /
 * h_mask must stay valid and unchanged, and h_logits must not be read, until
 * `stream` has been synchronized (cudaStreamSynchronize or ff_check); pinned
 * host memory is required for the copies to be asynchronous.  Use one stream
 * per model for these calls. */
FF_API ff_status ff_encode_host_async(ff_model *m, const int32_t *h_token_ids, const int32_t *h_mask, int32_t batch,
                                      int32_t seq, float *h_logits, void *stream);

/* Synchronize `stream`; FF_E_INPUT (and clear the flag) if an input error was
 * flagged by an earlier ff_encode, else FF_OK. */
FF_API ff_status ff_check(ff_model *m, void *stream);

/* Options: FF_OPT_GRAPHS (1 = capture/replay CUDA graphs, default 1);
 * FF_OPT_CTA_PAIRS (1 = let large GEMMs use CTA pairs / 256-row tiles,
 * default 1; 0 = single-CTA 128-row tiles only -- results are identical). */
#define FF_OPT_GRAPHS 1
#define FF_OPT_CTA_PAIRS 2
/* FF_OPT_ATTN_TC (1 = tcgen05 attention for head_dim 64, S <= 128, default 1;
 * 0 = the mma.sync attention kernel everywhere). */
#define FF_OPT_ATTN_TC 3
/* FF_OPT_FUSED_EPILOGUES (1: where the output row is 256 x 1..8 columns,
 * fuse residual + LayerNorm (+ s8 requant) into the out-proj / FFN2 GEMM
 * epilogues and the FFN-intermediate requant into FFN1, using clusters that
 * span the row; 0: separate add_ln / quant_rows kernels everywhere; the
 * default is FF_OPT_FUSED_MASK = -1, auto).  With 1, ff_encode_trace does not fill the O16 / Y16 dumps (never
 * materialised). */
#define FF_OPT_FUSED_EPILOGUES 4
/* FF_OPT_PDL (1 = default: launch every forward kernel of this model with
 * programmatic dependent launch so its prologue overlaps the previous
 * kernel's tail; per model). */
#define FF_OPT_PDL 5
/* FF_OPT_ACT_QUANT: activation quantizer of the int8 layers.  0 = default:
 * Q8row, per-row symmetric s8 (north_star; DESIGN R6-R8); 1 = Q8tensor, the
 * paper's per-tensor dynamic range as u8 with a zero point, u8 x s8
 * tcgen05 GEMMs with an exact zero-point x column-sum correction (DESIGN
 * R22).  1 disables FF_OPT_FUSED_EPILOGUES and breaks batch / padding
 * invariance by construction (the range spans the whole batch). */
#define FF_OPT_ACT_QUANT 6
/* FF_OPT_FUSED_MASK: per-fusion control of FF_OPT_FUSED_EPILOGUES (which sets
 * 0 or 7): bit 0 out-proj + residual + LN1, bit 1 FFN1 + activation + requant
 * (int8 layers), bit 2 FFN2 + residual + LN2.  Value 0..7, or -1 = auto (the
 * default): FFN1 + requant always, and each LN fusion where the GEMM's K row
 * is at most 3 KB (with longer rows the row-reduction kernel's single-CTA
 * tiles lose to the CTA-pair GEMM + add_ln).  The LN fusions combine
 * the LN statistics across the cluster in another order than add_ln, so their
 * logits agree with the unfused path within the DESIGN §3 bounds, not bit for
 * bit; mask 2 is bit-identical to the unfused path. */
#define FF_OPT_FUSED_MASK 8
/* FF_OPT_PDL_RR (per model): 1 = the LN-mode row-reduction GEMMs
 * (FF_OPT_FUSED_MASK bits 0 / 2) also launch with PDL; default 0 (with PDL
 * they slowed the step by 5-10%). */
#define FF_OPT_PDL_RR 9
/* FF_OPT_CLS_LAST_LAYER (per model, default 0): the pooler reads only the first
 * token of each sequence (a11; "pooler = tanh of first-token
 * projection") and every step of a layer after the attention (out-projection,
 * residual + LN1, FFN, residual + LN2, the per-row requants) is row-local, so
 * with 1 the LAST layer runs those steps on the B first-token rows only (its
 * QKV projection and attention still see every token).  The logits are
 * bit-identical to the default path (tests/test_gpu_model.py); hidden states of
 * the last layer other than the first tokens are not computed (ff_encode_trace
 * of the last layer disables it).  Off by default: the bench's headline runs
 * every row of every layer; this is reported as a variant. */
#define FF_OPT_CLS_LAST_LAYER 13
/* FF_OPT_ROW_DIRS (per model): row-tile walking direction per launch role,
 * bits high to low QKV, attention, out-projection, FFN1, FFN2 (1 = last row
 * tile first).  Results do not depend on it (every step is row-local; tested);
 * it only decides which rows a kernel reads first -- a consumer walking
 * opposite to its producer first reads the rows written last, the most likely
 * to still be in L2.  Default 0b01010 (attention and FFN1 reversed; measured,
 * DESIGN §6).  Value 0..31, else FF_E_INVALID. */
#define FF_OPT_ROW_DIRS 14
/* Set `option` to `value` on model m (invalidates its captured graphs).  Every
 * option is per model: the library holds no process-wide mutable state on the
 * launch path, so models may be driven from different host threads (one
 * thread at a time per model).  Option ids 7, 10, 11 and 12 (round-1
 * experiments measured slower and removed) are rejected.
 * FF_E_INVALID for an unknown option / bad value / NULL m. */
FF_API ff_status ff_set_option(ff_model *m, int32_t option, int64_t value);
/* Read the current value of `option` on model m into *value (host pointer).
 * FF_E_INVALID for an unknown option / NULL m / NULL value. */
FF_API ff_status ff_get_option(const ff_model *m, int32_t option, int64_t *value);

FF_API void ff_model_destroy(ff_model *m);

/* Number of kernels one ff_encode launches for (batch, seq). */
FF_API ff_status ff_launch_count(const ff_model *m, int32_t batch, int32_t seq, int32_t *count);

/* Kernel kinds reported by ff_profile. */
typedef enum {
  FF_K_EMBED_LN = 0, FF_K_GEMM_F16 = 1, FF_K_GEMM_I8 = 2, FF_K_ATTENTION = 3, FF_K_QUANT = 4,
  FF_K_ADD_LN = 5, FF_K_HEAD = 6,
  /* row-reduction GEMMs (FF_OPT_FUSED_MASK): GEMM + fused LayerNorm / requant */
  FF_K_GEMM_RR_F16 = 7, FF_K_GEMM_RR_I8 = 8
} ff_kernel_kind;

/* Run one forward WITHOUT graphs with a CUDA-event pair around every kernel
 * launch on `stream`, synchronize, and return per launch its kind and device
 * duration in ms (capacity = size of the output arrays; *count = launches). */
FF_API ff_status ff_profile(ff_model *m, const int32_t *d_token_ids, const int32_t *d_mask, int32_t batch,
                            int32_t seq, float *d_logits, int32_t capacity, int32_t *kinds, float *ms,
                            int32_t *count, void *stream);

/* ------------------------------------------------------------------------
 * Test / lockstep exports (not part of the user contract).
 * ------------------------------------------------------------------------ */

/* Run ff_encode and additionally copy the fp16 stage tensors of layer
 * `layer` into caller device buffers (each packed row-major, NULL = skip):
 * d_dump[0] X16 input [M,H], [1] QKV16 [M,3D], [2] CTX16 [M,D], [3] O16 [M,H],
 * [4] H1_16 [M,H], [5] I16 [M,F], [6] Y16 [M,H], [7] X16 output [M,H]
 * (M = batch*seq, D = A'_l*d, F = F'_l).  Never uses graphs. */
FF_API ff_status ff_encode_trace(ff_model *m, const int32_t *d_token_ids, const int32_t *d_mask, int32_t batch,
                          int32_t seq, float *d_logits, int32_t layer, void *const *d_dump, void *stream);

/* One GEMM through the production tcgen05 kernel: C[M,N] = A[M,K] W[N,K]^T.
 * dtype FF_F16: A, W fp16 (row pitches lda, ldw in elements, 16-B aligned
 * rows); dtype FF_I8: A, W int8.  out_mode 0: raw accumulators (int32 for i8,
 * fp32 for f16) into d_C with pitch ldc; out_mode 1: production epilogue
 * (i8: fma(float(acc), sx[m]*sw[n], bias[n]); f16: acc + bias[n]; then act
 * (act < 0 = none); fp16 output).  d_bias/d_sx/d_sw may be NULL where unused.
 * out_mode | 16 forces the CTA-pair (cta_group::2, 256-row tile) kernel,
 * out_mode | 32 forces the single-CTA kernel (default: chosen by size). */
FF_API ff_status ff_debug_gemm(int32_t dtype, const void *d_A, int32_t lda, const void *d_W, int32_t ldw, int32_t M,
                        int32_t N, int32_t K, int32_t out_mode, void *d_C, int32_t ldc, const float *d_bias,
                        const float *d_sx, const float *d_sw, int32_t act, void *stream);

/* Per-row int8 quantization of an fp16 matrix (R6-R8): d_q [M, ldq] s8,
 * d_s [M] fp32 scales. */
FF_API ff_status ff_debug_quant_rows(const void *d_x16, int32_t M, int32_t K, int32_t ldx, int8_t *d_q, int32_t ldq,
                              float *d_s, void *stream);

/* Fused masked-softmax attention of one layer: qkv16 [B*S, 3*A*d] -> ctx16
 * [B*S, A*d] (packed rows).  impl: 0 = auto (the tcgen05 kernel where it
 * applies: head_dim 64, S <= 128), 1 = the mma.sync kernel (any even d <= 128),
 * 2 = tcgen05 only (FF_E_UNSUPPORTED otherwise). */
FF_API ff_status ff_debug_attention(const void *d_qkv16, const int32_t *d_mask, int32_t B, int32_t S, int32_t A,
                                    int32_t d, void *d_ctx16, int32_t impl, void *stream);
/* Debug timeline (NULL = off): uint64 [grid x 64 x 24] per-CTA per-tile
 * %globaltimer stamps (events documented in csrc/gemm_tc.cu); the buffer must
 * be zeroed by the caller.  which = 0: subsequent ff_debug_gemm launches;
 * 1 / 2 / 3: the layer-0 fused out-proj+LN / FFN1+requant / FFN2+LN GEMM of
 * subsequent forwards (FF_OPT_FUSED_EPILOGUES); 4: the S > 128 attention of
 * subsequent ff_debug_attention calls (uint64 [grid x 32 x 8], events in
 * csrc/attention_long.cu). */
FF_API ff_status ff_debug_set_trace(uint64_t *d_trace, int32_t which);

/* The tcgen05 attention with the int8 ctx requant fused (a3 + a4; the path
 * int8 layers take): ctx rows are quantized per row, Q8row (DESIGN R6-R8),
 * from their fp16-rounded values.  d_ctxq: s8 [B*S x A*d] (pitch A*d),
 * d_ctxs: fp32 [B*S] scales; d_ctx16 (optional, may be NULL) also receives
 * the fp16 ctx.  Requires head_dim 64, S <= 128, 1 <= A <= 8 (else
 * FF_E_UNSUPPORTED).  d_trace (optional, may be NULL): uint64 [grid x 32 x 8]
 * per-CTA per-head event timestamps (%globaltimer, ns) for pipeline analysis;
 * grid = min(B, 148). */
FF_API ff_status ff_debug_attention_q8(const void *d_qkv16, const int32_t *d_mask, int32_t B, int32_t S, int32_t A,
                                       int32_t d, void *d_ctx16, int8_t *d_ctxq, float *d_ctxs, uint64_t *d_trace,
                                       void *stream);

/* ------------------------------------------------------------------------
 * Structured-pruning importance scores (PAPER.md P:93:
 * "we add a mask variable to each attention head for the gradient computation
 * of the heads.  Next, we run forward and backward passes of the model on the
 * entire validation data set, then the absolute values of the gradients are
 * accumulated.")  A scorer holds the UNPRUNED model in fp32 and, per batch,
 * runs the encoder forward keeping its activations, the classifier's mean
 * cross-entropy against the labels (DESIGN R24), and the backward pass, adding
 * |dL/dxi[l][h]| (head mask on the context of head h, R23) and |dL/dnu[l][f]|
 * (FFN-unit mask after the activation) to fp64 score arrays.  Selection and
 * reconnection of the kept units ("re-group and reconnect") are host
 * steps (paper_2010_13382_b200/pruning.py) whose result is a new ff_config.
 * Errors: ff_scorer_last_error() (thread-local).  Same call order as the
 * model: create -> memory -> bind -> load_weights x N -> finalize -> score*.
 * cfg: as for ff_model_create (dtype ignored: fp32 throughout; C <= 64);
 * workspace grows with max_tokens * (layers x (12 H + 4 D + 2 F + A * max_positions));
 * the weight arena holds the fp32 weights plus four TF32 split copies of each
 * linear's weight (about 5x the linears' fp32 bytes). */
typedef struct ff_scorer ff_scorer;
FF_API const char *ff_scorer_last_error(void);
FF_API ff_status ff_scorer_create(const ff_config *cfg, int32_t cuda_device, ff_scorer **out);
/* fp32 weight arena and workspace sizes (bytes) the caller must allocate. */
FF_API ff_status ff_scorer_memory(const ff_scorer *s, size_t *weight_bytes, size_t *workspace_bytes);
/* Caller-owned device arenas, 256-byte aligned, at least the sizes above. */
FF_API ff_status ff_scorer_bind_memory(ff_scorer *s, void *d_weights, size_t weight_bytes, void *d_workspace,
                                       size_t workspace_bytes);
/* Same HF names / shapes as ff_load_weights (fp32 host data, copied before
 * return); FF_E_SHAPE for an unknown name or a wrong shape. */
FF_API ff_status ff_scorer_load_weights(ff_scorer *s, const char *name, const float *h_data, const int64_t *shape,
                                        int32_t rank, void *stream);
/* FF_E_STATE unless every tensor was loaded.  Derives the TF32 hi / lo splits
 * of the linears' weights (and their transposes) inside the weight arena;
 * synchronizes `stream`.  Loading a tensor after finalize requires finalizing
 * again (ff_score_batch returns FF_E_STATE until then). */
FF_API ff_status ff_scorer_finalize(ff_scorer *s, void *stream);
/* One batch (device buffers, async on `stream`): d_ids / d_mask int32 [B, S]
 * (mask[b][0] must be 1), d_labels int32 [B] in [0, C).  Accumulates into
 * d_head_scores fp64 [num_layers x max_l heads[l]] and d_ffn_scores fp64
 * [num_layers x max_l ffn_dim[l]] (row l holds layer l's units; the caller
 * zeroes them before the first batch).  d_loss (optional) fp32 [1] receives
 * this batch's mean cross-entropy, d_logits (optional) fp32 [B x C] its
 * logits.  FF_E_SHAPE if B*S > max_tokens or S > max_positions. */
FF_API ff_status ff_score_batch(ff_scorer *s, const int32_t *d_ids, const int32_t *d_mask, const int32_t *d_labels,
                                int32_t batch, int32_t seq, double *d_head_scores, double *d_ffn_scores,
                                float *d_loss, float *d_logits, void *stream);
/* Synchronize `stream`; FF_E_INPUT (and clear the flag) if an earlier
 * ff_score_batch saw a token id outside [0, V), a mask value not 0/1 or
 * mask[b][0] != 1, or a label outside [0, C) (such inputs are read as 0, never
 * out of bounds, and that batch's scores are not meaningful), else FF_OK. */
FF_API ff_status ff_scorer_check(ff_scorer *s, void *stream);
/* Scorer options (any time after create; apply to later ff_score_batch calls).
 * FF_SCORER_OPT_TC_LINEARS (default 1): the eight linears per layer (QKV,
 *   out-proj, FFN1, FFN2 and their input gradients) run on the tcgen05 tensor
 *   cores as 3xTF32 (hi / lo TF32 splits, fp32 accumulation: fp32-level error,
 *   DESIGN §6 "importance scorer"); 0 = the SIMT fp32 SGEMM.  The per-head
 *   attention products always use the SIMT SGEMM.
 * FF_E_INVALID for an unknown option or value. */
#define FF_SCORER_OPT_TC_LINEARS 1
/* Test hook: one 3xTF32 tcgen05 GEMM as the scorer's linears run it,
 * d_C[M x N] (+)= d_A[M x K] d_B[N x K]^T (+ d_bias[N], optional), fp32 device
 * buffers with row pitches lda, ldb, ldc (elements); kc = k-blocks of 32 per
 * TMEM accumulation chunk (the scorer uses 4).  Split-K is chosen as in the
 * scorer (workspace for up to 4 partial sums).  Split buffers are allocated
 * stream-ordered (cudaMallocAsync) and freed before return.  Errors via
 * ff_scorer_last_error(). */
FF_API ff_status ff_debug_gemm_x3(const float *d_A, int32_t lda, const float *d_B, int32_t ldb, int32_t M, int32_t N,
                                  int32_t K, const float *d_bias, float *d_C, int32_t ldc, int32_t accumulate,
                                  int32_t kc, void *stream);
FF_API ff_status ff_scorer_set_option(ff_scorer *s, int32_t option, int32_t value);
/* Frees host state only (the arenas belong to the caller). */
FF_API void ff_scorer_destroy(ff_scorer *s);

#ifdef __cplusplus
}
#endif
#endif /* FASTFORMERS_H_ */
