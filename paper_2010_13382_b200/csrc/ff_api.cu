// ff_api.cu -- host side of the C ABI in include/fastformers.h: config
// validation, arena / workspace planning, GPU weight packing at load time
// ("cached weight packing"), TMA tensor maps, the per-call launch
// sequence of the encoder forward and its CUDA-graph cache.
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "fastformers.h"
#include "ff_kernels.h"

namespace ff {
thread_local LaunchPolicy tl_launch;  // set per forward by LaunchScope (ff_kernels.h)
}

namespace {

thread_local std::string g_err;

ff_status fail(ff_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define FF_CK(x)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) return fail(FF_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
int round_up(int x, int a) { return (x + a - 1) / a * a; }

struct Arena {
  size_t off = 0;
  size_t take(size_t bytes) {
    off = align_up(off, 256);
    const size_t o = off;
    off += bytes;
    return o;
  }
};

enum { W_QKV = 0, W_O = 1, W_FFN1 = 2, W_FFN2 = 3 };

// The 16 per-layer HF tensors (bit index = position in this list).
const char* kLayerKeys[16] = {
    "attention.self.query.weight", "attention.self.key.weight", "attention.self.value.weight",
    "attention.self.query.bias", "attention.self.key.bias", "attention.self.value.bias",
    "attention.output.dense.weight", "attention.output.dense.bias", "attention.output.LayerNorm.weight",
    "attention.output.LayerNorm.bias", "intermediate.dense.weight", "intermediate.dense.bias",
    "output.dense.weight", "output.dense.bias", "output.LayerNorm.weight", "output.LayerNorm.bias"};
const char* kTopKeys[9] = {"embeddings.word_embeddings.weight", "embeddings.position_embeddings.weight",
                           "embeddings.token_type_embeddings.weight", "embeddings.LayerNorm.weight",
                           "embeddings.LayerNorm.bias", "pooler.dense.weight", "pooler.dense.bias",
                           "classifier.weight", "classifier.bias"};

struct LayerPlan {
  int A, F, dt, D;
  int Dq;  // QKV section width A * hs (hs = the model's QKV head stride)
  int N[4], K[4], ldw[4];  // GEMM shapes; ldw = packed row pitch in elements
  size_t w[4], sw[4], bias[4], cs[4];  // cs: int32 weight column sums (int8 layers)
  size_t ln1g, ln1b, ln2g, ln2b;
  uint32_t loaded = 0;
  ff::GemmPlan gp[4];
  // row-reduction GEMMs: [0] out-proj + LN1, [1] FFN1 + requant, [2] FFN2 + LN2
  ff::RRPlan rp[3];
  bool rr_ok[2] = {false, false};  // [0] LN fusion (N = H), [1] FFN1 requant fusion (N = F', int8)
};

}  // namespace

struct ff_model {
  ff_config cfg;
  std::vector<int> heads, ffn, dtype;
  int device = 0;
  int state = 0;  // 0 created, 1 bound, 2 ready
  std::vector<LayerPlan> L;
  size_t emb_tok, emb_pos, emb_type, emb_g, emb_b, pool_w, pool_b, cls_w, cls_b;
  uint32_t top_loaded = 0;
  size_t wbytes = 0;
  int Dmax = 0, Fmax = 0, Dqmax = 0;
  // QKV head stride: head_dim rounded up to 8 elements, so every head slice
  // of the QKV buffer starts on a 16-byte boundary (TMA); for head_dim 26
  // (TinyBERT) the fused QKV GEMM writes zero-padded 32-column heads
  int hs = 0;
  // head-major QKV buffer (hs = 64): [3 A heads x hm_rows, 64], every (section,
  // head) slice of a sequence one contiguous block, so the attention's TMA tiles
  // are contiguous 16 KB (the row-major layout reads 128 B from each of 128
  // rows 3 KB apart); hm_rows = max_tokens rounded up to 256 (0: row-major)
  int hm_rows = 0;
  bool any_i8 = false;
  // workspace pitches (elements) and offsets
  int ldx16, ldx8, ldqkv, ldc16, ldc8, ldi16, ldi8;
  size_t ws_x16, ws_xq, ws_xs, ws_qkv, ws_ctx, ws_ctxq, ws_ctxs, ws_o, ws_h1, ws_h1q, ws_h1s, ws_i, ws_iq, ws_is;
  size_t ws_err, ws_ids, ws_mask, ws_logits, ws_pooled, ws_tq;
  size_t ws_ids2, ws_mask2, ws_logits2;  // second host-I/O set (ff_encode_host_async double buffering)
  // ff_encode_host_async: a copy stream brings set k+1's ids / mask in while set k computes
  cudaStream_t io_stream = nullptr;
  cudaEvent_t io_ready[2] = {nullptr, nullptr}, io_free[2] = {nullptr, nullptr};
  int io_set = 0;
  size_t wsbytes = 0;
  uint8_t* dW = nullptr;
  uint8_t* dWS = nullptr;
  bool use_graphs = true;
  int pair_mode = -1;  // FF_OPT_CTA_PAIRS: -1 auto, 0 never (GemmPlan::force_pair)
  bool attn_tc = true;  // FF_OPT_ATTN_TC: tcgen05 attention where supported
  int fused = -1;  // FF_OPT_FUSED_EPILOGUES / _MASK: cluster row-reduction GEMM epilogues,
                  // bit 0 out-proj + LN1, bit 1 FFN1 + requant, bit 2 FFN2 + LN2; -1 = auto
  int act_quant = 0;    // FF_OPT_ACT_QUANT: 0 per-row s8, 1 per-tensor u8 + zero point
  bool cls_last = false;  // FF_OPT_CLS_LAST_LAYER: last layer's row-local steps on the B first-token rows only
  int row_dirs = 0b01010;  // FF_OPT_ROW_DIRS: row-tile direction per launch role (run_forward)
  ff::LaunchPolicy launch{true, false};  // FF_OPT_PDL / FF_OPT_PDL_RR of this model's forwards
  ff::AttnTCPlan tm_qkv;  // QKV buffer map for the tcgen05 attention
  // CUDA-graph cache of ff_encode, keyed by (batch, seq, ids, mask, logits);
  // bounded: the least recently used graph is destroyed beyond kMaxGraphs
  struct CachedGraph {
    cudaGraphExec_t exec;
    uint64_t last_use;
  };
  static constexpr size_t kMaxGraphs = 64;
  std::map<std::tuple<int, int, const void*, const void*, const void*>, CachedGraph> graphs;
  uint64_t graph_clock = 0;

  template <typename T>
  T* w(size_t off) const { return reinterpret_cast<T*>(dW + off); }
  template <typename T>
  T* ws(size_t off) const { return reinterpret_cast<T*>(dWS + off); }
};

namespace {

// Fusions of one layer: an explicit FF_OPT_FUSED_MASK as given; auto (-1,
// the default) fuses the FFN1 requant always and residual + LN into a GEMM
// whose K row is at most 3 KB -- with longer K rows the single-CTA 128-row
// tiles of the row-reduction kernel feed the tensor cores worse than the
// CTA-pair GEMM + add_ln (measured, whole step: C3 fp16 FFN2 3 KB rows fused
// +1.9%, C4 int8 FFN2 3 KB +1.7%, C5 int8 FFN2 4 KB -0.3%, C5 fp16 8 KB -1.1%,
// C4 fp16 FFN2 6 KB fused 337 us vs 220 + 59 us).
constexpr int kFuseMaxKRowBytes = 3072;
int fused_mask(const ff_model* m, const LayerPlan& P) {
  if (m->fused >= 0) return m->fused;
  const int eb = P.dt == FF_I8 ? 1 : 2;
  return 2 | (P.K[1] * eb <= kFuseMaxKRowBytes ? 1 : 0) | (P.K[3] * eb <= kFuseMaxKRowBytes ? 4 : 0);
}

void drop_graphs(ff_model* m) {
  for (auto& kv : m->graphs) cudaGraphExecDestroy(kv.second.exec);
  m->graphs.clear();
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool strip_prefix(std::string& s, const char* p) {
  const size_t n = std::strlen(p);
  if (s.compare(0, n, p) == 0) {
    s = s.substr(n);
    return true;
  }
  return false;
}

void plan_memory(ff_model* m) {
  const ff_config& c = m->cfg;
  const int H = c.hidden;
  Arena wa;
  m->emb_tok = wa.take((size_t)c.vocab_size * H * 4);
  m->emb_pos = wa.take((size_t)c.max_positions * H * 4);
  m->emb_type = wa.take((size_t)H * 4);
  m->emb_g = wa.take((size_t)H * 4);
  m->emb_b = wa.take((size_t)H * 4);
  m->hs = round_up(c.head_dim, 8);
  m->L.resize(c.num_layers);
  for (int l = 0; l < c.num_layers; ++l) {
    LayerPlan& P = m->L[l];
    P.A = m->heads[l];
    P.F = m->ffn[l];
    P.dt = m->dtype[l];
    P.D = P.A * c.head_dim;
    P.Dq = P.A * m->hs;
    const int Ns[4] = {3 * P.Dq, H, P.F, H}, Ks[4] = {H, P.D, H, P.F};
    const int eb = P.dt == FF_I8 ? 1 : 2;
    for (int i = 0; i < 4; ++i) {
      P.N[i] = Ns[i];
      P.K[i] = Ks[i];
      P.ldw[i] = round_up(Ks[i], 16 / eb);
      P.w[i] = wa.take((size_t)Ns[i] * P.ldw[i] * eb);
      P.sw[i] = P.dt == FF_I8 ? wa.take((size_t)Ns[i] * 4) : 0;
      P.cs[i] = P.dt == FF_I8 ? wa.take((size_t)Ns[i] * 4) : 0;
      P.bias[i] = wa.take((size_t)Ns[i] * 4);
    }
    P.ln1g = wa.take((size_t)H * 4);
    P.ln1b = wa.take((size_t)H * 4);
    P.ln2g = wa.take((size_t)H * 4);
    P.ln2b = wa.take((size_t)H * 4);
    m->Dmax = std::max(m->Dmax, P.D);
    m->Dqmax = std::max(m->Dqmax, P.Dq);
    m->Fmax = std::max(m->Fmax, P.F);
    m->any_i8 = m->any_i8 || P.dt == FF_I8;
  }
  m->pool_w = wa.take((size_t)H * H * 4);
  m->pool_b = wa.take((size_t)H * 4);
  m->cls_w = wa.take((size_t)c.num_classes * H * 4);
  m->cls_b = wa.take((size_t)c.num_classes * 4);
  m->wbytes = align_up(wa.off, 256);

  const size_t M = (size_t)c.max_tokens;
  m->ldx16 = round_up(H, 8);
  m->ldx8 = round_up(H, 16);
  m->ldqkv = round_up(3 * m->Dqmax, 8);
  m->ldc16 = round_up(m->Dmax, 8);
  m->ldc8 = round_up(m->Dmax, 16);
  m->ldi16 = round_up(m->Fmax, 8);
  m->ldi8 = round_up(m->Fmax, 16);
  Arena a;
  const bool q = m->any_i8;
  m->ws_x16 = a.take(M * m->ldx16 * 2);
  m->ws_xq = q ? a.take(M * m->ldx8) : 0;
  m->ws_xs = q ? a.take(M * 4) : 0;
  m->hm_rows = m->hs == 64 ? round_up((int)M, 256) : 0;
  m->ws_qkv = m->hm_rows > 0 ? a.take((size_t)3 * (m->Dqmax / 64) * m->hm_rows * 64 * 2) : a.take(M * m->ldqkv * 2);
  m->ws_ctx = a.take(M * m->ldc16 * 2);
  m->ws_ctxq = q ? a.take(M * m->ldc8) : 0;
  m->ws_ctxs = q ? a.take(M * 4) : 0;
  m->ws_o = a.take(M * m->ldx16 * 2);
  m->ws_h1 = a.take(M * m->ldx16 * 2);
  m->ws_h1q = q ? a.take(M * m->ldx8) : 0;
  m->ws_h1s = q ? a.take(M * 4) : 0;
  m->ws_i = a.take(M * m->ldi16 * 2);
  m->ws_iq = q ? a.take(M * m->ldi8) : 0;
  m->ws_is = q ? a.take(M * 4) : 0;
  m->ws_err = a.take(256);
  m->ws_tq = a.take(256);  // per-tensor quantizer: uint mm[2], float qp[2]
  m->ws_ids = a.take(M * 4);
  m->ws_mask = a.take(M * 4);
  m->ws_logits = a.take(M * c.num_classes * 4);
  m->ws_ids2 = a.take(M * 4);
  m->ws_mask2 = a.take(M * 4);
  m->ws_logits2 = a.take(M * c.num_classes * 4);
  m->ws_pooled = a.take(M * H * 4);  // pooler split-K partials [<= S][B][H] fp32
  m->wsbytes = align_up(a.off, 256);
}

// A-operand buffer of GEMM i of layer P.
const void* gemm_a(const ff_model* m, const LayerPlan& P, int i, int* lda) {
  const bool q = P.dt == FF_I8;
  switch (i) {
    case W_QKV: *lda = q ? m->ldx8 : m->ldx16; return m->dWS + (q ? m->ws_xq : m->ws_x16);
    case W_O: *lda = q ? m->ldc8 : m->ldc16; return m->dWS + (q ? m->ws_ctxq : m->ws_ctx);
    case W_FFN1: *lda = q ? m->ldx8 : m->ldx16; return m->dWS + (q ? m->ws_h1q : m->ws_h1);
    default: *lda = q ? m->ldi8 : m->ldi16; return m->dWS + (q ? m->ws_iq : m->ws_i);
  }
}

ff_status build_gemm_plans(ff_model* m) {
  for (size_t l = 0; l < m->L.size(); ++l) {
    LayerPlan& P = m->L[l];
    for (int i = 0; i < 4; ++i) {
      int lda;
      const void* A = gemm_a(m, P, i, &lda);
      const char* err = nullptr;
      if (!ff::plan_gemm(&P.gp[i], P.dt == FF_I8, A, m->cfg.max_tokens, lda, m->dW + P.w[i], P.ldw[i], P.N[i],
                         P.K[i], &err))
        return fail(FF_E_CUDA, std::string("tensor map: ") + err);
      void* out = nullptr;
      int ldo = 0;
      switch (i) {
        case W_QKV: out = m->dWS + m->ws_qkv; ldo = m->ldqkv; break;
        case W_O: out = m->dWS + m->ws_o; ldo = m->ldx16; break;
        case W_FFN1: out = m->dWS + m->ws_i; ldo = m->ldi16; break;
        default: out = m->dWS + m->ws_o; ldo = m->ldx16; break;
      }
      const bool ok = (i == W_QKV && m->hm_rows > 0) ? ff::plan_gemm_output_hm(&P.gp[i], out, m->hm_rows, &err)
                                                     : ff::plan_gemm_output(&P.gp[i], out, ldo, &err);
      if (!ok) return fail(FF_E_CUDA, std::string("output tensor map: ") + err);
    }
    // fused row-reduction epilogues where the output row fits a cluster (N = 256 x 1..8)
    const bool q = P.dt == FF_I8;
    const char* err = nullptr;
    P.rr_ok[0] = ff::rr_supported(m->cfg.hidden);
    P.rr_ok[1] = q && ff::rr_supported(P.F);
    if (P.rr_ok[0]) {
      int lda;
      const void* A = gemm_a(m, P, W_O, &lda);
      if (!ff::plan_rr(&P.rp[0], q, A, m->cfg.max_tokens, lda, m->dW + P.w[W_O], P.ldw[W_O], P.N[W_O], P.K[W_O],
                       m->dWS + m->ws_h1, m->ldx16, &err))
        return fail(FF_E_CUDA, std::string("rr tensor map: ") + err);
      P.rp[0].p.mode = ff::RR_LN;
      if (!ff::plan_rr_io(&P.rp[0], m->dWS + m->ws_x16, m->ldx16, q ? m->dWS + m->ws_h1q : nullptr, m->ldx8, &err))
        return fail(FF_E_CUDA, std::string("rr tensor map: ") + err);
      A = gemm_a(m, P, W_FFN2, &lda);
      if (!ff::plan_rr(&P.rp[2], q, A, m->cfg.max_tokens, lda, m->dW + P.w[W_FFN2], P.ldw[W_FFN2], P.N[W_FFN2],
                       P.K[W_FFN2], m->dWS + m->ws_x16, m->ldx16, &err))
        return fail(FF_E_CUDA, std::string("rr tensor map: ") + err);
      P.rp[2].p.mode = ff::RR_LN;
      const bool nq = l + 1 < m->L.size() && m->L[l + 1].dt == FF_I8;
      if (!ff::plan_rr_io(&P.rp[2], m->dWS + m->ws_h1, m->ldx16, nq ? m->dWS + m->ws_xq : nullptr, m->ldx8, &err))
        return fail(FF_E_CUDA, std::string("rr tensor map: ") + err);
    }
    if (P.rr_ok[1]) {
      int lda;
      const void* A = gemm_a(m, P, W_FFN1, &lda);
      if (!ff::plan_rr(&P.rp[1], true, A, m->cfg.max_tokens, lda, m->dW + P.w[W_FFN1], P.ldw[W_FFN1], P.N[W_FFN1],
                       P.K[W_FFN1], m->dWS + m->ws_i, m->ldi16, &err))
        return fail(FF_E_CUDA, std::string("rr tensor map: ") + err);
      P.rp[1].p.mode = ff::RR_QUANT;
      if (!ff::plan_rr_io(&P.rp[1], nullptr, 0, m->dWS + m->ws_iq, m->ldi8, &err))
        return fail(FF_E_CUDA, std::string("rr tensor map: ") + err);
    }
  }
  return FF_OK;
}

ff_status check_launch(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(FF_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return FF_OK;
}

// Optional per-launch CUDA-event timing (ff_profile).
struct Prof {
  std::vector<cudaEvent_t> ev;
  std::vector<int> kind;
  void mark(cudaStream_t s) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
  }
  ~Prof() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};

#define FF_LAUNCH(kind_, x, what)                   \
  do {                                              \
    if (prof) {                                     \
      prof->kind.push_back(kind_);                  \
      prof->mark(s);                                \
    }                                               \
    ff_status s_ = check_launch((x), what);         \
    if (s_ != FF_OK) return s_;                     \
    if (prof) prof->mark(s);                        \
  } while (0)

ff_status dump(void* dst, const void* src, int ld_elems, int cols, int M, cudaStream_t s) {
  if (!dst) return FF_OK;
  FF_CK(cudaMemcpy2DAsync(dst, (size_t)cols * 2, src, (size_t)ld_elems * 2, (size_t)cols * 2, M,
                          cudaMemcpyDeviceToDevice, s));
  return FF_OK;
}

// int8 layer whose ctx requant (a4) runs inside the tcgen05 attention kernel:
// the fused kernel needs a whole sequence per work item, so it is used only
// when the batch alone fills the SMs (C3: B = 256); smaller batches (C2: 64)
// spread heads over all SMs and requantize with quant_rows.
bool attention_fuses_quant(const ff_model* m, const LayerPlan& P, int B, int S) {
  return P.dt == FF_I8 && m->attn_tc && B >= ff::kNumSMs &&
         ff::attention_tc_supported(S, m->cfg.head_dim, m->hs, m->ldqkv, m->ldc16) &&
         ff::attention_tc_fuses_quant(P.A, m->cfg.head_dim);
}

// ff_debug_set_trace: timeline buffer and target (0 debug GEMMs; 1 / 2 / 3 the
// layer-0 fused out-proj+LN / FFN1+requant / FFN2+LN of the next forward).
static unsigned long long* g_debug_trace = nullptr;
static int g_debug_trace_which = 0;

// The launch sequence of one encoder forward.
ff_status run_forward(ff_model* m, const int32_t* ids, const int32_t* mask, int B, int S, float* logits,
                      cudaStream_t s, int trace_layer, void* const* d_dump, Prof* prof = nullptr) {
  const ff::LaunchScope launch_scope(m->launch);  // this model's PDL policy for the launches below
  const ff_config& c = m->cfg;
  const int H = c.hidden, M = B * S;
  __half* X16 = m->ws<__half>(m->ws_x16);
  int8_t* Xq = m->ws<int8_t>(m->ws_xq);
  float* Xs = m->ws<float>(m->ws_xs);
  __half* QKV = m->ws<__half>(m->ws_qkv);
  __half* CTX = m->ws<__half>(m->ws_ctx);
  int8_t* CTXq = m->ws<int8_t>(m->ws_ctxq);
  float* CTXs = m->ws<float>(m->ws_ctxs);
  __half* O16 = m->ws<__half>(m->ws_o);
  __half* H1 = m->ws<__half>(m->ws_h1);
  int8_t* H1q = m->ws<int8_t>(m->ws_h1q);
  float* H1s = m->ws<float>(m->ws_h1s);
  __half* I16 = m->ws<__half>(m->ws_i);
  int8_t* Iq = m->ws<int8_t>(m->ws_iq);
  float* Is = m->ws<float>(m->ws_is);
  // per-tensor u8 activations (FF_OPT_ACT_QUANT = 1, DESIGN R22): the s8
  // producers write fp16 only and every int8 GEMM input is quantized as a
  // whole tensor right before its GEMM
  const bool pt = m->act_quant == 1;
  const bool l0q = m->L[0].dt == FF_I8 && !pt;
  unsigned* tq_mm = reinterpret_cast<unsigned*>(m->dWS + m->ws_tq);
  float* tq_qp = reinterpret_cast<float*>(m->dWS + m->ws_tq + 64);
  auto tensor_quant = [&](const __half* x, int ldx, int K, int8_t* q8, int ldq, ff::GemmPlan& gp,
                          const LayerPlan& P, int which) -> ff_status {
    FF_LAUNCH(FF_K_QUANT, ff::launch_quant_tensor(x, ldx, M, K, tq_mm, reinterpret_cast<uint8_t*>(q8), ldq, tq_qp, s),
              "quant tensor");
    gp.p.row_scale = nullptr;
    gp.p.tensor_qp = tq_qp;
    gp.p.colsum = m->w<int>(P.cs[which]);
    return FF_OK;
  };

  FF_LAUNCH(FF_K_EMBED_LN, ff::launch_embed_ln(ids, mask, B, S, H, c.vocab_size, m->w<float>(m->emb_tok), m->w<float>(m->emb_pos),
                                m->w<float>(m->emb_g), m->w<float>(m->emb_b), c.ln_eps, X16, m->ldx16,
                                l0q ? Xq : nullptr, m->ldx8, l0q ? Xs : nullptr, m->ws<int>(m->ws_err), s),
            "embed_ln");
  // Row-tile direction per launch role (bits, high to low: QKV, attention,
  // out-proj, FFN1, FFN2; 1 = last row tile first).  A kernel that walks its
  // rows opposite to its producer first reads the rows written last, the
  // most likely to still be in L2: the attention reads the QKV GEMM's output
  // last-written-first, the FFN1 GEMM the out-proj's, and their successors
  // (out-proj, FFN2) then read in increasing order what was written in
  // decreasing order.  Measured on C3 int8 (same-box A/B, every mask):
  // 0b01010 +1.1% over all-forward; 0b01000 +0.7%; alternating every launch
  // +0.3%.
  const int rmask = m->row_dirs;
  int role = 0;
  int rdir = (rmask >> 4) & 1;
  for (int l = 0; l < c.num_layers; ++l) {
    LayerPlan& P = m->L[l];
    const bool q = P.dt == FF_I8;
    const bool tr = l == trace_layer;
    if (tr && dump(d_dump[0], X16, m->ldx16, H, M, s) != FF_OK) return FF_E_CUDA;
    // a2: fused QKV projection
    ff::GemmPlan g = P.gp[W_QKV];
    g.force_pair = m->pair_mode;
    ff::plan_gemm_set_m(&g, M);
    g.p.out = QKV;
    g.p.ldo = m->hm_rows > 0 ? 64 : m->ldqkv;
    g.p.bias = m->w<float>(P.bias[W_QKV]);
    g.p.row_scale = q ? Xs : nullptr;
    g.p.col_scale = q ? m->w<float>(P.sw[W_QKV]) : nullptr;
    g.p.act = ff::ACT_NONE;
    g.p.rev = rdir;
    role = (role + 1) % 5;
    rdir = (rmask >> (4 - role)) & 1;
    if (q && pt && tensor_quant(X16, m->ldx16, H, Xq, m->ldx8, g, P, W_QKV) != FF_OK) return FF_E_CUDA;
    FF_LAUNCH(q ? FF_K_GEMM_I8 : FF_K_GEMM_F16, ff::launch_gemm(g, s), "gemm qkv");
    if (tr) {  // the trace holds the unpadded row-major [M, 3 D] Q | K | V rows
      if (m->hm_rows == 0 && m->hs == c.head_dim) {
        if (dump(d_dump[1], QKV, m->ldqkv, 3 * P.D, M, s) != FF_OK) return FF_E_CUDA;
      } else if (d_dump[1]) {
        for (int t = 0; t < 3; ++t)
          for (int h = 0; h < P.A; ++h) {
            const __half* src = m->hm_rows > 0 ? QKV + (size_t)(t * P.A + h) * m->hm_rows * 64
                                               : QKV + t * P.Dq + h * m->hs;
            const size_t spitch = m->hm_rows > 0 ? 128 : (size_t)m->ldqkv * 2;
            FF_CK(cudaMemcpy2DAsync(static_cast<__half*>(d_dump[1]) + t * P.D + h * c.head_dim, (size_t)3 * P.D * 2,
                                    src, spitch, (size_t)c.head_dim * 2, M, cudaMemcpyDeviceToDevice, s));
          }
      }
    }
    // a3: fused masked-softmax attention over this layer's A'_l heads
    // (int8 layers: a4, the ctx requant, fused into the tcgen05 attention)
    const bool att_q = attention_fuses_quant(m, P, B, S) && !pt;
    if (m->attn_tc && ff::attention_tc_supported(S, c.head_dim, m->hs, m->ldqkv, m->ldc16))
      FF_LAUNCH(FF_K_ATTENTION,
                ff::launch_attention_tc(m->tm_qkv, mask, B, S, P.A, c.head_dim, m->hs, (att_q && !tr) ? nullptr : CTX,
                                        m->ldc16,
                                        att_q ? CTXq : nullptr, m->ldc8, att_q ? CTXs : nullptr, s, nullptr, rdir),
                "attention_tc");
    else if (m->attn_tc && m->hs == c.head_dim && ff::attention_long_supported(S, c.head_dim, m->ldqkv, m->ldc16))
      FF_LAUNCH(FF_K_ATTENTION, ff::launch_attention_long(m->tm_qkv, mask, B, S, P.A, CTX, m->ldc16, s),
                "attention_long");
    else
      FF_LAUNCH(FF_K_ATTENTION,
                ff::launch_attention(QKV, m->hm_rows > 0 ? 64 : m->ldqkv, mask, B, S, P.A, c.head_dim, m->hs,
                                     m->hm_rows, CTX, m->ldc16, s),
                "attention");
    role = (role + 1) % 5;
    rdir = (rmask >> (4 - role)) & 1;
    if (tr && dump(d_dump[2], CTX, m->ldc16, P.D, M, s) != FF_OK) return FF_E_CUDA;
    // a4 + a5: requant (int8 layers) and out-projection
    if (q && !att_q && !pt)
      FF_LAUNCH(FF_K_QUANT, ff::launch_quant_rows(CTX, m->ldc16, M, P.D, CTXq, m->ldc8, CTXs, s), "quant ctx");
    // FF_OPT_CLS_LAST_LAYER: the classifier reads only the first token of each
    // sequence (a11), and a5-a10 are row-local, so in the last layer they run
    // on the B rows b*S (read with an S-row pitch) and write compact rows
    // [0, B); the logits are bit-identical (tests/test_gpu_model.py)
    const bool cls = m->cls_last && l + 1 == c.num_layers && !pt && !tr;
    const int Mr = cls ? B : M;
    const char* rerr = nullptr;
    const int lda_o = q ? m->ldc8 : m->ldc16;
    const void* A_o = q ? static_cast<const void*>(CTXq) : static_cast<const void*>(CTX);
    const int fm = fused_mask(m, P);
    const bool fuse_ln = (fm & 1) && !pt && P.rr_ok[0];
    const bool fuse_q = (fm & 2) && !pt && q && P.rr_ok[1];
    const bool fuse_ln2 = (fm & 4) && !pt && P.rr_ok[0];
    if (fuse_ln) {
      // a5 + a6 fused: H1 = LN1(R16(O) + X16) (+ s8 rows) in the out-proj epilogue
      ff::RRPlan r = P.rp[0];
      if (cls) {
        if (!ff::rebind_rr_rows(&r, A_o, lda_o * S, X16, m->ldx16 * S, B, &rerr))
          return fail(FF_E_CUDA, std::string("rr tensor map: ") + rerr);
        r.p.rs_stride = S;
      }
      ff::plan_rr_set_m(&r, Mr);
      r.p.bias = m->w<float>(P.bias[W_O]);
      r.p.row_scale = q ? CTXs : nullptr;
      r.p.col_scale = q ? m->w<float>(P.sw[W_O]) : nullptr;
      r.p.residual = X16;
      r.p.ldr = cls ? m->ldx16 * S : m->ldx16;
      r.p.gamma = m->w<float>(P.ln1g);
      r.p.beta = m->w<float>(P.ln1b);
      r.p.eps = c.ln_eps;
      r.p.store16 = 1;
      r.p.outq = q ? H1q : nullptr;
      r.p.ldq = m->ldx8;
      r.p.out_scale = q ? H1s : nullptr;
      r.p.trace = (l == 0 && g_debug_trace_which == 1) ? g_debug_trace : nullptr;
      r.p.rev = rdir;
      FF_LAUNCH(q ? FF_K_GEMM_RR_I8 : FF_K_GEMM_RR_F16, ff::launch_rr(r, s), "gemm o + ln1");
    } else {
    g = P.gp[W_O];
    g.force_pair = m->pair_mode;
    if (cls) {
      if (!ff::rebind_gemm_rows(&g, A_o, lda_o * S, B, &rerr)) return fail(FF_E_CUDA, std::string("tensor map: ") + rerr);
      g.p.rs_stride = S;
    }
    ff::plan_gemm_set_m(&g, Mr);
    g.p.out = O16;
    g.p.ldo = m->ldx16;
    g.p.bias = m->w<float>(P.bias[W_O]);
    g.p.row_scale = q ? CTXs : nullptr;
    g.p.col_scale = q ? m->w<float>(P.sw[W_O]) : nullptr;
    g.p.act = ff::ACT_NONE;
    g.p.rev = rdir;
    if (q && pt && tensor_quant(CTX, m->ldc16, P.D, CTXq, m->ldc8, g, P, W_O) != FF_OK) return FF_E_CUDA;
    FF_LAUNCH(q ? FF_K_GEMM_I8 : FF_K_GEMM_F16, ff::launch_gemm(g, s), "gemm o");
    if (tr && dump(d_dump[3], O16, m->ldx16, H, M, s) != FF_OK) return FF_E_CUDA;
    // a6: residual + LN1 (+ s8 rows for FFN1)
    FF_LAUNCH(FF_K_ADD_LN, ff::launch_add_ln(O16, m->ldx16, X16, cls ? m->ldx16 * S : m->ldx16, Mr, H, m->w<float>(P.ln1g), m->w<float>(P.ln1b),
                                c.ln_eps, H1, m->ldx16, (q && !pt) ? H1q : nullptr, m->ldx8,
                                (q && !pt) ? H1s : nullptr, s),
              "add_ln1");
    }
    role = (role + 1) % 5;
    rdir = (rmask >> (4 - role)) & 1;
    if (tr && dump(d_dump[4], H1, m->ldx16, H, M, s) != FF_OK) return FF_E_CUDA;
    // a7: FFN1 + bias + activation
    if (fuse_q) {
      // a7 + a8 fused: Iq, Is = Q8row(R16(act(FFN1))) in the FFN1 epilogue; the
      // fp16 copy of I is only materialised when a trace asks for it
      ff::RRPlan r = P.rp[1];
      ff::plan_rr_set_m(&r, Mr);
      r.p.bias = m->w<float>(P.bias[W_FFN1]);
      r.p.row_scale = H1s;
      r.p.col_scale = m->w<float>(P.sw[W_FFN1]);
      r.p.act = c.act;
      r.p.store16 = tr ? 1 : 0;
      r.p.outq = Iq;
      r.p.ldq = m->ldi8;
      r.p.out_scale = Is;
      r.p.trace = (l == 0 && g_debug_trace_which == 2) ? g_debug_trace : nullptr;
      r.p.rev = rdir;
      FF_LAUNCH(FF_K_GEMM_RR_I8, ff::launch_rr(r, s), "gemm ffn1 + quant");
      if (tr && dump(d_dump[5], I16, m->ldi16, P.F, M, s) != FF_OK) return FF_E_CUDA;
    } else {
    g = P.gp[W_FFN1];
    g.force_pair = m->pair_mode;
    ff::plan_gemm_set_m(&g, Mr);
    g.p.out = I16;
    g.p.ldo = m->ldi16;
    g.p.bias = m->w<float>(P.bias[W_FFN1]);
    g.p.row_scale = q ? H1s : nullptr;
    g.p.col_scale = q ? m->w<float>(P.sw[W_FFN1]) : nullptr;
    g.p.act = c.act;
    g.p.rev = rdir;
    if (q && pt && tensor_quant(H1, m->ldx16, H, H1q, m->ldx8, g, P, W_FFN1) != FF_OK) return FF_E_CUDA;
    FF_LAUNCH(q ? FF_K_GEMM_I8 : FF_K_GEMM_F16, ff::launch_gemm(g, s), "gemm ffn1");
    if (tr && dump(d_dump[5], I16, m->ldi16, P.F, M, s) != FF_OK) return FF_E_CUDA;
    // a8 + a9: requant and FFN2
    if (q && !pt) FF_LAUNCH(FF_K_QUANT, ff::launch_quant_rows(I16, m->ldi16, Mr, P.F, Iq, m->ldi8, Is, s), "quant ffn");
    }
    role = (role + 1) % 5;
    rdir = (rmask >> (4 - role)) & 1;
    const bool nq = l + 1 < c.num_layers && m->L[l + 1].dt == FF_I8 && !pt;
    if (fuse_ln2) {
      // a9 + a10 fused: X16 = LN2(R16(Y) + H1) (+ s8 rows for the next int8 layer)
      ff::RRPlan r = P.rp[2];
      ff::plan_rr_set_m(&r, Mr);
      r.p.bias = m->w<float>(P.bias[W_FFN2]);
      r.p.row_scale = q ? Is : nullptr;
      r.p.col_scale = q ? m->w<float>(P.sw[W_FFN2]) : nullptr;
      r.p.residual = H1;
      r.p.ldr = m->ldx16;
      r.p.gamma = m->w<float>(P.ln2g);
      r.p.beta = m->w<float>(P.ln2b);
      r.p.eps = c.ln_eps;
      r.p.store16 = 1;
      r.p.outq = nq ? Xq : nullptr;
      r.p.ldq = m->ldx8;
      r.p.out_scale = nq ? Xs : nullptr;
      r.p.trace = (l == 0 && g_debug_trace_which == 3) ? g_debug_trace : nullptr;
      r.p.rev = rdir;
      FF_LAUNCH(q ? FF_K_GEMM_RR_I8 : FF_K_GEMM_RR_F16, ff::launch_rr(r, s), "gemm ffn2 + ln2");
    } else {
    g = P.gp[W_FFN2];
    g.force_pair = m->pair_mode;
    ff::plan_gemm_set_m(&g, Mr);
    g.p.out = O16;
    g.p.ldo = m->ldx16;
    g.p.bias = m->w<float>(P.bias[W_FFN2]);
    g.p.row_scale = q ? Is : nullptr;
    g.p.col_scale = q ? m->w<float>(P.sw[W_FFN2]) : nullptr;
    g.p.act = ff::ACT_NONE;
    g.p.rev = rdir;
    if (q && pt && tensor_quant(I16, m->ldi16, P.F, Iq, m->ldi8, g, P, W_FFN2) != FF_OK) return FF_E_CUDA;
    FF_LAUNCH(q ? FF_K_GEMM_I8 : FF_K_GEMM_F16, ff::launch_gemm(g, s), "gemm ffn2");
    if (tr && dump(d_dump[6], O16, m->ldx16, H, M, s) != FF_OK) return FF_E_CUDA;
    // a10: residual + LN2 (+ s8 rows when the next layer is int8)
    FF_LAUNCH(FF_K_ADD_LN, ff::launch_add_ln(O16, m->ldx16, H1, m->ldx16, Mr, H, m->w<float>(P.ln2g), m->w<float>(P.ln2b),
                                c.ln_eps, X16, m->ldx16, nq ? Xq : nullptr, m->ldx8, nq ? Xs : nullptr, s),
              "add_ln2");
    }
    role = (role + 1) % 5;
    rdir = (rmask >> (4 - role)) & 1;
    if (tr && dump(d_dump[7], X16, m->ldx16, H, M, s) != FF_OK) return FF_E_CUDA;
  }
  // a11: pooler + classifier
  // (with FF_OPT_CLS_LAST_LAYER the first-token rows are compact rows [0, B))
  const bool cls_out = m->cls_last && !pt && trace_layer != c.num_layers - 1;
  FF_LAUNCH(FF_K_HEAD, ff::launch_head(X16, m->ldx16, B, S, H, c.num_classes, m->w<float>(m->pool_w), m->w<float>(m->pool_b),
                            m->w<float>(m->cls_w), m->w<float>(m->cls_b), m->ws<float>(m->ws_pooled), logits, s, cls_out ? 1 : S),
            "head");
  return FF_OK;
}

ff_status check_call(const ff_model* m, int B, int S) {
  if (!m) return fail(FF_E_INVALID, "null model");
  if (m->state != 2) return fail(FF_E_STATE, "model not finalized");
  if (B < 1 || S < 1) return fail(FF_E_SHAPE, "batch and seq must be >= 1");
  if (S > m->cfg.max_positions) return fail(FF_E_SHAPE, "seq > max_positions");
  if ((int64_t)B * S > m->cfg.max_tokens) return fail(FF_E_SHAPE, "batch*seq > max_tokens");
  if (ff::attention_smem_bytes(S, m->cfg.head_dim) > 227 * 1024)
    return fail(FF_E_UNSUPPORTED, "seq too long for the attention kernel at this head_dim");
  return FF_OK;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int32_t ff_abi_version(void) { return FF_ABI_VERSION; }
const char* ff_last_error(void) { return g_err.c_str(); }

ff_status ff_model_create(const ff_config* cfg, int32_t cuda_device, ff_model** out) {
  if (!cfg || !out) return fail(FF_E_INVALID, "null argument");
  *out = nullptr;
  if (cfg->abi_version != FF_ABI_VERSION) return fail(FF_E_INVALID, "abi_version mismatch");
  const ff_config& c = *cfg;
  if (c.num_layers < 1 || c.hidden < 1 || c.head_dim < 1 || c.vocab_size < 1 || c.max_positions < 1 ||
      c.num_classes < 1 || c.max_tokens < 1 || !(c.ln_eps > 0.0f))
    return fail(FF_E_INVALID, "config values must be positive");
  if (c.act < FF_ACT_GELU || c.act > FF_ACT_GELU_TANH) return fail(FF_E_INVALID, "bad act");
  if (!c.heads || !c.ffn_dim || !c.dtype) return fail(FF_E_INVALID, "null per-layer array");
  if (c.head_dim > 128 || (c.head_dim & 1)) return fail(FF_E_INVALID, "head_dim must be even and <= 128");
  if (c.hidden % 8 || c.hidden > 1024) return fail(FF_E_UNSUPPORTED, "hidden must be a multiple of 8 and <= 1024");
  ff_model* m = new ff_model();
  m->cfg = c;
  for (int l = 0; l < c.num_layers; ++l) {
    if (c.heads[l] < 1 || c.ffn_dim[l] < 1 || (c.dtype[l] != FF_F16 && c.dtype[l] != FF_I8)) {
      delete m;
      return fail(FF_E_INVALID, "layer " + std::to_string(l) + ": heads/ffn_dim must be >= 1, dtype 0/1");
    }
    m->heads.push_back(c.heads[l]);
    m->ffn.push_back(c.ffn_dim[l]);
    m->dtype.push_back(c.dtype[l]);
  }
  m->cfg.heads = m->heads.data();
  m->cfg.ffn_dim = m->ffn.data();
  m->cfg.dtype = m->dtype.data();
  m->device = cuda_device;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, cuda_device);
  if (e != cudaSuccess) {
    delete m;
    return fail(FF_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  if (prop.major != 10 || prop.minor != 0) {
    delete m;
    return fail(FF_E_CUDA, "this library is built for sm_100a (B200) only");
  }
  plan_memory(m);
  *out = m;
  return FF_OK;
}

ff_status ff_model_memory(const ff_model* m, size_t* weight_bytes, size_t* workspace_bytes) {
  if (!m) return fail(FF_E_INVALID, "null model");
  if (weight_bytes) *weight_bytes = m->wbytes;
  if (workspace_bytes) *workspace_bytes = m->wsbytes;
  return FF_OK;
}

ff_status ff_bind_memory(ff_model* m, void* d_weights, size_t weight_bytes, void* d_workspace, size_t workspace_bytes,
                         void* stream) {
  if (!m) return fail(FF_E_INVALID, "null model");
  if (m->state != 0) return fail(FF_E_STATE, "memory already bound");
  if (!d_weights || !d_workspace) return fail(FF_E_INVALID, "null buffer");
  if (weight_bytes < m->wbytes || workspace_bytes < m->wsbytes) return fail(FF_E_NOMEM, "buffer too small");
  if ((reinterpret_cast<uintptr_t>(d_weights) & 255) || (reinterpret_cast<uintptr_t>(d_workspace) & 255))
    return fail(FF_E_INVALID, "buffers must be 256-byte aligned");
  DeviceGuard dg(m->device);
  m->dW = static_cast<uint8_t*>(d_weights);
  m->dWS = static_cast<uint8_t*>(d_workspace);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FF_CK(cudaMemsetAsync(m->dW, 0, m->wbytes, s));
  FF_CK(cudaMemsetAsync(m->dWS, 0, m->wsbytes, s));
  FF_CK(cudaStreamSynchronize(s));
  m->state = 1;
  return FF_OK;
}

ff_status ff_load_weights(ff_model* m, const char* cname, const float* h_data, const int64_t* shape, int32_t rank,
                          void* stream) {
  if (!m || !cname || !h_data || !shape) return fail(FF_E_INVALID, "null argument");
  if (m->state != 1) return fail(FF_E_STATE, m->state == 0 ? "bind memory first" : "model already finalized");
  DeviceGuard dg(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const ff_config& c = m->cfg;
  const int H = c.hidden;
  std::string name(cname);
  strip_prefix(name, "bert.") || strip_prefix(name, "roberta.");
  if (name == "classifier.dense.weight") name = "pooler.dense.weight";
  else if (name == "classifier.dense.bias") name = "pooler.dense.bias";
  else if (name == "classifier.out_proj.weight") name = "classifier.weight";
  else if (name == "classifier.out_proj.bias") name = "classifier.bias";

  auto shape_is = [&](std::initializer_list<int64_t> want) {
    if ((int)want.size() != rank) return false;
    int i = 0;
    for (int64_t w : want) {
      if (w >= 0 && shape[i] != w) return false;
      if (shape[i] < 1) return false;
      ++i;
    }
    return true;
  };
  auto bad_shape = [&]() { return fail(FF_E_SHAPE, "wrong shape for " + name); };
  auto copy_f32 = [&](size_t off, size_t n) -> ff_status {
    FF_CK(cudaMemcpyAsync(m->dW + off, h_data, n * 4, cudaMemcpyHostToDevice, s));
    FF_CK(cudaStreamSynchronize(s));
    return FF_OK;
  };

  // ---- non-layer tensors
  for (int i = 0; i < 9; ++i) {
    if (name != kTopKeys[i]) continue;
    ff_status st;
    switch (i) {
      case 0: if (!shape_is({c.vocab_size, H})) return bad_shape(); st = copy_f32(m->emb_tok, (size_t)c.vocab_size * H); break;
      case 1: if (!shape_is({c.max_positions, H})) return bad_shape(); st = copy_f32(m->emb_pos, (size_t)c.max_positions * H); break;
      case 2: if (!shape_is({-1, H})) return bad_shape(); st = copy_f32(m->emb_type, H); break;  // row 0 only
      case 3: if (!shape_is({H})) return bad_shape(); st = copy_f32(m->emb_g, H); break;
      case 4: if (!shape_is({H})) return bad_shape(); st = copy_f32(m->emb_b, H); break;
      case 5: if (!shape_is({H, H})) return bad_shape(); st = copy_f32(m->pool_w, (size_t)H * H); break;
      case 6: if (!shape_is({H})) return bad_shape(); st = copy_f32(m->pool_b, H); break;
      case 7: if (!shape_is({c.num_classes, H})) return bad_shape(); st = copy_f32(m->cls_w, (size_t)c.num_classes * H); break;
      default: if (!shape_is({c.num_classes})) return bad_shape(); st = copy_f32(m->cls_b, c.num_classes); break;
    }
    if (st != FF_OK) return st;
    m->top_loaded |= 1u << i;
    return FF_OK;
  }
  // ---- per-layer tensors
  std::string rest = name;
  if (!strip_prefix(rest, "encoder.layer.")) return fail(FF_E_SHAPE, "unknown tensor " + name);
  const size_t dot = rest.find('.');
  if (dot == std::string::npos || dot == 0) return fail(FF_E_SHAPE, "unknown tensor " + name);
  for (size_t i = 0; i < dot; ++i)
    if (rest[i] < '0' || rest[i] > '9') return fail(FF_E_SHAPE, "unknown tensor " + name);
  const int l = std::atoi(rest.substr(0, dot).c_str());
  if (l < 0 || l >= c.num_layers) return fail(FF_E_SHAPE, "layer index out of range in " + name);
  const std::string key = rest.substr(dot + 1);
  int ki = -1;
  for (int i = 0; i < 16; ++i)
    if (key == kLayerKeys[i]) ki = i;
  if (ki < 0) return fail(FF_E_SHAPE, "unknown tensor " + name);
  LayerPlan& P = m->L[l];
  const int D = P.D, F = P.F;

  // GEMM weights go through a device staging buffer and a packing kernel.
  auto pack_weight = [&](int which, int row0, int N, int K) -> ff_status {
    float* stage = nullptr;
    FF_CK(cudaMalloc(&stage, (size_t)N * K * 4));
    cudaError_t e = cudaMemcpyAsync(stage, h_data, (size_t)N * K * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
      if (P.dt == FF_I8)
        e = ff::launch_quant_weight(stage, N, K, reinterpret_cast<int8_t*>(m->dW + P.w[which]) + (size_t)row0 * P.ldw[which], P.ldw[which],
                                    reinterpret_cast<float*>(m->dW + P.sw[which]) + row0, s);
      else
        e = ff::launch_cast_f16(stage, N, K, reinterpret_cast<__half*>(m->dW + P.w[which]) + (size_t)row0 * P.ldw[which],
                                P.ldw[which], s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(stage);
    if (e != cudaSuccess) return fail(FF_E_CUDA, std::string("weight packing: ") + cudaGetErrorString(e));
    return FF_OK;
  };
  ff_status st = FF_OK;
  switch (ki) {
    case 0: case 1: case 2:  // query / key / value weight -> section ki of the fused QKV
      if (!shape_is({D, H})) return bad_shape();
      if (m->hs == c.head_dim) {
        st = pack_weight(W_QKV, ki * D, D, H);
      } else {  // head h -> rows [ki Dq + h hs, + d); rows up to + hs stay zero (bind memset)
        const float* all = h_data;
        for (int h = 0; h < P.A && st == FF_OK; ++h) {
          h_data = all + (size_t)h * c.head_dim * H;
          st = pack_weight(W_QKV, ki * P.Dq + h * m->hs, c.head_dim, H);
        }
        h_data = all;
      }
      break;
    case 3: case 4: case 5:
      if (!shape_is({D})) return bad_shape();
      if (m->hs == c.head_dim) {
        st = copy_f32(P.bias[W_QKV] + (size_t)(ki - 3) * D * 4, D);
      } else {
        const float* all = h_data;
        for (int h = 0; h < P.A && st == FF_OK; ++h) {
          h_data = all + (size_t)h * c.head_dim;
          st = copy_f32(P.bias[W_QKV] + ((size_t)(ki - 3) * P.Dq + (size_t)h * m->hs) * 4, c.head_dim);
        }
        h_data = all;
      }
      break;
    case 6: if (!shape_is({H, D})) return bad_shape(); st = pack_weight(W_O, 0, H, D); break;
    case 7: if (!shape_is({H})) return bad_shape(); st = copy_f32(P.bias[W_O], H); break;
    case 8: if (!shape_is({H})) return bad_shape(); st = copy_f32(P.ln1g, H); break;
    case 9: if (!shape_is({H})) return bad_shape(); st = copy_f32(P.ln1b, H); break;
    case 10: if (!shape_is({F, H})) return bad_shape(); st = pack_weight(W_FFN1, 0, F, H); break;
    case 11: if (!shape_is({F})) return bad_shape(); st = copy_f32(P.bias[W_FFN1], F); break;
    case 12: if (!shape_is({H, F})) return bad_shape(); st = pack_weight(W_FFN2, 0, H, F); break;
    case 13: if (!shape_is({H})) return bad_shape(); st = copy_f32(P.bias[W_FFN2], H); break;
    case 14: if (!shape_is({H})) return bad_shape(); st = copy_f32(P.ln2g, H); break;
    default: if (!shape_is({H})) return bad_shape(); st = copy_f32(P.ln2b, H); break;
  }
  if (st != FF_OK) return st;
  P.loaded |= 1u << ki;
  return FF_OK;
}

ff_status ff_finalize(ff_model* m, void* stream) {
  if (!m) return fail(FF_E_INVALID, "null model");
  if (m->state != 1) return fail(FF_E_STATE, m->state == 0 ? "bind memory first" : "already finalized");
  std::string missing;
  for (int i = 0; i < 9; ++i)
    if (!(m->top_loaded & (1u << i))) missing += std::string(" ") + kTopKeys[i];
  for (size_t l = 0; l < m->L.size(); ++l)
    for (int i = 0; i < 16; ++i)
      if (!(m->L[l].loaded & (1u << i))) missing += " encoder.layer." + std::to_string(l) + "." + kLayerKeys[i];
  if (!missing.empty()) return fail(FF_E_STATE, "missing tensors:" + missing.substr(0, 2000));
  DeviceGuard dg(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // P' = P + T[0] in fp32 (R16)
  float* pos = m->w<float>(m->emb_pos);
  FF_CK(ff::launch_add_row(pos, m->cfg.max_positions, m->cfg.hidden, m->w<float>(m->emb_type), pos, s));
  FF_CK(cudaStreamSynchronize(s));
  FF_CK(ff::prepare_gemm_kernels());
  FF_CK(ff::prepare_attention_kernels());
  FF_CK(ff::prepare_attention_tc_kernel());
  FF_CK(ff::prepare_attention_long_kernel());
  FF_CK(ff::prepare_rr_kernels());
  FF_CK(ff::prepare_row_kernels());
  for (LayerPlan& P : m->L)  // zero-point corrections of the per-tensor u8 mode (DESIGN R22)
    if (P.dt == FF_I8)
      for (int i = 0; i < 4; ++i)
        FF_CK(ff::launch_weight_colsum(reinterpret_cast<const int8_t*>(m->dW + P.w[i]), P.ldw[i], P.N[i], P.K[i],
                                       reinterpret_cast<int*>(m->dW + P.cs[i]), s));
  FF_CK(cudaStreamSynchronize(s));
  {
    const char* err = nullptr;
    const bool ok = m->hm_rows > 0
                        ? ff::plan_attention_tc_hm(&m->tm_qkv, m->dWS + m->ws_qkv, 3 * (m->Dqmax / 64), m->hm_rows, &err)
                        : ff::plan_attention_tc(&m->tm_qkv, m->dWS + m->ws_qkv, m->cfg.max_tokens, m->ldqkv, &err);
    if (!ok)
      return fail(FF_E_CUDA, std::string("attention tensor map: ") + err);
  }
  ff_status st = build_gemm_plans(m);
  if (st != FF_OK) return st;
  m->state = 2;
  return FF_OK;
}

ff_status ff_encode(ff_model* m, const int32_t* d_token_ids, const int32_t* d_mask, int32_t batch, int32_t seq,
                    float* d_logits, void* stream) {
  ff_status st = check_call(m, batch, seq);
  if (st != FF_OK) return st;
  if (!d_token_ids || !d_mask || !d_logits) return fail(FF_E_INVALID, "null buffer");
  DeviceGuard dg(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!m->use_graphs || s == nullptr) return run_forward(m, d_token_ids, d_mask, batch, seq, d_logits, s, -1, nullptr);
  auto key = std::make_tuple((int)batch, (int)seq, (const void*)d_token_ids, (const void*)d_mask, (const void*)d_logits);
  auto it = m->graphs.find(key);
  if (it == m->graphs.end()) {
    if (m->graphs.size() >= ff_model::kMaxGraphs) {  // evict the least recently used graph
      auto lru = m->graphs.begin();
      for (auto g = m->graphs.begin(); g != m->graphs.end(); ++g)
        if (g->second.last_use < lru->second.last_use) lru = g;
      FF_CK(cudaStreamSynchronize(s));  // (rare) its last launch may still be in flight
      cudaGraphExecDestroy(lru->second.exec);
      m->graphs.erase(lru);
    }
    cudaGraph_t graph;
    FF_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    st = run_forward(m, d_token_ids, d_mask, batch, seq, d_logits, s, -1, nullptr);
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (st != FF_OK) return st;
    if (e != cudaSuccess) return fail(FF_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    cudaGraphExec_t exec;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(FF_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    it = m->graphs.emplace(key, ff_model::CachedGraph{exec, 0}).first;
  }
  it->second.last_use = ++m->graph_clock;
  FF_CK(cudaGraphLaunch(it->second.exec, s));
  return FF_OK;
}

// ff_encode_host / ff_encode_host_async: copies in, forward, copy out on the
// caller's stream (stream order makes the shared workspace ids / mask / logits
// buffers safe to reuse by the next call); the sync form then waits.
static ff_status encode_host_impl(ff_model* m, const int32_t* h_token_ids, const int32_t* h_mask, int32_t batch,
                                  int32_t seq, float* h_logits, void* stream, bool sync) {
  ff_status st = check_call(m, batch, seq);
  if (st != FF_OK) return st;
  if (!h_token_ids || !h_mask || !h_logits) return fail(FF_E_INVALID, "null buffer");
  DeviceGuard dg(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t n = (size_t)batch * seq;
  int32_t* ids = m->ws<int32_t>(m->ws_ids);
  int32_t* mask = m->ws<int32_t>(m->ws_mask);
  float* logits = m->ws<float>(m->ws_logits);
  FF_CK(cudaMemcpyAsync(ids, h_token_ids, n * 4, cudaMemcpyHostToDevice, s));
  FF_CK(cudaMemcpyAsync(mask, h_mask, n * 4, cudaMemcpyHostToDevice, s));
  st = ff_encode(m, ids, mask, batch, seq, logits, stream);
  if (st != FF_OK) return st;
  FF_CK(cudaMemcpyAsync(h_logits, logits, (size_t)batch * m->cfg.num_classes * 4, cudaMemcpyDeviceToHost, s));
  if (sync) FF_CK(cudaStreamSynchronize(s));
  return FF_OK;
}

ff_status ff_encode_host(ff_model* m, const int32_t* h_token_ids, const int32_t* h_mask, int32_t batch, int32_t seq,
                         float* h_logits, void* stream) {
  return encode_host_impl(m, h_token_ids, h_mask, batch, seq, h_logits, stream, true);
}

ff_status ff_encode_host_async(ff_model* m, const int32_t* h_token_ids, const int32_t* h_mask, int32_t batch,
                               int32_t seq, float* h_logits, void* stream) {
  ff_status st = check_call(m, batch, seq);
  if (st != FF_OK) return st;
  if (!h_token_ids || !h_mask || !h_logits) return fail(FF_E_INVALID, "null buffer");
  DeviceGuard dg(m->device);
  if (!m->io_stream) {
    FF_CK(cudaStreamCreateWithFlags(&m->io_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      FF_CK(cudaEventCreateWithFlags(&m->io_ready[i], cudaEventDisableTiming));
      FF_CK(cudaEventCreateWithFlags(&m->io_free[i], cudaEventDisableTiming));
      FF_CK(cudaEventRecord(m->io_free[i], static_cast<cudaStream_t>(stream)));
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int k = m->io_set;
  m->io_set ^= 1;
  const size_t n = (size_t)batch * seq;
  int32_t* ids = m->ws<int32_t>(k ? m->ws_ids2 : m->ws_ids);
  int32_t* mask = m->ws<int32_t>(k ? m->ws_mask2 : m->ws_mask);
  float* logits = m->ws<float>(k ? m->ws_logits2 : m->ws_logits);
  // inputs of set k on the copy stream, once the forward that last used set k is done
  FF_CK(cudaStreamWaitEvent(m->io_stream, m->io_free[k], 0));
  FF_CK(cudaMemcpyAsync(ids, h_token_ids, n * 4, cudaMemcpyHostToDevice, m->io_stream));
  FF_CK(cudaMemcpyAsync(mask, h_mask, n * 4, cudaMemcpyHostToDevice, m->io_stream));
  FF_CK(cudaEventRecord(m->io_ready[k], m->io_stream));
  FF_CK(cudaStreamWaitEvent(s, m->io_ready[k], 0));
  st = ff_encode(m, ids, mask, batch, seq, logits, stream);
  if (st != FF_OK) return st;
  FF_CK(cudaMemcpyAsync(h_logits, logits, (size_t)batch * m->cfg.num_classes * 4, cudaMemcpyDeviceToHost, s));
  FF_CK(cudaEventRecord(m->io_free[k], s));
  return FF_OK;
}

ff_status ff_check(ff_model* m, void* stream) {
  if (!m) return fail(FF_E_INVALID, "null model");
  if (m->state != 2) return fail(FF_E_STATE, "model not finalized");
  DeviceGuard dg(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FF_CK(cudaStreamSynchronize(s));
  int flag = 0;
  FF_CK(cudaMemcpy(&flag, m->dWS + m->ws_err, 4, cudaMemcpyDeviceToHost));
  if (flag) {
    FF_CK(cudaMemset(m->dWS + m->ws_err, 0, 4));
    std::string why;
    if (flag & 1) why += " token id outside [0, vocab)";
    if (flag & 2) why += " mask value not 0/1";
    if (flag & 4) why += " mask[b,0] != 1";
    return fail(FF_E_INPUT, "input error:" + why);
  }
  return FF_OK;
}

ff_status ff_set_option(ff_model* m, int32_t option, int64_t value) {
  if (!m) return fail(FF_E_INVALID, "null model");
  if (option == FF_OPT_GRAPHS) {
    m->use_graphs = value != 0;
    return FF_OK;
  }
  if (option == FF_OPT_PDL || option == FF_OPT_PDL_RR) {
    (option == FF_OPT_PDL ? m->launch.pdl : m->launch.pdl_rr) = value != 0;
    drop_graphs(m);  // captured launch attributes change
    return FF_OK;
  }
  if (option == FF_OPT_ACT_QUANT) {
    if (value != 0 && value != 1) return fail(FF_E_INVALID, "FF_OPT_ACT_QUANT must be 0 or 1");
    m->act_quant = (int)value;
    drop_graphs(m);
    return FF_OK;
  }
  if (option == FF_OPT_FUSED_EPILOGUES) {
    m->fused = value != 0 ? 7 : 0;
    drop_graphs(m);
    return FF_OK;
  }
  if (option == FF_OPT_FUSED_MASK) {
    if (value < -1 || value > 7) return fail(FF_E_INVALID, "FF_OPT_FUSED_MASK must be -1 (auto) or 0..7");
    m->fused = (int)value;
    drop_graphs(m);
    return FF_OK;
  }
  if (option == FF_OPT_ATTN_TC) {
    m->attn_tc = value != 0;
    drop_graphs(m);
    return FF_OK;
  }
  if (option == FF_OPT_CTA_PAIRS) {
    m->pair_mode = value != 0 ? -1 : 0;
    drop_graphs(m);  // captured launch configs change
    return FF_OK;
  }
  if (option == FF_OPT_CLS_LAST_LAYER) {
    m->cls_last = value != 0;
    drop_graphs(m);
    return FF_OK;
  }
  if (option == FF_OPT_ROW_DIRS) {
    if (value < 0 || value > 31) return fail(FF_E_INVALID, "FF_OPT_ROW_DIRS must be 0..31");
    m->row_dirs = (int)value;
    drop_graphs(m);
    return FF_OK;
  }
  return fail(FF_E_INVALID, "unknown option");
}

ff_status ff_get_option(const ff_model* m, int32_t option, int64_t* value) {
  if (!m || !value) return fail(FF_E_INVALID, "null argument");
  switch (option) {
    case FF_OPT_GRAPHS: *value = m->use_graphs ? 1 : 0; return FF_OK;
    case FF_OPT_CTA_PAIRS: *value = m->pair_mode == 0 ? 0 : 1; return FF_OK;
    case FF_OPT_ATTN_TC: *value = m->attn_tc ? 1 : 0; return FF_OK;
    case FF_OPT_FUSED_EPILOGUES: *value = m->fused != 0 ? 1 : 0; return FF_OK;
    case FF_OPT_PDL: *value = m->launch.pdl ? 1 : 0; return FF_OK;
    case FF_OPT_ACT_QUANT: *value = m->act_quant; return FF_OK;
    case FF_OPT_FUSED_MASK: *value = m->fused; return FF_OK;
    case FF_OPT_PDL_RR: *value = m->launch.pdl_rr ? 1 : 0; return FF_OK;
    case FF_OPT_CLS_LAST_LAYER: *value = m->cls_last ? 1 : 0; return FF_OK;
    case FF_OPT_ROW_DIRS: *value = m->row_dirs; return FF_OK;
    default: return fail(FF_E_INVALID, "unknown option");
  }
}

void ff_model_destroy(ff_model* m) {
  if (!m) return;
  drop_graphs(m);
  if (m->io_stream) {
    cudaStreamSynchronize(m->io_stream);
    cudaStreamDestroy(m->io_stream);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(m->io_ready[i]);
      cudaEventDestroy(m->io_free[i]);
    }
  }
  delete m;
}

ff_status ff_launch_count(const ff_model* m, int32_t batch, int32_t seq, int32_t* count) {
  if (!m || !count) return fail(FF_E_INVALID, "null argument");
  int n = 3;  // embed_ln + pooler + classifier
  for (const LayerPlan& P : m->L) {
    const bool q = P.dt == FF_I8;
    if (m->act_quant == 1) {  // per-tensor u8: 4 GEMMs + attention + 2 add_ln, 2 quant kernels per int8 GEMM
      n += 7 + (q ? 8 : 0);
      continue;
    }
    const int fm = fused_mask(m, P);
    const bool fln = (fm & 1) && P.rr_ok[0], fq = (fm & 2) && q && P.rr_ok[1];
    const bool fln2 = (fm & 4) && P.rr_ok[0];
    n += 2;                              // QKV GEMM + attention
    n += (q && !attention_fuses_quant(m, P, batch, seq)) ? 1 : 0;  // ctx requant
    n += fln ? 1 : 2;                    // out-proj (+ add_ln1)
    n += fq ? 1 : (q ? 2 : 1);           // FFN1 (+ requant)
    n += fln2 ? 1 : 2;                   // FFN2 (+ add_ln2)
  }
  *count = n;
  return FF_OK;
}

ff_status ff_encode_trace(ff_model* m, const int32_t* d_token_ids, const int32_t* d_mask, int32_t batch, int32_t seq,
                          float* d_logits, int32_t layer, void* const* d_dump, void* stream) {
  ff_status st = check_call(m, batch, seq);
  if (st != FF_OK) return st;
  if (!d_dump || layer < 0 || layer >= m->cfg.num_layers) return fail(FF_E_INVALID, "bad trace layer / dump");
  DeviceGuard dg(m->device);
  return run_forward(m, d_token_ids, d_mask, batch, seq, d_logits, static_cast<cudaStream_t>(stream), layer, d_dump);
}

ff_status ff_profile(ff_model* m, const int32_t* d_token_ids, const int32_t* d_mask, int32_t batch, int32_t seq,
                     float* d_logits, int32_t capacity, int32_t* kinds, float* ms, int32_t* count, void* stream) {
  ff_status st = check_call(m, batch, seq);
  if (st != FF_OK) return st;
  if (!kinds || !ms || !count) return fail(FF_E_INVALID, "null output");
  DeviceGuard dg(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Prof prof;
  st = run_forward(m, d_token_ids, d_mask, batch, seq, d_logits, s, -1, nullptr, &prof);
  if (st != FF_OK) return st;
  FF_CK(cudaStreamSynchronize(s));
  const int n = (int)prof.kind.size();
  if (n > capacity) return fail(FF_E_NOMEM, "profile capacity too small");
  for (int i = 0; i < n; ++i) {
    kinds[i] = prof.kind[i];
    FF_CK(cudaEventElapsedTime(&ms[i], prof.ev[2 * i], prof.ev[2 * i + 1]));
  }
  *count = n;
  return FF_OK;
}

ff_status ff_debug_gemm(int32_t dtype, const void* d_A, int32_t lda, const void* d_W, int32_t ldw, int32_t M,
                        int32_t N, int32_t K, int32_t out_mode, void* d_C, int32_t ldc, const float* d_bias,
                        const float* d_sx, const float* d_sw, int32_t act, void* stream) {
  if (M < 1 || N < 1 || K < 1 || !d_A || !d_W || !d_C) return fail(FF_E_INVALID, "bad gemm args");
  if (dtype == FF_I8 && out_mode == 1 && (!d_sx || !d_sw)) return fail(FF_E_INVALID, "i8 epilogue needs scales");
  static bool prepared = false;
  if (!prepared) {
    FF_CK(ff::prepare_gemm_kernels());
    prepared = true;
  }
  const int force = (out_mode >> 4) & 3;  // bit 4: force CTA pairs, bit 5: force single CTAs
  const int noload = (out_mode >> 6) & 1;  // bit 6: MMA-rate probe (operand loads skipped, results garbage)
  out_mode &= 15;
  ff::GemmPlan g;
  const char* err = nullptr;
  if (!ff::plan_gemm(&g, dtype == FF_I8, d_A, M, lda, d_W, ldw, N, K, &err))
    return fail(FF_E_INVALID, std::string("gemm plan: ") + err);
  if (force == 1 || force == 2) {
    g.force_pair = force == 1 ? 1 : 0;
    ff::plan_gemm_set_m(&g, M);
  }
  if (out_mode == 1) {
    if (!ff::plan_gemm_output(&g, d_C, ldc, &err)) return fail(FF_E_INVALID, std::string("gemm output: ") + err);
  } else {
    g.p.out = d_C;
    g.p.ldo = ldc;
  }
  g.p.out_mode = out_mode;
  g.p.bias = d_bias;
  g.p.row_scale = d_sx;
  g.p.col_scale = d_sw;
  g.p.act = act;
  g.p.trace = g_debug_trace_which == 0 ? g_debug_trace : nullptr;
  g.p.dbg_noload = noload;
  FF_CK(ff::launch_gemm(g, static_cast<cudaStream_t>(stream)));
  return FF_OK;
}

ff_status ff_debug_set_trace(uint64_t* d_trace, int32_t which) {
  g_debug_trace = reinterpret_cast<unsigned long long*>(d_trace);
  g_debug_trace_which = which;
  return FF_OK;
}

ff_status ff_debug_quant_rows(const void* d_x16, int32_t M, int32_t K, int32_t ldx, int8_t* d_q, int32_t ldq,
                              float* d_s, void* stream) {
  if (M < 1 || K < 1 || !d_x16 || !d_q || !d_s) return fail(FF_E_INVALID, "bad quant args");
  FF_CK(ff::launch_quant_rows(static_cast<const __half*>(d_x16), ldx, M, K, d_q, ldq, d_s,
                              static_cast<cudaStream_t>(stream)));
  return FF_OK;
}

ff_status ff_debug_attention(const void* d_qkv16, const int32_t* d_mask, int32_t B, int32_t S, int32_t A, int32_t d,
                             void* d_ctx16, int32_t impl, void* stream) {
  if (B < 1 || S < 1 || A < 1 || d < 2 || d > 128 || (d & 1)) return fail(FF_E_INVALID, "bad attention args");
  if (ff::attention_smem_bytes(S, d) > 227 * 1024) return fail(FF_E_UNSUPPORTED, "seq too long");
  static bool prepared = false;
  if (!prepared) {
    FF_CK(ff::prepare_attention_kernels());
    FF_CK(ff::prepare_attention_tc_kernel());
    FF_CK(ff::prepare_attention_long_kernel());
    prepared = true;
  }
  const int mode = impl;  // 0 auto (tcgen05 where supported), 1 mma.sync kernel, 2 tcgen05 (must be supported)
  const bool aligned = (reinterpret_cast<uintptr_t>(d_qkv16) & 15) == 0;
  const bool tc = mode != 1 && aligned && ff::attention_tc_supported(S, d, d, 3 * A * d, A * d);
  const bool tcl = mode != 1 && aligned && !tc && ff::attention_long_supported(S, d, 3 * A * d, A * d);
  if (mode == 2 && !tc && !tcl)
    return fail(FF_E_UNSUPPORTED,
                "tcgen05 attention needs head_dim 64 (S <= 512) or an even head_dim <= 32 (S <= 128)");
  if (tc || tcl) {
    ff::AttnTCPlan map;
    const char* err = nullptr;
    if (!ff::plan_attention_tc(&map, d_qkv16, B * S, 3 * A * d, &err))
      return fail(FF_E_INVALID, std::string("attention tensor map: ") + err);
    if (tc)
      FF_CK(ff::launch_attention_tc(map, d_mask, B, S, A, d, d, static_cast<__half*>(d_ctx16), A * d, nullptr, 0,
                                    nullptr, static_cast<cudaStream_t>(stream)));
    else
      FF_CK(ff::launch_attention_long(map, d_mask, B, S, A, static_cast<__half*>(d_ctx16), A * d,
                                      static_cast<cudaStream_t>(stream),
                                      g_debug_trace_which == 4 ? g_debug_trace : nullptr));
    return FF_OK;
  }
  FF_CK(ff::launch_attention(static_cast<const __half*>(d_qkv16), 3 * A * d, d_mask, B, S, A, d, d, 0,
                             static_cast<__half*>(d_ctx16), A * d, static_cast<cudaStream_t>(stream)));
  return FF_OK;
}

ff_status ff_debug_attention_q8(const void* d_qkv16, const int32_t* d_mask, int32_t B, int32_t S, int32_t A,
                                int32_t d, void* d_ctx16, int8_t* d_ctxq, float* d_ctxs, uint64_t* d_trace,
                                void* stream) {
  if (B < 1 || S < 1 || A < 1 || !d_ctxq || !d_ctxs) return fail(FF_E_INVALID, "bad attention args");
  if (!ff::attention_tc_supported(S, d, d, 3 * A * d, A * d) || !ff::attention_tc_fuses_quant(A, d) ||
      (reinterpret_cast<uintptr_t>(d_qkv16) & 15) != 0 || (A * d) % 16 != 0)
    return fail(FF_E_UNSUPPORTED, "fused attention + requant needs head_dim 64 (A <= 8) or an even head_dim <= 32 (A <= 16), S <= 128");
  static bool prepared = false;
  if (!prepared) {
    FF_CK(ff::prepare_attention_tc_kernel());
    FF_CK(ff::prepare_attention_long_kernel());
    prepared = true;
  }
  ff::AttnTCPlan map;
  const char* err = nullptr;
  if (!ff::plan_attention_tc(&map, d_qkv16, B * S, 3 * A * d, &err))
    return fail(FF_E_INVALID, std::string("attention tensor map: ") + err);
  FF_CK(ff::launch_attention_tc(map, d_mask, B, S, A, d, d, static_cast<__half*>(d_ctx16), A * d, d_ctxq, A * d, d_ctxs,
                                static_cast<cudaStream_t>(stream),
                                reinterpret_cast<unsigned long long*>(d_trace)));
  return FF_OK;
}

}  // extern "C"
