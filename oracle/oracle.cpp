// oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY (never on the product path).
//
// A plain, slow, obviously-correct CPU implementation of the FastFormers
// (arXiv 2010.13382) inference hot path: the batched forward pass of a
// distilled, structurally pruned post-LN BERT/RoBERTa encoder classifier whose
// layers each have their own surviving head count A'_l, FFN width F'_l and
// GEMM dtype (fp16 or dynamically quantized int8).
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
// --impl reference) may load this library.  It shares NO code with the CUDA
// library under paper_2010_13382_b200/csrc (no headers, helpers or tables).
//
// Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
// "DESIGN R<k>" = the k-th reading listed in DESIGN.md section "Readings".
//
// Two modes (DESIGN R1..R21):
//   mode 0 "ref64": the textbook definition of the (possibly pruned) model in
//     fp64 with no rounding and no quantization.  Pinned against HuggingFace
//     BertForSequenceClassification (fp64, eager) in tests/test_oracle.py.
//   mode 1 "emu":   the approximation the paper describes, step by step, with
//     the rounding points the GPU path uses: every stored activation is fp16
//     (R16 = round-to-nearest-even), fp16 layers multiply R16(W) with fp32
//     accumulation, int8 layers quantize activations per row and
//     weights per output channel, symmetric s8, RNE (DESIGN R6-R8,R13),
//     Q.K^T and P.V stay in floating point ("we do not use 8-bit matrix
//     product for the Q, K inner product").
//   Reductions accumulate in fp64 and are rounded to fp32 where the GPU holds
//   fp32 (acc32=1 switches to sequential fp32 accumulation; used only to
//   calibrate the drift bound of DESIGN "Tolerances").
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fPIC -shared (no fast-math).

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

typedef _Float16 half_t;

namespace {

// ---------------------------------------------------------------- rounding
// R16: fp32 -> fp16, round-to-nearest-even (GCC _Float16 conversion is IEEE).
inline float r16(float x) { return (float)(half_t)x; }
// Round an fp64 result to the fp32 the GPU would hold, then to fp16.
inline float r16_of(double x) { return r16((float)x); }

enum { ACT_GELU = 0, ACT_RELU = 1, ACT_GELU_TANH = 2 };
enum { DT_F16 = 0, DT_I8 = 1 };
enum { MODE_REF64 = 0, MODE_EMU = 1 };

// Activation (P:135 GELU->ReLU swap; S:64 tanh-GELU; DESIGN R2), in fp64.
double act64(double y, int act) {
  if (act == ACT_RELU) return y > 0.0 ? y : 0.0;
  if (act == ACT_GELU_TANH)
    return 0.5 * y * (1.0 + std::tanh(std::sqrt(2.0 / M_PI) * (y + 0.044715 * y * y * y)));
  return 0.5 * y * (1.0 + std::erf(y / std::sqrt(2.0)));
}

// Q8row (DESIGN R6-R8): per-row symmetric s8, scale = amax/127 in fp32 IEEE
// division (1.0 for an all-zero row), q = clamp(RNE(x / s), -127, 127).
void q8row(const float* x, int K, int8_t* q, float* s_out) {
  float amax = 0.0f;
  for (int k = 0; k < K; ++k) amax = std::fmax(amax, std::fabs(x[k]));
  float s = (amax == 0.0f) ? 1.0f : amax / 127.0f;
  for (int k = 0; k < K; ++k) {
    float v = std::nearbyint(x[k] / s);  // default rounding mode = RNE
    if (v > 127.0f) v = 127.0f;
    if (v < -127.0f) v = -127.0f;
    q[k] = (int8_t)v;
  }
  *s_out = s;
}

// Q8tensor (DESIGN R22; "the quantization range for the input matrix
// is selected for entire input tensor", dynamic u8 quantization with a zero
// point as in the FBGEMM / PyTorch dynamic-quantization recipe the paper
// cites): over the whole [M, K] tensor,
//   lo = min(0, min x), hi = max(0, max x), scale = (hi - lo) / 255 (fp32
//   IEEE; 1.0 for an all-zero tensor), zp = clamp(RNE(-lo / scale), 0, 255),
//   q = clamp(RNE(x / scale) + zp, 0, 255)  (u8).
void q8tensor(const float* x, size_t n, uint8_t* q, float* scale_out, int* zp_out) {
  float lo = 0.0f, hi = 0.0f;
  for (size_t i = 0; i < n; ++i) {
    lo = std::fmin(lo, x[i]);
    hi = std::fmax(hi, x[i]);
  }
  float s = (hi - lo) / 255.0f;
  if (s == 0.0f) s = 1.0f;
  float z = std::nearbyint(-lo / s);
  if (z < 0.0f) z = 0.0f;
  if (z > 255.0f) z = 255.0f;
  const int zp = (int)z;
  for (size_t i = 0; i < n; ++i) {
    float v = std::nearbyint(x[i] / s) + (float)zp;
    if (v < 0.0f) v = 0.0f;
    if (v > 255.0f) v = 255.0f;
    q[i] = (uint8_t)v;
  }
  *scale_out = s;
  *zp_out = zp;
}

// Per-output-channel weight quantization ("quantization range ... for
// each column separately"; DESIGN R7): W is [N, K] (PyTorch
// [out, in]); channel n = row n.
void quant_weight(const float* W, int N, int K, int8_t* q, float* s) {
  for (int n = 0; n < N; ++n) q8row(W + (size_t)n * K, K, q + (size_t)n * K, s + n);
}

struct Layer {
  int A = 0, F = 0, dt = DT_F16;
  std::map<std::string, std::vector<float>> t;  // fp32 host weights by short name
  // prepared (emu) weights, built by finalize():
  std::vector<float> w16[4];          // R16(W) for f16 layers  [qkv, o, ffn1, ffn2]
  std::vector<int8_t> wq[4];          // s8 weights for i8 layers
  std::vector<float> sw[4];           // per-output-channel scales
  std::vector<float> wqkv, bqkv;      // concatenated [Q|K|V] rows (S:236 fused QKV)
};

struct Model {
  int L, H, d, V, P, C, act;
  int act_quant = 0;  // int8 activation quantizer: 0 Q8row (per row), 1 Q8tensor (per tensor, u8 + zero point)
  float eps;
  std::vector<Layer> layers;
  std::map<std::string, std::vector<float>> t;  // non-layer tensors
  bool ready = false;
};

// --------------------------------------------------------------- weights IO
bool strip_prefix(std::string& s, const char* p) {
  size_t n = std::strlen(p);
  if (s.compare(0, n, p) == 0) { s = s.substr(n); return true; }
  return false;
}

// Expected shape of a tensor, by HF name (SURVEY 8(b) weight-name table).
bool expected_shape(const Model& m, const std::string& name, int* layer, std::string* key,
                    std::vector<int64_t>* shape) {
  const int H = m.H, d = m.d;
  *layer = -1;
  if (name == "embeddings.word_embeddings.weight") { *key = name; *shape = {m.V, H}; return true; }
  if (name == "embeddings.position_embeddings.weight") { *key = name; *shape = {m.P, H}; return true; }
  if (name == "embeddings.token_type_embeddings.weight") { *key = name; *shape = {-1, H}; return true; }
  if (name == "embeddings.LayerNorm.weight" || name == "embeddings.LayerNorm.bias") { *key = name; *shape = {H}; return true; }
  if (name == "pooler.dense.weight") { *key = name; *shape = {H, H}; return true; }
  if (name == "pooler.dense.bias") { *key = name; *shape = {H}; return true; }
  if (name == "classifier.weight") { *key = name; *shape = {m.C, H}; return true; }
  if (name == "classifier.bias") { *key = name; *shape = {m.C}; return true; }
  std::string s = name;
  if (!strip_prefix(s, "encoder.layer.")) return false;
  size_t dot = s.find('.');
  if (dot == std::string::npos) return false;
  int l = std::atoi(s.substr(0, dot).c_str());
  if (l < 0 || l >= m.L) return false;
  std::string k = s.substr(dot + 1);
  const Layer& ly = m.layers[l];
  const int D = ly.A * d, F = ly.F;
  *layer = l;
  *key = k;
  if (k == "attention.self.query.weight" || k == "attention.self.key.weight" || k == "attention.self.value.weight") { *shape = {D, H}; return true; }
  if (k == "attention.self.query.bias" || k == "attention.self.key.bias" || k == "attention.self.value.bias") { *shape = {D}; return true; }
  if (k == "attention.output.dense.weight") { *shape = {H, D}; return true; }
  if (k == "attention.output.dense.bias" || k == "attention.output.LayerNorm.weight" || k == "attention.output.LayerNorm.bias") { *shape = {H}; return true; }
  if (k == "intermediate.dense.weight") { *shape = {F, H}; return true; }
  if (k == "intermediate.dense.bias") { *shape = {F}; return true; }
  if (k == "output.dense.weight") { *shape = {H, F}; return true; }
  if (k == "output.dense.bias" || k == "output.LayerNorm.weight" || k == "output.LayerNorm.bias") { *shape = {H}; return true; }
  return false;
}

const char* kLayerKeys[] = {
    "attention.self.query.weight", "attention.self.query.bias", "attention.self.key.weight",
    "attention.self.key.bias", "attention.self.value.weight", "attention.self.value.bias",
    "attention.output.dense.weight", "attention.output.dense.bias",
    "attention.output.LayerNorm.weight", "attention.output.LayerNorm.bias",
    "intermediate.dense.weight", "intermediate.dense.bias", "output.dense.weight",
    "output.dense.bias", "output.LayerNorm.weight", "output.LayerNorm.bias"};
const char* kTopKeys[] = {"embeddings.word_embeddings.weight", "embeddings.position_embeddings.weight",
                          "embeddings.token_type_embeddings.weight", "embeddings.LayerNorm.weight",
                          "embeddings.LayerNorm.bias", "pooler.dense.weight", "pooler.dense.bias",
                          "classifier.weight", "classifier.bias"};

// ------------------------------------------------------------ the math steps
// Linear layer y = x W^T + b for M rows, in the requested mode:
//   ref64: fp64 throughout.
//   emu f16: y32 = fp32(sum_k x16*R16(W)) + b   (fp32 accumulate)
//   emu i8 : acc = sum_k Xq*Wq (int32, exact); y32 = fma(float(acc), sx*sw, b)
//            (DESIGN R13; P:104 dynamic per-call activation range, per-row here)
// x: [M, K] (fp16-representable in emu mode).  y: [M, N] fp32/fp64 pre-activation.
void linear(const Model& mdl, const Layer& ly, int which, const std::vector<float>& Wf,
            const std::vector<float>& b, int N, int K, const double* x64, const float* x16,
            int M, int mode, int acc32, double* y64, float* y32) {
  if (mode == MODE_REF64) {
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double acc = 0.0;
        for (int k = 0; k < K; ++k) acc += x64[(size_t)m * K + k] * (double)Wf[(size_t)n * K + k];
        y64[(size_t)m * N + n] = acc + (double)b[n];
      }
    return;
  }
  if (ly.dt == DT_F16) {
    const std::vector<float>& W16 = ly.w16[which];
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        float acc32f;
        if (acc32) {
          float a = 0.0f;
          for (int k = 0; k < K; ++k) a += x16[(size_t)m * K + k] * W16[(size_t)n * K + k];
          acc32f = a;
        } else {
          double a = 0.0;
          for (int k = 0; k < K; ++k) a += (double)x16[(size_t)m * K + k] * (double)W16[(size_t)n * K + k];
          acc32f = (float)a;
        }
        y32[(size_t)m * N + n] = acc32f + b[n];
      }
    return;
  }
  const std::vector<int8_t>& Wq = ly.wq[which];
  const std::vector<float>& sw = ly.sw[which];
  if (mdl.act_quant == 1) {
    // per-tensor u8 activations with zero point: acc = sum_k q * w (int32,
    // exact), corrected by zp * sum_k w[n][k] (exact), then dequantized
    std::vector<uint8_t> xq((size_t)M * K);
    float st;
    int zp;
    q8tensor(x16, (size_t)M * K, xq.data(), &st, &zp);
    for (int n = 0; n < N; ++n) {
      int32_t colsum = 0;
      for (int k = 0; k < K; ++k) colsum += (int32_t)Wq[(size_t)n * K + k];
      for (int m = 0; m < M; ++m) {
        int32_t acc = 0;
        for (int k = 0; k < K; ++k) acc += (int32_t)xq[(size_t)m * K + k] * (int32_t)Wq[(size_t)n * K + k];
        const int32_t corr = acc - zp * colsum;
        y32[(size_t)m * N + n] = std::fma((float)corr, st * sw[n], b[n]);
      }
    }
    return;
  }
  // int8 (per-row activation scale, per-channel weight scale)
  std::vector<int8_t> xq((size_t)M * K);
  std::vector<float> sx(M);
  for (int m = 0; m < M; ++m) q8row(x16 + (size_t)m * K, K, &xq[(size_t)m * K], &sx[m]);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      int32_t acc = 0;
      for (int k = 0; k < K; ++k) acc += (int32_t)xq[(size_t)m * K + k] * (int32_t)Wq[(size_t)n * K + k];
      float scale = sx[m] * sw[n];
      y32[(size_t)m * N + n] = std::fma((float)acc, scale, b[n]);
    }
}

// LayerNorm over H of (a + r) (post-LN).  Two-pass mean and
// variance, biased variance, eps inside the sqrt (BERT convention, DESIGN R3).
// emu: inputs are fp16 values, the sum a+r is formed in fp32, the statistics
// in fp64, and the output is rounded to fp32 then fp16.
void layer_norm64(const double* x, int H, const float* g, const float* b, float eps, double* y) {
  double mu = 0.0;
  for (int j = 0; j < H; ++j) mu += x[j];
  mu /= H;
  double var = 0.0;
  for (int j = 0; j < H; ++j) var += (x[j] - mu) * (x[j] - mu);
  var /= H;
  double rstd = 1.0 / std::sqrt(var + (double)eps);
  for (int j = 0; j < H; ++j) y[j] = (x[j] - mu) * rstd * (double)g[j] + (double)b[j];
}

void layer_norm32(const float* x, int H, const float* g, const float* b, float eps, int acc32, float* y16) {
  if (acc32) {
    float mu = 0.0f;
    for (int j = 0; j < H; ++j) mu += x[j];
    mu /= H;
    float var = 0.0f;
    for (int j = 0; j < H; ++j) var += (x[j] - mu) * (x[j] - mu);
    var /= H;
    float rstd = 1.0f / std::sqrt(var + eps);
    for (int j = 0; j < H; ++j) y16[j] = r16((x[j] - mu) * rstd * g[j] + b[j]);
    return;
  }
  std::vector<double> xd(H), yd(H);
  for (int j = 0; j < H; ++j) xd[j] = x[j];
  layer_norm64(xd.data(), H, g, b, eps, yd.data());
  for (int j = 0; j < H; ++j) y16[j] = r16_of(yd[j]);
}

// Masked scaled-dot-product attention for one layer (DESIGN R4, R9, R10).
// qkv: [B*S, 3D] rows = tokens, columns [Q heads | K heads | V heads].
// ctx: [B*S, D], heads concatenated in head order.
// Keys with mask[b, j] == 0 are excluded from the softmax.
// emu: s = fp32(q.k) * fp32(1/sqrt(d)); p = e / l with e = exp(s - max),
//      l = sum(e) (normalized rounding point, DESIGN R9); P16 = R16(p);
//      ctx = R16(fp32(sum_j P16 * v_j)).
template <typename T>
void attention(const T* qkv, const int* mask, int B, int S, int A, int d, int mode, int acc32, T* ctx) {
  const int D = A * d, ld = 3 * D;
  const float cd32 = (float)(1.0 / std::sqrt((double)d));
  const double cd64 = 1.0 / std::sqrt((double)d);
  std::vector<double> s64(S), p64(S);
  std::vector<float> s32(S), p16(S);
  for (int b = 0; b < B; ++b)
    for (int h = 0; h < A; ++h)
      for (int i = 0; i < S; ++i) {
        const T* q = qkv + (size_t)(b * S + i) * ld + h * d;
        if (mode == MODE_REF64) {
          double mx = -INFINITY;
          for (int j = 0; j < S; ++j) {
            if (!mask[b * S + j]) continue;
            const T* k = qkv + (size_t)(b * S + j) * ld + D + h * d;
            double a = 0.0;
            for (int c = 0; c < d; ++c) a += (double)q[c] * (double)k[c];
            s64[j] = a * cd64;
            if (s64[j] > mx) mx = s64[j];
          }
          double l = 0.0;
          for (int j = 0; j < S; ++j) {
            if (!mask[b * S + j]) continue;
            p64[j] = std::exp(s64[j] - mx);
            l += p64[j];
          }
          for (int c = 0; c < d; ++c) {
            double a = 0.0;
            for (int j = 0; j < S; ++j) {
              if (!mask[b * S + j]) continue;
              const T* v = qkv + (size_t)(b * S + j) * ld + 2 * D + h * d;
              a += (p64[j] / l) * (double)v[c];
            }
            ctx[(size_t)(b * S + i) * D + h * d + c] = (T)a;
          }
          continue;
        }
        float mx = -INFINITY;
        for (int j = 0; j < S; ++j) {
          if (!mask[b * S + j]) continue;
          const T* k = qkv + (size_t)(b * S + j) * ld + D + h * d;
          float dot;
          if (acc32) {
            float a = 0.0f;
            for (int c = 0; c < d; ++c) a += (float)q[c] * (float)k[c];
            dot = a;
          } else {
            double a = 0.0;
            for (int c = 0; c < d; ++c) a += (double)q[c] * (double)k[c];
            dot = (float)a;
          }
          s32[j] = dot * cd32;
          if (s32[j] > mx) mx = s32[j];
        }
        float l;
        {
          double l64 = 0.0;
          float l32 = 0.0f;
          for (int j = 0; j < S; ++j) {
            if (!mask[b * S + j]) continue;
            float e = (float)std::exp((double)(s32[j] - mx));
            p16[j] = e;
            l64 += (double)e;
            l32 += e;
          }
          l = acc32 ? l32 : (float)l64;
        }
        for (int j = 0; j < S; ++j)
          if (mask[b * S + j]) p16[j] = r16(p16[j] / l);
        for (int c = 0; c < d; ++c) {
          double a = 0.0;
          float a32 = 0.0f;
          for (int j = 0; j < S; ++j) {
            if (!mask[b * S + j]) continue;
            const T* v = qkv + (size_t)(b * S + j) * ld + 2 * D + h * d;
            a += (double)p16[j] * (double)v[c];
            a32 += p16[j] * (float)v[c];
          }
          ctx[(size_t)(b * S + i) * D + h * d + c] = (T)r16(acc32 ? a32 : (float)a);
        }
      }
}

// ----------------------------------------------------------------- stages
// Stage ids for or_stage (lockstep protocol).
enum { ST_QKV = 0, ST_ATTN = 1, ST_OPROJ = 2, ST_LN1 = 3, ST_FFN1 = 4, ST_FFN2 = 5, ST_LN2 = 6 };

const std::vector<float>& T_(const Layer& ly, const char* k) { return ly.t.at(k); }

// One emu stage of layer l.  in_a/in_b/out are fp16 values stored as float.
int run_stage(const Model& m, int l, int stage, const float* in_a, const float* in_b, const int* mask,
              int B, int S, int acc32, float* out) {
  const Layer& ly = m.layers[l];
  const int H = m.H, D = ly.A * m.d, F = ly.F, M = B * S;
  switch (stage) {
    case ST_QKV: {
      std::vector<float> y((size_t)M * 3 * D);
      linear(m, ly, 0, ly.wqkv, ly.bqkv, 3 * D, H, nullptr, in_a, M, MODE_EMU, acc32, nullptr, y.data());
      for (size_t i = 0; i < y.size(); ++i) out[i] = r16(y[i]);
      return 0;
    }
    case ST_ATTN:
      attention<float>(in_a, mask, B, S, ly.A, m.d, MODE_EMU, acc32, out);
      return 0;
    case ST_OPROJ: {
      std::vector<float> y((size_t)M * H);
      linear(m, ly, 1, T_(ly, "attention.output.dense.weight"), T_(ly, "attention.output.dense.bias"), H, D,
             nullptr, in_a, M, MODE_EMU, acc32, nullptr, y.data());
      for (size_t i = 0; i < y.size(); ++i) out[i] = r16(y[i]);
      return 0;
    }
    case ST_LN1:
    case ST_LN2: {
      const char* g = stage == ST_LN1 ? "attention.output.LayerNorm.weight" : "output.LayerNorm.weight";
      const char* bb = stage == ST_LN1 ? "attention.output.LayerNorm.bias" : "output.LayerNorm.bias";
      std::vector<float> x(H);
      for (int r = 0; r < M; ++r) {
        for (int j = 0; j < H; ++j) x[j] = in_a[(size_t)r * H + j] + in_b[(size_t)r * H + j];
        layer_norm32(x.data(), H, T_(ly, g).data(), T_(ly, bb).data(), m.eps, acc32, out + (size_t)r * H);
      }
      return 0;
    }
    case ST_FFN1: {
      std::vector<float> y((size_t)M * F);
      linear(m, ly, 2, T_(ly, "intermediate.dense.weight"), T_(ly, "intermediate.dense.bias"), F, H, nullptr,
             in_a, M, MODE_EMU, acc32, nullptr, y.data());
      for (size_t i = 0; i < y.size(); ++i) out[i] = r16_of(act64((double)y[i], m.act));
      return 0;
    }
    case ST_FFN2: {
      std::vector<float> y((size_t)M * H);
      linear(m, ly, 3, T_(ly, "output.dense.weight"), T_(ly, "output.dense.bias"), H, F, nullptr, in_a, M,
             MODE_EMU, acc32, nullptr, y.data());
      for (size_t i = 0; i < y.size(); ++i) out[i] = r16(y[i]);
      return 0;
    }
  }
  return 1;
}

// Embedding + LN (BERT convention S:234; DESIGN R16): position
// ids 0..S-1, token type 0 folded into the position table in fp32.
void embed(const Model& m, const int* ids, int M, int S, int mode, int acc32, double* x64, float* x16) {
  const int H = m.H;
  const std::vector<float>& E = m.t.at("embeddings.word_embeddings.weight");
  const std::vector<float>& Pp = m.t.at("embeddings.position_embeddings.weight");
  const std::vector<float>& T = m.t.at("embeddings.token_type_embeddings.weight");
  const std::vector<float>& g = m.t.at("embeddings.LayerNorm.weight");
  const std::vector<float>& bb = m.t.at("embeddings.LayerNorm.bias");
  std::vector<double> e64(H);
  std::vector<float> e32(H);
  for (int r = 0; r < M; ++r) {
    const int id = ids[r], pos = r % S;
    for (int j = 0; j < H; ++j) {
      if (mode == MODE_REF64) {
        e64[j] = (double)E[(size_t)id * H + j] + (double)Pp[(size_t)pos * H + j] + (double)T[j];
      } else {
        float pprime = Pp[(size_t)pos * H + j] + T[j];  // P' = P + T[0] in fp32
        e32[j] = E[(size_t)id * H + j] + pprime;
      }
    }
    if (mode == MODE_REF64)
      layer_norm64(e64.data(), H, g.data(), bb.data(), m.eps, x64 + (size_t)r * H);
    else
      layer_norm32(e32.data(), H, g.data(), bb.data(), m.eps, acc32, x16 + (size_t)r * H);
  }
}

// Pooler + classifier (BERT convention S:237; DESIGN R15: fp32 output, fp64
// accumulation): pooled = tanh(Wp x0 + bp); logits = Wc pooled + bc.
void head(const Model& m, const double* x0, int B, float* logits, double* logits64) {
  const int H = m.H, C = m.C;
  const std::vector<float>& Wp = m.t.at("pooler.dense.weight");
  const std::vector<float>& bp = m.t.at("pooler.dense.bias");
  const std::vector<float>& Wc = m.t.at("classifier.weight");
  const std::vector<float>& bc = m.t.at("classifier.bias");
  std::vector<double> pooled(H);
  for (int b = 0; b < B; ++b) {
    const double* x = x0 + (size_t)b * H;
    for (int j = 0; j < H; ++j) {
      double a = 0.0;
      for (int k = 0; k < H; ++k) a += (double)Wp[(size_t)j * H + k] * x[k];
      pooled[j] = std::tanh(a + (double)bp[j]);
    }
    for (int c = 0; c < C; ++c) {
      double a = 0.0;
      for (int k = 0; k < H; ++k) a += (double)Wc[(size_t)c * H + k] * pooled[k];
      logits[(size_t)b * C + c] = (float)(a + (double)bc[c]);
      if (logits64) logits64[(size_t)b * C + c] = a + (double)bc[c];
    }
  }
}

bool validate_inputs(const Model& m, const int* ids, const int* mask, int B, int S) {
  if (B < 1 || S < 1 || S > m.P) return false;
  for (int r = 0; r < B * S; ++r) {
    if (ids[r] < 0 || ids[r] >= m.V) return false;
    if (mask[r] != 0 && mask[r] != 1) return false;
  }
  for (int b = 0; b < B; ++b)
    if (mask[b * S] != 1) return false;  // DESIGN R5: position 0 must be a real token
  return true;
}

thread_local std::string g_err;

}  // namespace

// =================================================================== C API
extern "C" {

int or_abi_version() { return 1; }
const char* or_last_error() { return g_err.c_str(); }

void* or_create(int L, int H, int d, int V, int P, int C, float eps, int act, const int* heads,
                const int* ffn, const int* dtype) {
  if (L < 1 || H < 1 || d < 1 || V < 1 || P < 1 || C < 1 || !(eps > 0.0f)) { g_err = "bad config"; return nullptr; }
  Model* m = new Model();
  m->L = L; m->H = H; m->d = d; m->V = V; m->P = P; m->C = C; m->eps = eps; m->act = act;
  m->layers.resize(L);
  for (int l = 0; l < L; ++l) {
    if (heads[l] < 1 || ffn[l] < 1 || (dtype[l] != DT_F16 && dtype[l] != DT_I8)) { delete m; g_err = "bad layer"; return nullptr; }
    m->layers[l].A = heads[l]; m->layers[l].F = ffn[l]; m->layers[l].dt = dtype[l];
  }
  return m;
}

void or_destroy(void* h) { delete (Model*)h; }

// Load one fp32 tensor by HF name (optional "bert."/"roberta." prefix;
// RoBERTa head aliases classifier.dense -> pooler.dense, classifier.out_proj
// -> classifier).  Returns 0 on success, 2 on unknown name / wrong shape.
int or_load(void* h, const char* cname, const float* data, const int64_t* shape, int rank) {
  Model& m = *(Model*)h;
  std::string name(cname);
  strip_prefix(name, "bert.") || strip_prefix(name, "roberta.");
  if (name == "classifier.dense.weight") name = "pooler.dense.weight";
  else if (name == "classifier.dense.bias") name = "pooler.dense.bias";
  else if (name == "classifier.out_proj.weight") name = "classifier.weight";
  else if (name == "classifier.out_proj.bias") name = "classifier.bias";
  int layer; std::string key; std::vector<int64_t> es;
  if (!expected_shape(m, name, &layer, &key, &es)) { g_err = "unknown tensor " + name; return 2; }
  if ((int)es.size() != rank) { g_err = "rank mismatch " + name; return 2; }
  size_t n = 1;
  for (int i = 0; i < rank; ++i) {
    if (es[i] >= 0 && es[i] != shape[i]) { g_err = "shape mismatch " + name; return 2; }
    if (shape[i] < 1) { g_err = "empty dim " + name; return 2; }
    n *= (size_t)shape[i];
  }
  std::vector<float> v(data, data + n);
  if (layer < 0) m.t[key] = std::move(v); else m.layers[layer].t[key] = std::move(v);
  m.ready = false;
  return 0;
}

// Check every tensor is present and build the emu weights (a0 of SURVEY 8(a)):
// fused [Q|K|V], R16(W) for fp16 layers, (Wq, sw) for int8 layers.
int or_finalize(void* h) {
  Model& m = *(Model*)h;
  for (const char* k : kTopKeys)
    if (!m.t.count(k)) { g_err = std::string("missing ") + k; return 3; }
  for (int l = 0; l < m.L; ++l) {
    Layer& ly = m.layers[l];
    for (const char* k : kLayerKeys)
      if (!ly.t.count(k)) { g_err = "missing layer " + std::to_string(l) + " " + k; return 3; }
    const int H = m.H, D = ly.A * m.d, F = ly.F;
    ly.wqkv.clear(); ly.bqkv.clear();
    for (const char* w : {"attention.self.query", "attention.self.key", "attention.self.value"}) {
      const std::vector<float>& W = ly.t[std::string(w) + ".weight"];
      const std::vector<float>& b = ly.t[std::string(w) + ".bias"];
      ly.wqkv.insert(ly.wqkv.end(), W.begin(), W.end());
      ly.bqkv.insert(ly.bqkv.end(), b.begin(), b.end());
    }
    const std::vector<float>* Ws[4] = {&ly.wqkv, &ly.t["attention.output.dense.weight"],
                                       &ly.t["intermediate.dense.weight"], &ly.t["output.dense.weight"]};
    const int Ns[4] = {3 * D, H, F, H}, Ks[4] = {H, D, H, F};
    for (int i = 0; i < 4; ++i) {
      const std::vector<float>& W = *Ws[i];
      ly.w16[i].resize(W.size());
      for (size_t j = 0; j < W.size(); ++j) ly.w16[i][j] = r16(W[j]);
      ly.wq[i].resize(W.size());
      ly.sw[i].resize(Ns[i]);
      quant_weight(W.data(), Ns[i], Ks[i], ly.wq[i].data(), ly.sw[i].data());
    }
  }
  m.ready = true;
  return 0;
}

// Full forward pass.  ids, mask: [B, S] int32.  logits: [B, C] fp32.
// mode 0 = ref64, 1 = emu.  final_hidden (nullable): [B*S, H] fp32 copy of the
// last layer's output (fp16 values in emu mode).
// logits64 (nullable): the same logits before the final fp32 rounding.
int or_encode(void* h, const int* ids, const int* mask, int B, int S, int mode, int acc32, float* logits,
              double* logits64, float* final_hidden) {
  const Model& m = *(const Model*)h;
  if (!m.ready) { g_err = "not finalized"; return 3; }
  if (!validate_inputs(m, ids, mask, B, S)) { g_err = "bad input"; return 5; }
  const int H = m.H, M = B * S;
  std::vector<double> x0((size_t)B * H);
  if (mode == MODE_REF64) {
    std::vector<double> x((size_t)M * H);
    embed(m, ids, M, S, MODE_REF64, 0, x.data(), nullptr);
    for (int l = 0; l < m.L; ++l) {
      const Layer& ly = m.layers[l];
      const int D = ly.A * m.d, F = ly.F;
      std::vector<double> qkv((size_t)M * 3 * D), ctx((size_t)M * D), o((size_t)M * H), h1((size_t)M * H),
          it((size_t)M * F), y((size_t)M * H), tmp(H);
      linear(m, ly, 0, ly.wqkv, ly.bqkv, 3 * D, H, x.data(), nullptr, M, MODE_REF64, 0, qkv.data(), nullptr);
      attention<double>(qkv.data(), mask, B, S, ly.A, m.d, MODE_REF64, 0, ctx.data());
      linear(m, ly, 1, T_(ly, "attention.output.dense.weight"), T_(ly, "attention.output.dense.bias"), H, D,
             ctx.data(), nullptr, M, MODE_REF64, 0, o.data(), nullptr);
      for (int r = 0; r < M; ++r) {
        for (int j = 0; j < H; ++j) tmp[j] = o[(size_t)r * H + j] + x[(size_t)r * H + j];
        layer_norm64(tmp.data(), H, T_(ly, "attention.output.LayerNorm.weight").data(),
                     T_(ly, "attention.output.LayerNorm.bias").data(), m.eps, h1.data() + (size_t)r * H);
      }
      linear(m, ly, 2, T_(ly, "intermediate.dense.weight"), T_(ly, "intermediate.dense.bias"), F, H, h1.data(),
             nullptr, M, MODE_REF64, 0, it.data(), nullptr);
      for (size_t i = 0; i < it.size(); ++i) it[i] = act64(it[i], m.act);
      linear(m, ly, 3, T_(ly, "output.dense.weight"), T_(ly, "output.dense.bias"), H, F, it.data(), nullptr, M,
             MODE_REF64, 0, y.data(), nullptr);
      for (int r = 0; r < M; ++r) {
        for (int j = 0; j < H; ++j) tmp[j] = y[(size_t)r * H + j] + h1[(size_t)r * H + j];
        layer_norm64(tmp.data(), H, T_(ly, "output.LayerNorm.weight").data(), T_(ly, "output.LayerNorm.bias").data(),
                     m.eps, x.data() + (size_t)r * H);
      }
    }
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < H; ++j) x0[(size_t)b * H + j] = x[(size_t)(b * S) * H + j];
    if (final_hidden)
      for (size_t i = 0; i < x.size(); ++i) final_hidden[i] = (float)x[i];
  } else {
    std::vector<float> x((size_t)M * H);
    embed(m, ids, M, S, MODE_EMU, acc32, nullptr, x.data());
    for (int l = 0; l < m.L; ++l) {
      const Layer& ly = m.layers[l];
      const int D = ly.A * m.d, F = ly.F;
      std::vector<float> qkv((size_t)M * 3 * D), ctx((size_t)M * D), o((size_t)M * H), h1((size_t)M * H),
          it((size_t)M * F), y((size_t)M * H);
      run_stage(m, l, ST_QKV, x.data(), nullptr, mask, B, S, acc32, qkv.data());
      run_stage(m, l, ST_ATTN, qkv.data(), nullptr, mask, B, S, acc32, ctx.data());
      run_stage(m, l, ST_OPROJ, ctx.data(), nullptr, mask, B, S, acc32, o.data());
      run_stage(m, l, ST_LN1, o.data(), x.data(), mask, B, S, acc32, h1.data());
      run_stage(m, l, ST_FFN1, h1.data(), nullptr, mask, B, S, acc32, it.data());
      run_stage(m, l, ST_FFN2, it.data(), nullptr, mask, B, S, acc32, y.data());
      run_stage(m, l, ST_LN2, y.data(), h1.data(), mask, B, S, acc32, x.data());
    }
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < H; ++j) x0[(size_t)b * H + j] = (double)x[(size_t)(b * S) * H + j];
    if (final_hidden) std::memcpy(final_hidden, x.data(), x.size() * sizeof(float));
  }
  head(m, x0.data(), B, logits, logits64);
  return 0;
}

// One emu stage of layer l from caller-supplied fp16 inputs (as float).
int or_stage(void* h, int l, int stage, const float* in_a, const float* in_b, const int* mask, int B, int S,
             int acc32, float* out) {
  const Model& m = *(const Model*)h;
  if (!m.ready) { g_err = "not finalized"; return 3; }
  if (l < 0 || l >= m.L) { g_err = "bad layer"; return 1; }
  return run_stage(m, l, stage, in_a, in_b, mask, B, S, acc32, out);
}

// Embedding stage alone (emu): ids [B,S] -> X16 [B*S, H].
int or_embed(void* h, const int* ids, int B, int S, int acc32, float* x16) {
  const Model& m = *(const Model*)h;
  if (!m.ready) { g_err = "not finalized"; return 3; }
  embed(m, ids, B * S, S, MODE_EMU, acc32, nullptr, x16);
  return 0;
}

// Head stage alone: X [B*S, H] (fp16 values) -> logits [B, C].
int or_head(void* h, const float* x, int B, int S, float* logits) {
  const Model& m = *(const Model*)h;
  if (!m.ready) { g_err = "not finalized"; return 3; }
  std::vector<double> x0((size_t)B * m.H);
  for (int b = 0; b < B; ++b)
    for (int j = 0; j < m.H; ++j) x0[(size_t)b * m.H + j] = (double)x[(size_t)(b * S) * m.H + j];
  head(m, x0.data(), B, logits, nullptr);
  return 0;
}

// Emu weights as the oracle prepared them (for packer parity tests).
// which: 0 qkv, 1 o, 2 ffn1, 3 ffn2.  q: [N*K] s8, s: [N], w16: [N*K] (nullable).
int or_prepared_weight(void* h, int l, int which, int8_t* q, float* s, float* w16) {
  const Model& m = *(const Model*)h;
  if (!m.ready) { g_err = "not finalized"; return 3; }
  const Layer& ly = m.layers[l];
  if (q) std::memcpy(q, ly.wq[which].data(), ly.wq[which].size());
  if (s) std::memcpy(s, ly.sw[which].data(), ly.sw[which].size() * sizeof(float));
  if (w16) std::memcpy(w16, ly.w16[which].data(), ly.w16[which].size() * sizeof(float));
  return 0;
}

// ---- primitives (stage-level pins) ----
int or_q8row(const float* x, int M, int K, int8_t* q, float* s) {
  for (int m = 0; m < M; ++m) q8row(x + (size_t)m * K, K, q + (size_t)m * K, s + m);
  return 0;
}

int or_q8tensor(const float* x, int M, int K, uint8_t* q, float* scale, int* zp) {
  q8tensor(x, (size_t)M * K, q, scale, zp);
  return 0;
}

// Activation quantizer of the int8 layers: 0 Q8row (default), 1 Q8tensor.
int or_set_act_quant(void* h, int mode) {
  if (!h || (mode != 0 && mode != 1)) return -1;
  static_cast<Model*>(h)->act_quant = mode;
  return 0;
}

int or_quant_weight(const float* W, int N, int K, int8_t* q, float* s) {
  quant_weight(W, N, K, q, s);
  return 0;
}

// Brute-force int32 GEMM C[M,N] = sum_k A[m,k] W[n,k] (exact integer arithmetic).
int or_gemm_s8(const int8_t* A, const int8_t* W, int M, int N, int K, int32_t* C) {
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      int32_t acc = 0;
      for (int k = 0; k < K; ++k) acc += (int32_t)A[(size_t)m * K + k] * (int32_t)W[(size_t)n * K + k];
      C[(size_t)m * N + n] = acc;
    }
  return 0;
}

// R16 of an fp32 array (fp16 round trip, RNE).
int or_r16(const float* x, size_t n, float* y) {
  for (size_t i = 0; i < n; ++i) y[i] = r16(x[i]);
  return 0;
}

// Activation in fp64 on fp32 inputs (for closed-form pins).
int or_act(const float* x, size_t n, int act, double* y) {
  for (size_t i = 0; i < n; ++i) y[i] = act64((double)x[i], act);
  return 0;
}

// LayerNorm of rows (fp64 statistics) for closed-form pins: x [M,H] -> y [M,H] fp64.
int or_layer_norm64(const double* x, int M, int H, const float* g, const float* b, float eps, double* y) {
  for (int r = 0; r < M; ++r) layer_norm64(x + (size_t)r * H, H, g, b, eps, y + (size_t)r * H);
  return 0;
}

// Attention on caller data (emu or ref64), single layer geometry (A heads, d).
int or_attention(const float* qkv, const int* mask, int B, int S, int A, int d, int mode, float* ctx) {
  if (mode == MODE_REF64) {
    size_t n = (size_t)B * S * 3 * A * d, nc = (size_t)B * S * A * d;
    std::vector<double> q(qkv, qkv + n), c(nc);
    attention<double>(q.data(), mask, B, S, A, d, MODE_REF64, 0, c.data());
    for (size_t i = 0; i < nc; ++i) ctx[i] = (float)c[i];
    return 0;
  }
  attention<float>(qkv, mask, B, S, A, d, MODE_EMU, 0, ctx);
  return 0;
}

}  // extern "C"
