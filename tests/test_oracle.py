"""CPU pins for the oracle (``-m "not gpu"``).

The oracle (oracle/oracle.cpp) is pinned against things other than itself:
SPEC worked examples (tests/golden/spec_examples.json, each cited), closed
forms, HuggingFace's BertForSequenceClassification in fp64 (a library
routine), numpy integer matmul (brute force), invariants the paper fixes
(pruned == zeroed; padding/batch invariance; quantization error
<= scale/2) and error bounds.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import MODE_EMU, MODE_REF64, Oracle
from paper_2010_13382_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def small_cfg(**kw):
    base = dict(name="t", num_layers=2, hidden=128, head_dim=64, heads=[2, 2], ffn_dim=[256, 256], dtype=[0, 0],
                vocab_size=1000, max_positions=64, num_classes=2, ln_eps=1e-12, batch=4, seq=32)
    base.update(kw)
    return synth.ModelConfig(**base)


# ------------------------------------------------------------ SPEC examples
def test_spec_softmax_examples():
    # d = 4 so 1/sqrt(d) = 0.5 exactly; q = [2,0,0,0], k_j = [s_j,0,0,0] -> score s_j;
    # v_j = one-hot e_j, so ctx = the probability row.
    for ex in GOLD["softmax"]:
        s = [math.log(2.0) if v == "ln2" else v for v in ex["scores"]]
        n = len(s)
        d = 4
        qkv = np.zeros((n, 3 * d), np.float32)
        qkv[0, 0] = 2.0
        for j in range(n):
            qkv[j, d + 0] = s[j]
            qkv[j, 2 * d + j] = 1.0
        ctx = oracle.attention(qkv, np.ones((1, n), np.int32), 1, d, mode=MODE_REF64)
        np.testing.assert_allclose(ctx[0, :n], ex["probs"], atol=ex["tol"], err_msg=ex["cite"])


def test_spec_layer_norm_examples():
    for ex in GOLD["layer_norm"]:
        y = oracle.layer_norm64(np.array([ex["x"]]), ex["gamma"], ex["beta"], ex["eps"])
        np.testing.assert_allclose(y[0], ex["y"], atol=ex["tol"], err_msg=ex["cite"])


def test_spec_activation_examples():
    kinds = {"gelu": synth.ACT_GELU, "relu": synth.ACT_RELU, "gelu_tanh": synth.ACT_GELU_TANH}
    for ex in GOLD["activation"]:
        y = oracle.act(np.array([ex["x"]]), kinds[ex["act"]])[0]
        assert abs(y - ex["y"]) <= ex["tol"], ex["cite"]


def test_spec_weight_quant_examples():
    for ex in GOLD["weight_quant"]:
        q, s = oracle.quant_weight(np.array([ex["channel"]], np.float32))
        assert s[0] == np.float32(ex["scale"]), ex["cite"]
        assert q[0].tolist() == ex["q"], ex["cite"]


def test_act_quant_examples_and_rne_tie():
    for ex in GOLD["act_quant"]:
        q, s = oracle.q8row(np.array([ex["row"]], np.float32))
        assert abs(float(s[0]) - ex["scale"]) <= ex["scale_tol"], ex["cite"]
        assert q[0].tolist() == ex["q"], ex["cite"]


def test_quant_round_trip_bound():
    # |q*s - x| <= s/2, up to one fp32 rounding of x/s (ratio 1.000007)
    rng = np.random.default_rng(0)
    x = np.float16(rng.standard_normal((64, 300)) * 3).astype(np.float32)
    x[5] = 0.0
    q, s = oracle.q8row(x)
    err = np.abs(q.astype(np.float64) * s[:, None] - x)
    assert np.all(err <= s[:, None] / 2 * (1 + 2e-5))
    assert np.all(np.abs(q) <= 127) and q.min() >= -127
    assert s[5] == 1.0 and np.all(q[5] == 0)
    # the row maximum maps to +-127
    assert np.all(np.abs(q[np.arange(64) != 5]).max(axis=1) == 127)


def test_gemm_s8_brute_force_vs_numpy():
    rng = np.random.default_rng(1)
    for M, N, K in [(1, 1, 1), (7, 13, 312), (33, 17, 1200), (5, 9, 4096)]:
        A = rng.integers(-127, 128, (M, K), dtype=np.int8)
        W = rng.integers(-127, 128, (N, K), dtype=np.int8)
        C = oracle.gemm_s8(A, W)
        ref = A.astype(np.int64) @ W.astype(np.int64).T
        assert np.array_equal(C.astype(np.int64), ref)
    # identity W -> acc = A
    A = rng.integers(-127, 128, (4, 16), dtype=np.int8)
    assert np.array_equal(oracle.gemm_s8(A, np.eye(16, dtype=np.int8)), A.astype(np.int32))


def _tiny_linear_model(H, A, d, Wo, bo):
    """1-layer model whose O-projection is Wo [H, A*d], bo [H]; other tensors random."""
    cfg = small_cfg(num_layers=1, hidden=H, head_dim=d, heads=[A], ffn_dim=[4], dtype=[synth.I8], vocab_size=16)
    w = synth.make_weights(cfg)
    w["encoder.layer.0.attention.output.dense.weight"] = np.asarray(Wo, np.float32)
    w["encoder.layer.0.attention.output.dense.bias"] = np.asarray(bo, np.float32)
    return cfg, Oracle(cfg, w)


def test_spec_gemm_i8_examples():
    ex = GOLD["gemm_i8"][0]
    cfg, o = _tiny_linear_model(1, 1, 1, ex["w"], [0.0])
    y = o.stage(0, oracle.ST_OPROJ, np.array(ex["a"], np.float32))
    assert abs(y[0, 0] - ex["y"][0][0]) <= ex["tol"], ex["cite"]
    ex = GOLD["gemm_i8"][1]
    cfg, o = _tiny_linear_model(3, 1, 2, ex["w"], ex["bias"])
    y = o.stage(0, oracle.ST_OPROJ, np.array(ex["a"], np.float32))
    # bias broadcast exactly (then stored as fp16: numpy's own fp16 conversion)
    expect = np.float16(np.array(ex["y"], np.float32)).astype(np.float32)
    assert np.array_equal(y, expect), ex["cite"]


def test_count_macs_formula():
    ex = GOLD["count_macs"][0]
    cfg = small_cfg(num_layers=1, hidden=ex["H"], head_dim=ex["H"], heads=[1], ffn_dim=[ex["F"]], dtype=[0])
    head = 2 * (ex["H"] ** 2 + ex["H"] * cfg.num_classes)
    assert (cfg.flops_per_seq(ex["s"]) - head) / 2 == ex["macs"], ex["cite"]


# ------------------------------------------------------- linear-layer bounds
def test_linear_f16_matches_fp64_matmul_within_one_ulp():
    rng = np.random.default_rng(2)
    H, A, d = 48, 2, 16
    Wo = (rng.standard_normal((H, A * d)) * 0.1).astype(np.float32)
    bo = (rng.standard_normal(H) * 0.1).astype(np.float32)
    cfg = small_cfg(num_layers=1, hidden=H, head_dim=d, heads=[A], ffn_dim=[4], dtype=[synth.F16], vocab_size=16)
    w = synth.make_weights(cfg)
    w["encoder.layer.0.attention.output.dense.weight"] = Wo
    w["encoder.layer.0.attention.output.dense.bias"] = bo
    o = Oracle(cfg, w)
    x = np.float16(rng.standard_normal((37, A * d))).astype(np.float32)
    y = o.stage(0, oracle.ST_OPROJ, x)
    W16 = np.float16(Wo).astype(np.float64)
    ref = x.astype(np.float64) @ W16.T + bo.astype(np.float64)
    # one fp16 rounding of the output (2^-11 relative) + fp32 rounding slack
    assert np.all(np.abs(y - ref) <= np.abs(ref) * 2.0 ** -11 + 1e-6)


def test_linear_i8_error_bound_and_frobenius():
    # rel. Frobenius vs fp32 <= 0.02; elementwise the quantization bound
    rng = np.random.default_rng(3)
    H, A, d = 256, 4, 64
    Wo = (rng.standard_normal((H, A * d)) * 0.02).astype(np.float32)
    bo = (rng.standard_normal(H) * 0.02).astype(np.float32)
    cfg, o = _tiny_linear_model(H, A, d, Wo, bo)
    x = np.float16(rng.standard_normal((64, A * d))).astype(np.float32)
    y = o.stage(0, oracle.ST_OPROJ, x).astype(np.float64)
    ref = x.astype(np.float64) @ Wo.astype(np.float64).T + bo
    rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert rel <= 0.02
    sx = np.abs(x).max(axis=1) / 127.0
    sw = np.abs(Wo).max(axis=1) / 127.0
    bound = (np.abs(x).sum(1)[:, None] * sw[None, :] / 2 + sx[:, None] * np.abs(Wo).sum(1)[None, :] / 2
             + sx[:, None] * sw[None, :] * (A * d) / 4)
    assert np.all(np.abs(y - ref) <= bound + np.abs(ref) * 2.0 ** -10 + 1e-6)


# ---------------------------------------------------------- HF fp64 parity
@pytest.mark.parametrize("act", ["gelu", "relu"])
def test_ref64_matches_hf_bert_fp64(act):
    torch = pytest.importorskip("torch")
    transformers = pytest.importorskip("transformers")
    cfg = small_cfg(act={"gelu": synth.ACT_GELU, "relu": synth.ACT_RELU}[act])
    w = synth.make_weights(cfg, seed=7)
    hf_cfg = transformers.BertConfig(vocab_size=cfg.vocab_size, hidden_size=cfg.hidden, num_hidden_layers=cfg.num_layers,
                                     num_attention_heads=cfg.heads[0], intermediate_size=cfg.ffn_dim[0],
                                     max_position_embeddings=cfg.max_positions, type_vocab_size=2, hidden_act=act,
                                     layer_norm_eps=cfg.ln_eps, num_labels=cfg.num_classes,
                                     hidden_dropout_prob=0.0, attention_probs_dropout_prob=0.0)
    hf_cfg._attn_implementation = "eager"
    model = transformers.BertForSequenceClassification(hf_cfg).double().eval()
    sd = {("bert." + k if not k.startswith("classifier") else k): torch.from_numpy(v.astype(np.float64))
          for k, v in w.items()}
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected and all("position_ids" in m for m in missing), (missing, unexpected)
    ids, mask = synth.make_inputs(cfg, lengths=[32, 20, 7, 31])
    with torch.no_grad():
        ref = model(input_ids=torch.from_numpy(ids.astype(np.int64)),
                    attention_mask=torch.from_numpy(mask.astype(np.int64)),
                    token_type_ids=torch.zeros(ids.shape, dtype=torch.int64)).logits.numpy()
    got = Oracle(cfg, w).encode(ids, mask, mode=MODE_REF64, fp64_logits=True)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.abs(ref).max()), np.max(np.abs(got - ref))


def test_hf_names_with_prefix_and_roberta_aliases():
    cfg = small_cfg(num_layers=1, heads=[2], ffn_dim=[64])
    w = synth.make_weights(cfg)
    w2 = {}
    for k, v in w.items():
        if k == "pooler.dense.weight":
            w2["classifier.dense.weight"] = v
        elif k == "pooler.dense.bias":
            w2["classifier.dense.bias"] = v
        elif k == "classifier.weight":
            w2["classifier.out_proj.weight"] = v
        elif k == "classifier.bias":
            w2["classifier.out_proj.bias"] = v
        else:
            w2["roberta." + k] = v
    ids, mask = synth.make_inputs(cfg)
    a = Oracle(cfg, w).encode(ids, mask, mode=MODE_EMU)
    b = Oracle(cfg, w2).encode(ids, mask, mode=MODE_EMU)
    assert np.array_equal(a, b)


def test_load_rejects_bad_names_and_shapes():
    cfg = small_cfg(num_layers=1, heads=[2], ffn_dim=[64])
    o = Oracle(cfg)
    with pytest.raises(RuntimeError):
        o.load({"encoder.layer.0.attention.self.query.weight": np.zeros((3, 3), np.float32)})
    with pytest.raises(RuntimeError):
        o.load({"no.such.tensor": np.zeros((3,), np.float32)})
    with pytest.raises(RuntimeError):  # finalize with missing tensors
        o.load({})


# ---------------------------------------------------------------- invariants
KEEP_HEADS = [[0, 1], [1]]          # ragged heads [2, 1] like BASELINE configs[0]
KEEP_FFN = [list(range(256)), list(range(0, 256, 2))]


@pytest.mark.parametrize("dt", [[0, 0], [1, 1], [1, 0]])
@pytest.mark.parametrize("mode", [MODE_REF64, MODE_EMU])
def test_pruned_equals_zeroed(dt, mode):
    """P:93 re-group/reconnect: a sliced (pruned) model computes exactly what the
    unpruned model computes with the removed heads / FFN units zeroed."""
    cfg = small_cfg(dtype=dt)
    w = synth.make_weights(cfg, seed=11)
    pcfg, pw = synth.prune_slice(cfg, w, KEEP_HEADS, KEEP_FFN)
    zw = synth.prune_zero(cfg, w, KEEP_HEADS, KEEP_FFN)
    assert pcfg.heads == [2, 1] and pcfg.ffn_dim == [256, 128]
    ids, mask = synth.make_inputs(cfg, lengths=[32, 20, 7, 31])
    a = Oracle(pcfg, pw).encode(ids, mask, mode=mode)
    b = Oracle(cfg, zw).encode(ids, mask, mode=mode)
    assert np.array_equal(a, b), np.abs(a - b).max()


@pytest.mark.parametrize("dt", [0, 1])
def test_padding_and_batch_invariance(dt):
    cfg = small_cfg(dtype=[dt, dt])
    w = synth.make_weights(cfg, seed=5)
    o = Oracle(cfg, w)
    lengths = [32, 20, 7, 31]
    ids, mask = synth.make_inputs(cfg, lengths=lengths)
    full = o.encode(ids, mask)
    for b, n in enumerate(lengths):
        alone = o.encode(ids[b:b + 1, :n], mask[b:b + 1, :n])
        assert np.array_equal(alone[0], full[b])
    # garbage in padded positions does not matter
    ids2 = ids.copy()
    ids2[mask == 0] = 17
    assert np.array_equal(o.encode(ids2, mask), full)


def test_attention_free_model_gives_bias():
    cfg = small_cfg(num_layers=1, heads=[2], ffn_dim=[64], dtype=[1])
    w = synth.make_weights(cfg, seed=3)
    p = "encoder.layer.0.attention."
    for t in ("query", "key", "value"):
        w[p + f"self.{t}.weight"][:] = 0
        w[p + f"self.{t}.bias"][:] = 0
    w[p + "output.dense.weight"][:] = 0
    o = Oracle(cfg, w)
    ids, mask = synth.make_inputs(cfg, B=2, S=8)
    x = o.embed(ids)
    qkv = o.stage(0, oracle.ST_QKV, x)
    assert np.all(qkv == 0)
    ctx = o.stage(0, oracle.ST_ATTN, qkv, mask=mask)
    assert np.all(ctx == 0)
    out = o.stage(0, oracle.ST_OPROJ, ctx)
    expect = np.float16(w[p + "output.dense.bias"]).astype(np.float32)
    assert np.array_equal(out, np.broadcast_to(expect, out.shape))


def test_attention_special_cases():
    rng = np.random.default_rng(9)
    B, S, A, d = 2, 8, 2, 16
    D = A * d
    qkv = np.float16(rng.standard_normal((B * S, 3 * D))).astype(np.float32)
    # one valid key -> ctx = v_0 exactly (P16 = 1)
    mask = np.zeros((B, S), np.int32)
    mask[:, 0] = 1
    ctx = oracle.attention(qkv, mask, A, d)
    for b in range(B):
        v0 = qkv[b * S, 2 * D:]
        assert np.array_equal(ctx[b * S:(b + 1) * S], np.broadcast_to(v0, (S, D)))
    # q = 0 -> uniform over valid keys -> ctx = mean of valid v (ref64)
    q0 = qkv.copy()
    q0[:, :D] = 0
    mask = np.ones((B, S), np.int32)
    mask[1, 5:] = 0
    ctx = oracle.attention(q0, mask, A, d, mode=MODE_REF64)
    for b in range(B):
        n = mask[b].sum()
        mean_v = q0[b * S:b * S + n, 2 * D:].astype(np.float64).mean(0)
        np.testing.assert_allclose(ctx[b * S:(b + 1) * S], np.broadcast_to(mean_v, (S, D)), atol=1e-6)
    # rows of p sum to 1: v = all ones -> ctx = sum p (ref64 exact; emu within fp16 rounding of p)
    q1 = qkv.copy()
    q1[:, 2 * D:] = 1.0
    c64 = oracle.attention(q1, mask, A, d, mode=MODE_REF64)
    np.testing.assert_allclose(c64, 1.0, atol=1e-6)
    c16 = oracle.attention(q1, mask, A, d, mode=MODE_EMU)
    np.testing.assert_allclose(c16, 1.0, atol=S * 2.0 ** -11)


def test_masked_keys_do_not_contribute():
    rng = np.random.default_rng(4)
    B, S, A, d = 1, 8, 1, 8
    qkv = np.float16(rng.standard_normal((S, 3 * A * d))).astype(np.float32)
    mask = np.ones((B, S), np.int32)
    mask[0, 6:] = 0
    a = oracle.attention(qkv, mask, A, d)
    qkv2 = qkv.copy()
    qkv2[6:, A * d:] = 50.0  # huge keys / values in masked positions
    b = oracle.attention(qkv2, mask, A, d)
    assert np.array_equal(a[:6], b[:6])


def test_layer_norm_zero_variance_row_gives_beta():
    g = np.array([2.0, 3.0, 4.0], np.float32)
    b = np.array([0.5, -0.25, 1.0], np.float32)
    y = oracle.layer_norm64(np.array([[7.0, 7.0, 7.0]]), g, b, 1e-5)
    assert np.array_equal(y[0], b.astype(np.float64))


def test_emu_close_to_ref64_c1():
    """Approximation error of the emulated numerics vs the fp64 definition
    (fp16 ~1e-4, int8 ~1e-3 relative on C1)."""
    cfg = synth.config("c1")
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, lengths=[32, 20, 7, 31])
    ref = Oracle(cfg.with_dtype(0), w).encode(ids, mask, mode=MODE_REF64)
    f16 = Oracle(cfg.with_dtype(0), w).encode(ids, mask, mode=MODE_EMU)
    i8 = Oracle(cfg.with_dtype(1), w).encode(ids, mask, mode=MODE_EMU)
    assert np.abs(f16 - ref).max() <= 1e-3
    assert np.abs(i8 - ref).max() <= 2e-2 * np.abs(ref).max()
    assert np.abs(i8 - ref).max() > 0  # quantization really happened


def test_acc32_drift_small_on_c1():
    cfg = synth.config("c1")
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, lengths=[32, 20, 7, 31])
    o = Oracle(cfg, w)
    a = o.encode(ids, mask)
    b = o.encode(ids, mask, acc32=True)
    assert np.abs(a - b).max() <= 1e-3 * np.abs(a).max()


def test_invalid_inputs_rejected():
    cfg = small_cfg(num_layers=1, heads=[2], ffn_dim=[64])
    o = Oracle(cfg, synth.make_weights(cfg))
    ids, mask = synth.make_inputs(cfg, B=2, S=8)
    bad = ids.copy()
    bad[0, 3] = cfg.vocab_size
    with pytest.raises(RuntimeError):
        o.encode(bad, mask)
    m2 = mask.copy()
    m2[1, 0] = 0
    with pytest.raises(RuntimeError):
        o.encode(ids, m2)


# ------------------------------------- per-tensor u8 activations (NEXT-2)
def test_q8tensor_worked_example():
    # DESIGN R22 by hand: x = [-1, 0, 2, 3]: lo = -1, hi = 3, scale = fl(4/255),
    # zp = RNE(1/scale) = RNE(63.75) = 64; q = RNE(x/scale) + 64 with
    # 2/scale = 127.4999.. -> 127 and 3/scale = 191.2499.. -> 191 (fl(4/255) >
    # 4/255), -1/scale -> -64: q = [0, 64, 191, 255]
    q, s, z = oracle.q8tensor(np.array([[-1, 0, 2, 3]], np.float32))
    assert s == np.float32(4.0) / np.float32(255.0) and z == 64
    np.testing.assert_array_equal(q, [[0, 64, 191, 255]])
    # all-positive tensor: lo = 0 -> zp = 0; all-zero tensor: scale 1, q = 0
    q, s, z = oracle.q8tensor(np.array([[0.5, 1.0]], np.float32))
    assert z == 0 and q[0, 1] == 255
    q, s, z = oracle.q8tensor(np.zeros((2, 3), np.float32))
    assert s == 1.0 and z == 0 and not q.any()


def test_q8tensor_round_trip_bound():
    # P:104 / S:152 analogue: |(q - zp) * scale - x| <= scale / 2 (plus the
    # zero-point rounding) for every element of the tensor
    rng = np.random.default_rng(12)
    for shift in (0.0, 0.7, -0.7):
        x = np.float16(rng.standard_normal((37, 91)) * 2 + shift).astype(np.float32)
        q, s, z = oracle.q8tensor(x)
        assert 0 <= z <= 255
        deq = (q.astype(np.float64) - z) * s
        assert np.abs(deq - x).max() <= s * 1.0 + 1e-7  # s/2 from x, s/2 from the nudged zero point
        lo, hi = min(0.0, x.min()), max(0.0, x.max())
        assert abs(s - (hi - lo) / 255) <= 1e-6 * abs(s)


def test_linear_i8_per_tensor_vs_dequantized_fp64():
    """The per-tensor int8 linear equals the fp64 product of the DEQUANTIZED
    operands (the zp * colsum correction is exact in int32), up to the fp32
    epilogue and fp16 output roundings."""
    rng = np.random.default_rng(4)
    H, A, d = 256, 4, 64
    Wo = (rng.standard_normal((H, A * d)) * 0.02).astype(np.float32)
    bo = (rng.standard_normal(H) * 0.02).astype(np.float32)
    cfg = small_cfg(num_layers=1, hidden=H, heads=[A], ffn_dim=[256], dtype=[1])
    o = Oracle(cfg, act_quant=1)
    w = synth.make_weights(cfg)
    w["encoder.layer.0.attention.output.dense.weight"] = Wo
    w["encoder.layer.0.attention.output.dense.bias"] = bo
    o.load(w)
    x = np.float16(rng.standard_normal((64, A * d)) + 0.3).astype(np.float32)
    y = o.stage(0, oracle.ST_OPROJ, x).astype(np.float64)
    q, s, z = oracle.q8tensor(x)
    wq, sw = oracle.quant_weight(Wo)
    ref = ((q.astype(np.float64) - z) * s) @ (wq.astype(np.float64) * sw[:, None].astype(np.float64)).T + bo
    # the stage output is rounded to fp16 (half an ulp) after the fp32 epilogue
    assert np.all(np.abs(y - ref) <= np.abs(ref) * 2.0 ** -11 + 4e-6 * np.abs(ref).max())
    # and it is a different quantizer from Q8row (per row) on the same input
    o_row = Oracle(cfg, w)
    assert not np.array_equal(o_row.stage(0, oracle.ST_OPROJ, x), y.astype(np.float32))


def test_per_tensor_and_per_row_accuracy_vs_ref64_c1():
    """Both int8 activation quantizers stay close to the fp64 reference; the
    per-row scheme (the north_star's) is the more accurate on average."""
    cfg = synth.config("c1").with_dtype([1, 1])
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, seed=31)
    ref = Oracle(cfg, w).encode(ids, mask, mode=MODE_REF64, fp64_logits=True)
    e_row = np.abs(Oracle(cfg, w).encode(ids, mask) - ref).max()
    e_ten = np.abs(Oracle(cfg, w, act_quant=1).encode(ids, mask) - ref).max()
    scale = np.abs(ref).max()
    assert e_row <= 0.05 * scale and e_ten <= 0.1 * scale


def test_per_tensor_linear_vs_pytorch_fbgemm_dynamic():
    """SURVEY 8(f) NEXT-2 pin: the oracle's per-tensor u8 (zero point) x
    per-channel s8 linear against PyTorch's FBGEMM dynamic quantized linear
    (the paper's CPU int8 path), activation range not reduced.  The two
    differ only in the weight scale convention (amax / 127 here, R7; amax /
    127.5 with codes in [-128, 127] in PyTorch) and the zero-point choice, so
    both sit within the int8 error envelope of the fp64 product and close to
    each other; a wrong zero-point correction (zp * colsum) would be off by
    orders of magnitude."""
    torch = pytest.importorskip("torch")
    if "fbgemm" not in torch.backends.quantized.supported_engines:
        pytest.skip("no FBGEMM engine")
    import warnings
    rng = np.random.default_rng(21)
    H, A, d, M = 256, 4, 64, 64
    Wo = (rng.standard_normal((H, A * d)) * 0.02).astype(np.float32)
    bo = (rng.standard_normal(H) * 0.02).astype(np.float32)
    cfg = small_cfg(num_layers=1, hidden=H, heads=[A], ffn_dim=[256], dtype=[1])
    w = synth.make_weights(cfg)
    w["encoder.layer.0.attention.output.dense.weight"] = Wo
    w["encoder.layer.0.attention.output.dense.bias"] = bo
    o = Oracle(cfg, w, act_quant=1)
    x = np.float16(rng.standard_normal((M, A * d)) + 0.3).astype(np.float32)
    ours = o.stage(0, oracle.ST_OPROJ, x).astype(np.float64)
    lin = torch.nn.Linear(A * d, H)
    with torch.no_grad():
        lin.weight.copy_(torch.from_numpy(Wo))
        lin.bias.copy_(torch.from_numpy(bo))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        torch.backends.quantized.engine = "fbgemm"
        from torch.ao.quantization import per_channel_dynamic_qconfig, quantize_dynamic
        q = quantize_dynamic(torch.nn.Sequential(lin), {torch.nn.Linear: per_channel_dynamic_qconfig},
                             dtype=torch.qint8)[0]
        fb = torch.ops.quantized.linear_dynamic(torch.from_numpy(x), q._packed_params._packed_params,
                                                False).numpy().astype(np.float64)
    ref = x.astype(np.float64) @ Wo.astype(np.float64).T + bo
    rel = lambda a: np.linalg.norm(a - ref) / np.linalg.norm(ref)
    assert rel(ours) < 2e-2 and rel(fb) < 2e-2, (rel(ours), rel(fb))  # measured 1.16e-2 and 1.14e-2
    assert np.linalg.norm(ours - fb) / np.linalg.norm(ref) < 1.5e-2
    # the zero point matters: dropping its correction is a gross error
    qx, s, z = oracle.q8tensor(x)
    wq, sw = oracle.quant_weight(Wo)
    no_zp = (qx.astype(np.float64) * s) @ (wq.astype(np.float64) * sw[:, None]).T + bo
    assert rel(no_zp) > 10 * rel(ours)
