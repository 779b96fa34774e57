"""Model-level parity on the GPU (``-m gpu``) through the C ABI:

* stage lockstep: each stage of layer l is re-run by the oracle on the GPU's
  own fp16 input of that stage; int8 GEMM stages must match BIT FOR BIT
  (int32 accumulators + fma dequant + R16, DESIGN "Tolerances");
* layer lockstep: the oracle runs a whole layer from the GPU's layer input;
* end to end: logits vs the oracle (emu) under the tolerance contract;
* invariants: padding / batch invariance, pruned == zeroed, graphs on/off,
  host-buffer path; input errors.
"""
import numpy as np
import pytest

import oracle
from oracle import Oracle
from paper_2010_13382_b200 import fastformers as ffb
from paper_2010_13382_b200 import synth
from paper_2010_13382_b200.fastformers import FF_E_INPUT, FF_E_SHAPE, Encoder, FFError

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def f32(t):
    return t.float().cpu().numpy()


def assert_close16(got, ref, what, frac=1e-4, slack=0.0):
    """fp16 stage tolerance (DESIGN "Tolerances"): elements differing by more
    than 2 fp16 ulps (2^-10 relative, floor 2^-14 = smallest normal fp16, which
    covers fp32 accumulation-order noise near zero) -- plus a per-element
    `slack` where an unobservable intermediate may round either way -- are
    <= 1e-4 of the tensor, no element is off by more than 8 ulps of max|ref|,
    rel. Frobenius <= 1e-3."""
    d = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    big = d > np.abs(ref) * 2.0 ** -10 + 2.0 ** -14 + slack
    rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert big.mean() <= frac, f"{what}: {int(big.sum())} elements beyond 2 ulp (max abs {d.max():.3e})"
    assert d.max() <= 8 * 2.0 ** -10 * max(np.abs(ref).max(), 2.0 ** -4), f"{what}: max abs {d.max():.3e}"
    assert rel <= 1e-3, f"{what}: rel {rel:.3e}"


def _ln_slack_of_fp16_gemm(a16, W, b, res, gamma, eps):
    """Per-element bound on how much LN(R16(a16 W16^T + b) + res) can move
    when R16 of the fp16 GEMM output is taken from any fp32 accumulation order:
    an output o_j is ambiguous when the fp32 accumulation error bound
    K 2^-24 sum_k |a_k w_k| (fp64 sums) reaches an fp16 rounding midpoint; then
    it may differ by one fp16 ulp u_j.  To first order, with x = o + res,
    r = 1/sqrt(var + eps):  |dy_i| <= |g_i| r (|do_i| + sum|do| / H
    + r^2 |x_i - mu| sum(|x - mu| |do|) / H)."""
    W16 = W.astype(np.float16).astype(np.float64)
    a = a16.astype(np.float64)
    acc = a @ W16.T
    K = a.shape[1]
    err = K * 2.0 ** -24 * (np.abs(a) @ np.abs(W16).T)
    lo = np.float16((acc - err).astype(np.float32) + b.astype(np.float32))
    hi = np.float16((acc + err).astype(np.float32) + b.astype(np.float32))
    o = np.float16(acc.astype(np.float32) + b.astype(np.float32)).astype(np.float64)
    do = np.where(lo != hi, np.spacing(np.abs(o).astype(np.float16)).astype(np.float64), 0.0)
    x = o + res.astype(np.float64)
    H = x.shape[1]
    mu = x.mean(1, keepdims=True)
    r = 1.0 / np.sqrt(((x - mu) ** 2).mean(1, keepdims=True) + eps)
    g = np.abs(gamma.astype(np.float64))[None, :]
    dmu = do.sum(1, keepdims=True) / H
    dvar = (np.abs(x - mu) * do).sum(1, keepdims=True) / H
    return 1.01 * g * r * (do + dmu + r * r * np.abs(x - mu) * dvar)


def small(cfg, B, S):
    return cfg.with_batch(B, S)


CASES = {
    "c1_i8": (synth.config("c1"), [1, 1], 4, 32),
    "c1_f16": (synth.config("c1"), [0, 0], 4, 32),
    "c1_mixed": (synth.config("c1"), [1, 0], 4, 32),
    "c2_i8": (synth.config("c2"), 1, 2, 128),
    "c2_f16": (synth.config("c2"), 0, 2, 128),
    "c3_i8": (synth.config("c3"), 1, 2, 128),
    "c3_f16": (synth.config("c3"), 0, 2, 128),
    "c4_f16": (synth.config("c4"), 0, 1, 512),
    "c5_f16": (synth.config("c5"), 0, 1, 256),
}


def build_case(name, ragged=True, act=None):
    cfg, dt, B, S = CASES[name]
    cfg = cfg.with_dtype(dt).with_batch(B, S)
    if act is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, act=act)
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, B=B, S=S, ragged=ragged, seed=77)
    return cfg, w, ids, mask


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("name", ["c1_i8", "c1_f16", "c1_mixed", "c2_i8", "c2_f16", "c3_i8", "c3_f16", "c4_f16",
                                  "c5_f16"])
def test_stage_lockstep(name, fused):
    """fused=False: separate add_ln / quant kernels, every stage checked on the
    GPU's own stage input.  fused=True: out-proj+LN1 / FFN1+requant / FFN2+LN2
    run as cluster row-reduction GEMMs (O16 and Y16 never exist): H1 and X_out
    are checked against the oracle's O-proj->LN1 and FFN2->LN2 from the GPU's
    ctx / I inputs."""
    cfg, w, ids, mask = build_case(name)
    enc = Encoder(cfg, w, fused=fused)
    orc = Oracle(cfg, w)
    B, S = ids.shape
    layers = range(cfg.num_layers) if cfg.num_layers <= 4 else [0, cfg.num_layers - 1]
    for l in layers:
        t = {k: f32(v) for k, v in enc.trace(dev(ids), dev(mask), l).items()}
        i8 = cfg.dtype[l] == 1
        st = lambda s_, a, b=None: orc.stage(l, s_, a, b, mask=mask, B=B, S=S)  # noqa: E731
        if fused:
            checks = [
                ("qkv", lambda: st(oracle.ST_QKV, t["x_in"]), True),
                ("ctx", lambda: st(oracle.ST_ATTN, t["qkv"]), False),
                ("h1", lambda: st(oracle.ST_LN1, st(oracle.ST_OPROJ, t["ctx"]), t["x_in"]), False),
                ("i", lambda: st(oracle.ST_FFN1, t["h1"]), cfg.act == synth.ACT_RELU),
                ("x_out", lambda: st(oracle.ST_LN2, st(oracle.ST_FFN2, t["i"]), t["h1"]), False),
            ]
        else:
            checks = [
                ("qkv", lambda: st(oracle.ST_QKV, t["x_in"]), True),
                ("ctx", lambda: st(oracle.ST_ATTN, t["qkv"]), False),
                ("o", lambda: st(oracle.ST_OPROJ, t["ctx"]), True),
                ("h1", lambda: st(oracle.ST_LN1, t["o"], t["x_in"]), False),
                ("i", lambda: st(oracle.ST_FFN1, t["h1"]), cfg.act == synth.ACT_RELU),
                ("y", lambda: st(oracle.ST_FFN2, t["i"]), True),
                ("x_out", lambda: st(oracle.ST_LN2, t["y"], t["h1"]), False),
            ]
        for key, ref_fn, exact_if_i8 in checks:
            ref = ref_fn()
            got = t[key]
            if i8 and exact_if_i8:
                nbad = int((got != ref).sum())
                assert nbad == 0, f"{name} layer {l} {key}: {nbad} elements differ (int8 stage must be bit-exact)"
            elif fused and not i8 and key in ("h1", "x_out"):
                # two composed stages whose intermediate R16(O) / R16(Y) (an
                # fp16 GEMM with fp32 accumulation) never reaches memory: the
                # LN check allows, per element, what a legitimately different
                # rounding of that intermediate can move it
                pre = "attention.output" if key == "h1" else "output"
                a_in, res = (t["ctx"], t["x_in"]) if key == "h1" else (t["i"], t["h1"])
                slack = _ln_slack_of_fp16_gemm(a_in, w[f"encoder.layer.{l}.{pre}.dense.weight"],
                                               w[f"encoder.layer.{l}.{pre}.dense.bias"], res,
                                               w[f"encoder.layer.{l}.{pre}.LayerNorm.weight"], cfg.ln_eps)
                assert_close16(got, ref, f"{name} layer {l} {key} fused", slack=slack)
            else:
                assert_close16(got, ref, f"{name} layer {l} {key} fused={fused}")


@pytest.mark.parametrize("name", ["c2_i8", "c3_i8"])
def test_gelu_epilogue_follows_oracle_rounding(name):
    """DESIGN R2: in int8 layers the FFN1 dequant is bit-exact, so the stored
    fp16 intermediate differs from the oracle's RN16(RN32(GELU_fp64(y))) only
    where the degree-11 GELU's fp32 error crosses an fp16 rounding midpoint:
    <= 2e-4 of the elements (measured 6.6e-5 on the device, 2^28 points,
    tools/micro/exp_accuracy.cu; the round-1 degree-6 fit flipped 0.2-0.4%),
    and never by more than one fp16 ulp."""
    cfg, w, ids, mask = build_case(name)
    enc = Encoder(cfg, w)
    orc = Oracle(cfg, w)
    B, S = ids.shape
    nd = tot = 0
    for l in range(cfg.num_layers):
        t = {k: f32(v) for k, v in enc.trace(dev(ids), dev(mask), l).items()}
        ref = orc.stage(l, oracle.ST_FFN1, t["h1"], None, mask=mask, B=B, S=S)
        got = t["i"]
        diff = got != ref
        ulp = np.spacing(np.abs(ref).astype(np.float16)).astype(np.float64)
        assert np.all(np.abs(got - ref)[diff] <= ulp[diff] * 1.0001 + 2.0 ** -24), f"layer {l}: > 1 ulp"
        nd += int(diff.sum())
        tot += diff.size
    assert nd <= 2e-4 * tot, f"{nd} of {tot} GELU outputs differ from the oracle's rounding"


@pytest.mark.parametrize("name", ["c1_i8", "c3_i8", "c3_f16"])
def test_fused_epilogues_match_unfused(name):
    """Same layer input -> the fused cluster epilogues reproduce the unfused
    kernels: identical FFN1 output (same epilogue math) and LN outputs that
    differ only by the order of the LN sums (rare 1-ulp flips)."""
    cfg, w, ids, mask = build_case(name)
    a = {k: f32(v) for k, v in Encoder(cfg, w, fused=True).trace(dev(ids), dev(mask), 0).items()}
    b = {k: f32(v) for k, v in Encoder(cfg, w, fused=False).trace(dev(ids), dev(mask), 0).items()}
    for k in ("x_in", "qkv", "ctx"):
        assert np.array_equal(a[k], b[k]), k
    assert_close16(a["h1"], b["h1"], f"{name} h1")


@pytest.mark.parametrize("name", ["c1_i8", "c2_i8", "c3_i8", "c3_f16"])
def test_stage_lockstep_gelu_vs_relu_ffn1(name):
    """With ReLU the int8 FFN1 stage has no transcendental: bit-exact."""
    cfg, w, ids, mask = build_case(name, act=synth.ACT_RELU)
    enc = Encoder(cfg, w)
    orc = Oracle(cfg, w)
    B, S = ids.shape
    t = {k: f32(v) for k, v in enc.trace(dev(ids), dev(mask), 0).items()}
    ref = orc.stage(0, oracle.ST_FFN1, t["h1"], mask=mask, B=B, S=S)
    if cfg.dtype[0] == 1:
        assert np.array_equal(t["i"], ref)
    else:
        assert_close16(t["i"], ref, name)


@pytest.mark.parametrize("name", ["c1_i8", "c2_i8", "c3_i8", "c3_f16", "c4_f16"])
def test_layer_lockstep(name):
    """Oracle runs a whole layer from the GPU's layer input (c4 tolerance: 1e-3 rel)."""
    cfg, w, ids, mask = build_case(name)
    enc = Encoder(cfg, w)
    orc = Oracle(cfg, w)
    B, S = ids.shape
    for l in [0, cfg.num_layers - 1]:
        t = {k: f32(v) for k, v in enc.trace(dev(ids), dev(mask), l).items()}
        x = t["x_in"]
        qkv = orc.stage(l, oracle.ST_QKV, x, mask=mask, B=B, S=S)
        ctx = orc.stage(l, oracle.ST_ATTN, qkv, mask=mask, B=B, S=S)
        o = orc.stage(l, oracle.ST_OPROJ, ctx, mask=mask, B=B, S=S)
        h1 = orc.stage(l, oracle.ST_LN1, o, x, mask=mask, B=B, S=S)
        i = orc.stage(l, oracle.ST_FFN1, h1, mask=mask, B=B, S=S)
        y = orc.stage(l, oracle.ST_FFN2, i, mask=mask, B=B, S=S)
        xo = orc.stage(l, oracle.ST_LN2, y, h1, mask=mask, B=B, S=S)
        valid = mask.reshape(-1) == 1
        got, ref = t["x_out"][valid], xo[valid]
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel <= 1e-3, f"{name} layer {l}: rel {rel}"


def _margin_ok(ref, got, margin):
    srt = np.sort(ref, axis=1)
    m = srt[:, -1] - srt[:, -2]
    keep = m > margin
    return (ref.argmax(1)[keep] == got.argmax(1)[keep]).mean() if keep.any() else 1.0


@pytest.mark.parametrize("name", ["c1_i8", "c1_f16", "c1_mixed"])
def test_end_to_end_c1(name):
    """BASELINE configs[0]: int8 <= 1e-3 relative; fp16 max-abs <= 1e-2; argmax."""
    cfg, w, ids, mask = build_case(name)
    ids, mask = synth.make_inputs(cfg, lengths=[32, 20, 7, 31])
    enc = Encoder(cfg, w)
    got = f32(enc.encode(dev(ids), dev(mask)))
    enc.check_inputs()
    ref = Oracle(cfg, w).encode(ids, mask)
    err = np.abs(got - ref).max()
    if name == "c1_i8":
        assert err <= 1e-3 * np.abs(ref).max(), err
    else:
        assert err <= 1e-2, err
    assert (got.argmax(1) == ref.argmax(1)).all()


@pytest.mark.parametrize("name,B", [("c2_i8", 8), ("c2_f16", 8), ("c3_i8", 6), ("c3_f16", 6)])
def test_end_to_end_deep_calibrated(name, B):
    """Deep models: fp16 max-abs <= 1e-2; int8 within the calibrated drift bound
    (2 x the oracle's own fp32-vs-fp64 accumulation drift, DESIGN "Tolerances")."""
    cfg, w, _, _ = build_case(name)
    cfg = cfg.with_batch(B, cfg.seq)
    ids, mask = synth.make_inputs(cfg, B=B, S=128, ragged=True, seed=99)
    enc = Encoder(cfg, w)
    got = f32(enc.encode(dev(ids), dev(mask)))
    orc = Oracle(cfg, w)
    ref = orc.encode(ids, mask)
    if cfg.dtype[0] == 0:
        assert np.abs(got - ref).max() <= 1e-2
    else:
        drift = np.abs(orc.encode(ids, mask, acc32=True) - ref).max()
        bound = max(2 * drift, 1e-3 * np.abs(ref).max())
        assert np.abs(got - ref).max() <= bound, (np.abs(got - ref).max(), drift)
    assert _margin_ok(ref, got, 2e-2) >= 0.999


@pytest.mark.parametrize("name,S", [("c4_f16", 128), ("c5_f16", 64)])
def test_end_to_end_c4_c5_fp16(name, S):
    cfg, w, _, _ = build_case(name)
    ids, mask = synth.make_inputs(cfg, B=1, S=S, ragged=False, seed=5)
    enc = Encoder(cfg, w, max_tokens=S)
    got = f32(enc.encode(dev(ids), dev(mask)))
    ref = Oracle(cfg, w).encode(ids, mask)
    assert np.abs(got - ref).max() <= 1e-2


@pytest.mark.parametrize("dt", [1, 0])
def test_padding_and_batch_invariance_on_gpu(dt):
    cfg = synth.config("c1").with_dtype(dt)
    w = synth.make_weights(cfg)
    lengths = [32, 20, 7, 31]
    ids, mask = synth.make_inputs(cfg, lengths=lengths)
    enc = Encoder(cfg, w)
    full = f32(enc.encode(dev(ids), dev(mask)))
    for b, n in enumerate(lengths):
        alone = f32(enc.encode(dev(ids[b:b + 1, :n]), dev(mask[b:b + 1, :n])))
        same_s = f32(enc.encode(dev(ids[b:b + 1]), dev(mask[b:b + 1])))
        assert np.array_equal(same_s[0], full[b]), "batch invariance"
        assert np.abs(alone[0] - full[b]).max() <= (0 if dt == 1 else 1e-3), "padding invariance"


def test_pruned_equals_zeroed_on_gpu_int8_bit_exact():
    base = synth.ModelConfig("t", 2, 128, 64, [2, 2], [256, 256], [1, 1], 1000, 64, 2, 1e-12, batch=4, seq=32)
    w = synth.make_weights(base, seed=11)
    keep_h, keep_f = [[0, 1], [1]], [list(range(256)), list(range(0, 256, 2))]
    pcfg, pw = synth.prune_slice(base, w, keep_h, keep_f)
    zw = synth.prune_zero(base, w, keep_h, keep_f)
    ids, mask = synth.make_inputs(base, lengths=[32, 20, 7, 31])
    a = f32(Encoder(pcfg, pw).encode(dev(ids), dev(mask)))
    b = f32(Encoder(base, zw).encode(dev(ids), dev(mask)))
    assert np.array_equal(a, b)
    f16cfg = base.with_dtype(0)
    a = f32(Encoder(pcfg.with_dtype(0), pw).encode(dev(ids), dev(mask)))
    b = f32(Encoder(f16cfg, zw).encode(dev(ids), dev(mask)))
    assert np.abs(a - b).max() <= 1e-3


def test_graphs_host_path_and_repeatability():
    cfg, w, ids, mask = build_case("c3_i8")
    e1 = Encoder(cfg, w)
    e2 = Encoder(cfg, w, use_graphs=False)
    a = f32(e1.encode(dev(ids), dev(mask)))
    a2 = f32(e1.encode(dev(ids), dev(mask)))
    b = f32(e2.encode(dev(ids), dev(mask)))
    h = e1.encode_host(torch.from_numpy(ids).pin_memory(), torch.from_numpy(mask).pin_memory()).numpy()
    assert np.array_equal(a, a2) and np.array_equal(a, b) and np.array_equal(a, h)


@pytest.mark.parametrize("name", ["c3_i8", "c2_i8", "c3_f16"])
def test_full_size_forward_deterministic_under_repetition(name):
    """Stress for the hand-rolled pipelines (mbarrier rings, cluster st.async
    row exchanges, TMEM hand-offs, the attention's half-row max / sum
    exchange): 30 back-to-back full-size forwards, with the L2 scrubbed in
    between to vary timing, must all give the same logits bit for bit (a race
    shows up as a run-to-run difference; compute-sanitizer is not available on
    the GPU pool)."""
    cfg = synth.config(name.split("_")[0]).with_dtype(1 if name.endswith("i8") else 0)
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, seed=11)
    enc = Encoder(cfg, w)
    ref = f32(enc.encode(dev(ids), dev(mask)))
    junk = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    for k in range(30):
        if k % 3 == 0:
            junk.fill_(k)
        got = f32(enc.encode(dev(ids), dev(mask)))
        assert np.array_equal(got, ref), (k, float(np.abs(got - ref).max()))


@pytest.mark.parametrize("name,fused", [("c1_i8", None), ("c1_i8", 0), ("c1_f16", None), ("c1_mixed", 7),
                                        ("c3_i8", None), ("c3_f16", None), ("c3_i8", 0), ("c2_i8", None),
                                        ("c4_f16", None), ("c3_full", None)])
def test_cls_last_layer_logits_bit_identical(name, fused):
    """FF_OPT_CLS_LAST_LAYER: the last layer's out-projection / LN / FFN run on
    the first-token rows only (strided A / residual / row scales, compact
    outputs); every step is row-local and the pooler reads only those rows, so
    the logits must equal the default path bit for bit (ragged masks)."""
    if name == "c3_full":  # BASELINE configs[2] at full size (B 256 x S 128)
        cfg = synth.config("c3").with_dtype(1)
        w = synth.make_weights(cfg)
        ids, mask = synth.make_inputs(cfg, seed=5)
    else:
        cfg, w, ids, mask = build_case(name)
    kw = {} if fused is None else {"fused": fused}
    ref = f32(Encoder(cfg, w, **kw).encode(dev(ids), dev(mask)))
    enc = Encoder(cfg, w, cls_last=True, **kw)
    got = f32(enc.encode(dev(ids), dev(mask)))
    assert np.array_equal(got, ref), float(np.abs(got - ref).max())
    got2 = f32(enc.encode(dev(ids), dev(mask)))  # graph replay
    assert np.array_equal(got2, ref)


@pytest.mark.parametrize("name", ["c1_i8", "c3_full", "c3_f16"])
def test_row_tile_directions_do_not_change_results(name):
    """FF_OPT_ROW_DIRS only changes the order in which the GEMM / attention
    kernels walk their row tiles (L2 locality): every direction mask gives the
    same logits bit for bit (both directions of every kernel role run)."""
    if name == "c3_full":
        cfg = synth.config("c3").with_dtype(1)
        w = synth.make_weights(cfg)
        ids, mask = synth.make_inputs(cfg, seed=9)
    else:
        cfg, w, ids, mask = build_case(name)
    enc = Encoder(cfg, w)
    assert enc.get_option(ffb.FF_OPT_ROW_DIRS) == 0b01010
    ref = f32(enc.encode(dev(ids), dev(mask)))
    for dirs in (0, 31, 0b10101, 0b01010):
        ffb.check(ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_ROW_DIRS, dirs))
        got = f32(enc.encode(dev(ids), dev(mask)))
        assert np.array_equal(got, ref), (dirs, float(np.abs(got - ref).max()))
    assert ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_ROW_DIRS, 32) != ffb.FF_OK


def test_input_errors_are_reported():
    cfg, w, ids, mask = build_case("c1_i8")
    enc = Encoder(cfg, w)
    bad = ids.copy()
    bad[1, 3] = cfg.vocab_size + 5
    enc.encode(dev(bad), dev(mask))
    with pytest.raises(FFError) as e:
        enc.check_inputs()
    assert e.value.status == FF_E_INPUT
    enc.check_inputs()  # flag cleared
    m2 = mask.copy()
    m2[2, 0] = 0
    enc.encode(dev(ids), dev(m2))
    with pytest.raises(FFError) as e:
        enc.check_inputs()
    assert e.value.status == FF_E_INPUT
    big = np.zeros((1, cfg.max_positions + 1), np.int32)
    with pytest.raises(FFError) as e:
        enc.encode(dev(big), dev(np.ones_like(big)))
    assert e.value.status == FF_E_SHAPE
    with pytest.raises(FFError) as e:
        enc.encode(dev(np.zeros((8, 32), np.int32)), dev(np.ones((8, 32), np.int32)))  # > max_tokens
    assert e.value.status == FF_E_SHAPE


def test_full_size_c3_sampled_rows_vs_oracle():
    """BASELINE configs[2] at full size (B=256, S=128, the bench launch config):
    sampled sequences recomputed by the oracle one by one (batch invariance
    makes each row independent)."""
    cfg = synth.config("c3")
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, seed=1000)
    enc = Encoder(cfg, w)
    got = f32(enc.encode(dev(ids), dev(mask)))
    assert np.isfinite(got).all()
    orc = Oracle(cfg, w)
    # 32 rows: both maxima of the 2x-drift comparison are taken over enough
    # rows to be stable (with 4-8 rows the GPU / drift ratio of the maxima
    # exceeds 2 for ~1-2% of row sets although the per-row error
    # distributions agree, tools/drift_ratio.py)
    rows = list(range(0, 256, 8))
    ref = _oracle_rows_parallel(orc, ids, mask, rows)
    drift = np.abs(_oracle_rows_parallel(orc, ids, mask, rows, acc32=True) - ref).max()
    err = np.abs(got[rows] - ref).max()
    # DESIGN "Tolerances": 6 int8 layers amplify
    # rounding-boundary flips, so the bound is 2 x the oracle's own
    # fp32-vs-fp64 accumulation drift on the same rows.
    bound = max(2 * drift, 1e-3 * np.abs(ref).max())
    assert err <= bound, (err, drift, np.abs(ref).max())
    assert _margin_ok(ref, got[rows], 2e-2) == 1.0


@pytest.mark.parametrize("dt", [1, 0])
def test_cta_pairs_equal_single_cta_at_full_size(dt):
    """The CTA-pair GEMM (cta_group::2, 256-row tiles, used at the bench size)
    and the single-CTA GEMM compute the same accumulators: identical logits."""
    cfg = synth.config("c3").with_dtype(dt)
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, seed=1000)
    a = f32(Encoder(cfg, w).encode(dev(ids), dev(mask)))
    b = f32(Encoder(cfg, w, cta_pairs=False).encode(dev(ids), dev(mask)))
    assert np.array_equal(a, b), np.abs(a - b).max()


@pytest.mark.parametrize("name,dtype", [("c1", [1, 1]), ("c1", [0, 0]), ("c1", [1, 0]), ("c3", [1] * 6)])
def test_dynamic_batching_modes_identical(name, dtype):
    """SURVEY 8(f) NEXT-1 / S:458: the CUDA path's logits do not depend on the
    batching mode (padding is inert): fixed_pad, dynamic and dynamic_sorted
    give bit-identical logits; and they match the oracle."""
    from paper_2010_13382_b200 import batching
    cfg = synth.config(name).with_dtype(dtype)
    w = synth.make_weights(cfg)
    n, bs = (13, 4) if name == "c1" else (40, 16)
    enc = Encoder(cfg, w, max_tokens=bs * cfg.seq)
    lengths = batching.ragged_lengths(n, max(1, cfg.seq // 4), cfg.seq, seed=21)
    corpus = batching.make_corpus(cfg, lengths, seed=22)

    def run(ids, mask):
        out = enc.encode(torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda())
        return out.cpu().numpy()

    ref = batching.classify(run, corpus, bs, "fixed_pad", fixed_len=cfg.seq)
    for mode, mult in [("dynamic", 1), ("dynamic_sorted", 1), ("dynamic_sorted", 8)]:
        got = batching.classify(run, corpus, bs, mode, fixed_len=cfg.seq, multiple=mult)
        np.testing.assert_array_equal(got, ref)
    if name == "c1":
        orc = oracle.Oracle(cfg, w)
        exp = batching.classify(lambda i, m: orc.encode(i, m), corpus, bs, "dynamic")
        tol = 1e-3 if all(dtype) else 1e-2
        assert np.abs(ref - exp).max() <= tol * max(1.0, np.abs(exp).max())


def _oracle_rows_parallel(orc, ids, mask, rows, **kw):
    """Oracle logits of sampled sequences, one oracle call per sequence on host threads."""
    import concurrent.futures as cf
    with cf.ThreadPoolExecutor(max_workers=len(rows)) as ex:
        outs = list(ex.map(lambda r: orc.encode(ids[r:r + 1], mask[r:r + 1], **kw), rows))
    return np.concatenate(outs, 0)


@pytest.mark.parametrize("name,rows", [("c2_i8", list(range(0, 64, 4))), ("c2_f16", [0, 21, 42, 63]),
                                       ("c3_f16", [0, 85, 170, 255]), ("c4_f16", [0, 127]), ("c5_f16", [0, 63])])
def test_full_size_sampled_rows_vs_oracle(name, rows):
    """BASELINE configs[1], [2] (fp16 variant), [3], [4] at their full sizes in
    the launch configuration the bench uses (graphs, CTA pairs, tcgen05 or
    mma.sync attention by shape): sampled sequences recomputed by the oracle
    one by one (batch invariance makes each row independent).  fp16: max-abs
    <= 1e-2 (north_star); int8: the calibrated drift bound of DESIGN §3."""
    base, dt, _, _ = CASES[name]
    cfg = base.with_dtype(dt)  # the config's own (full) batch and seq
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, seed=1000)
    enc = Encoder(cfg, w)
    got = f32(enc.encode(dev(ids), dev(mask)))
    assert np.isfinite(got).all() and got.shape[0] == cfg.batch
    orc = Oracle(cfg, w)
    ref = _oracle_rows_parallel(orc, ids, mask, rows)
    err = np.abs(got[rows] - ref).max()
    if cfg.dtype[0] == 0:
        assert err <= 1e-2, err
    else:
        drift = np.abs(_oracle_rows_parallel(orc, ids, mask, rows, acc32=True) - ref).max()
        assert err <= max(2 * drift, 1e-3 * np.abs(ref).max()), (err, drift)
    assert _margin_ok(ref, got[rows], 2e-2) == 1.0


def test_full_size_c3_ffn1_only_fusion_sampled_rows():
    """FF_OPT_FUSED_MASK 2 (separate add_ln kernels, the LN order of the
    oracle-shaped two-pass kernel) at the bench size: sampled rows within the
    same bound as the default (all-fused) path."""
    cfg = synth.config("c3")
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, seed=1000)
    got = f32(Encoder(cfg, w, fused=2).encode(dev(ids), dev(mask)))
    orc = Oracle(cfg, w)
    rows = list(range(4, 256, 16))
    ref = _oracle_rows_parallel(orc, ids, mask, rows)
    drift = np.abs(_oracle_rows_parallel(orc, ids, mask, rows, acc32=True) - ref).max()
    assert np.abs(got[rows] - ref).max() <= max(2 * drift, 1e-3 * np.abs(ref).max())
    assert _margin_ok(ref, got[rows], 2e-2) == 1.0


@pytest.mark.parametrize("name,B,S", [("c1", 4, 32), ("c2", 4, 128), ("c3", 6, 128)])
def test_per_tensor_u8_activations_vs_oracle(name, B, S):
    """NEXT-2 (DESIGN R22): per-tensor u8 activations with a zero point,
    u8 x s8 tcgen05 GEMMs + exact zp * colsum correction, against the oracle
    running the same quantizer (whole-batch statistics, so the whole batch is
    compared); the drift bound of DESIGN §3."""
    cfg = synth.config(name).with_dtype(1).with_batch(B, S)
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, B=B, S=S, ragged=True, seed=123)
    enc = Encoder(cfg, w, act_quant=1)
    got = f32(enc.encode(dev(ids), dev(mask)))
    orc = Oracle(cfg, w, act_quant=1)
    ref = orc.encode(ids, mask)
    drift = np.abs(orc.encode(ids, mask, acc32=True) - ref).max()
    err = np.abs(got - ref).max()
    assert err <= max(2 * drift, 1e-3 * np.abs(ref).max()), (err, drift)
    assert _margin_ok(ref, got, 2e-2) >= 0.999
    # a genuinely different quantizer from the per-row default
    row = f32(Encoder(cfg, w).encode(dev(ids), dev(mask)))
    assert not np.array_equal(row, got)
    assert enc.launch_count(B, S) == 3 + cfg.num_layers * 15


def test_per_tensor_quantizer_kernel_bit_exact():
    """The per-tensor u8 quantizer kernels (min/max reduction + quantize)
    reproduce the oracle's Q8tensor bit for bit through the model's first
    GEMM input: the u8 tensor is not exported, so compare the layer-0 stage
    through the trace (QKV output) with the oracle stage run on the GPU's own
    layer input."""
    cfg = synth.config("c1").with_dtype([1, 1])
    w = synth.make_weights(cfg)
    B, S = cfg.batch, cfg.seq
    ids, mask = synth.make_inputs(cfg, B=B, S=S, ragged=True, seed=5)
    enc = Encoder(cfg, w, act_quant=1)
    dumps = enc.trace(dev(ids), dev(mask), 0)
    orc = Oracle(cfg, w, act_quant=1)
    x_in = f32(dumps["x_in"])
    qkv_ref = orc.stage(0, oracle.ST_QKV, x_in)
    # same u8 tensor, same scale / zero point, exact int32 accumulation and
    # correction, the same fp32 fma epilogue: bit-identical fp16 outputs
    np.testing.assert_array_equal(f32(dumps["qkv"]), qkv_ref)


@pytest.mark.parametrize("name,B,S", [("c1", 4, 32), ("c2", 16, 128), ("c3", 256, 128)])
def test_ffn1_fusion_bit_identical_to_separate_kernels(name, B, S):
    """FF_OPT_FUSED_MASK = 2 (FFN1 + GELU + per-row requant in one
    cluster row-reduction GEMM) computes Q8row from the same R16 values as the
    separate quant_rows kernel (R12), so the logits are bit-identical to the
    fully unfused path (mask 0), which the lockstep tests check stage by stage."""
    cfg = synth.config(name).with_dtype(1).with_batch(B, S)
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, B=B, S=S, ragged=True, seed=77)
    fused = Encoder(cfg, w, fused=2)
    n_fused, n_sep = fused.launch_count(B, S), Encoder(cfg, w, fused=False).launch_count(B, S)
    fusable = cfg.ffn_dim[0] % 256 == 0  # row = 256 x 1..8 columns (C2's F' = 1200 is not)
    assert (n_fused < n_sep) if fusable else (n_fused == n_sep)
    a = fused.encode(dev(ids), dev(mask)).cpu()
    b = Encoder(cfg, w, fused=False).encode(dev(ids), dev(mask)).cpu()
    assert torch.equal(a, b)


def test_encode_host_async_matches_sync():
    """ff_encode_host_async (no per-call sync, stream-ordered workspace reuse)
    returns the same logits as ff_encode_host for several batches in flight."""
    cfg = synth.config("c1").with_dtype(1)
    w = synth.make_weights(cfg)
    enc = Encoder(cfg, w)
    batches = [synth.make_inputs(cfg, seed=700 + k, ragged=True) for k in range(4)]
    host = [(torch.from_numpy(i).pin_memory(), torch.from_numpy(m).pin_memory()) for i, m in batches]
    outs = [torch.empty((cfg.batch, cfg.num_classes), dtype=torch.float32).pin_memory() for _ in batches]
    for (i, m), o in zip(host, outs):
        enc.encode_host_async(i, m, o)
    torch.cuda.synchronize()
    for (i, m), o in zip(host, outs):
        assert torch.equal(o, enc.encode_host(i, m))


@pytest.mark.parametrize("mask_bits", [1, 3, 4, 5, 6, 7])
def test_every_fusion_mask_within_drift_bound(mask_bits):
    """FF_OPT_FUSED_MASK combinations with a LayerNorm fusion (the LN sums run in
    another order): C3-shaped int8 logits (B 16, ragged) within the
    DESIGN §3 drift bound of the oracle, like the default path."""
    cfg = synth.config("c3").with_dtype(1).with_batch(16, 128)
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, B=16, S=128, ragged=True, seed=55)
    got = f32(Encoder(cfg, w, fused=mask_bits).encode(dev(ids), dev(mask)))
    orc = Oracle(cfg, w)
    rows = list(range(16))
    ref = _oracle_rows_parallel(orc, ids, mask, rows)
    drift = np.abs(_oracle_rows_parallel(orc, ids, mask, rows, acc32=True) - ref).max()
    assert np.abs(got[rows] - ref).max() <= max(2 * drift, 1e-3 * np.abs(ref).max())
    assert (got[rows].argmax(1) == ref.argmax(1)).all() or _margin_ok(ref, got[rows], 2e-2) == 1.0
