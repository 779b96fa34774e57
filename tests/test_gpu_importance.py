"""GPU parity of the importance scorer (C-ABI ff_score_batch; SURVEY 8(f)
NEXT-3) against the fp64 oracle (oracle/importance.py).

Tolerance: the scorer runs fp32 end to end; a score is a sum over
B*S tokens of products of forward activations and back-propagated gradients,
so its fp32-vs-fp64 error is relative to the layer's score scale, not to the
(possibly cancelling) score itself: |gpu - ref| <= 1e-4 |ref| + 2e-5 max_l(ref)
(measured, tools/importance_err.py: <= 2.2e-6 of the layer max on all three
configs with the SIMT linears, so the bound has ~10x headroom).  The default
linears are 3xFP16 on tcgen05 (gemm_x3.cu: row-scaled fp16 hi / lo splits,
per-product error <= ~2^-21 relative, fp32 accumulation in TMEM in 128-wide
K chunks summed with IEEE adds); every parity test runs both paths against the
same oracle and the same bound."""
import numpy as np
import pytest

from oracle import importance as imp
from paper_2010_13382_b200 import fastformers as ffb
from paper_2010_13382_b200 import pruning, synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _batch(cfg, B, S, seed, ragged=True):
    rng = np.random.default_rng(seed)
    ids = rng.integers(5, cfg.vocab_size, (B, S)).astype(np.int32)
    ids[:, 0] = cfg.cls_id
    mask = np.ones((B, S), np.int32)
    if ragged:
        for b in range(B):
            mask[b, rng.integers(max(1, S // 4), S + 1):] = 0
    labels = rng.integers(0, cfg.num_classes, B).astype(np.int32)
    return ids, mask, labels


def _cuda(*arrs):
    return [torch.from_numpy(a).cuda() for a in arrs]


def _close(gpu, ref):
    for l, (g, r) in enumerate(zip(gpu, ref)):
        tol = 1e-4 * np.abs(r) + 2e-5 * np.abs(r).max()
        bad = np.abs(g - r) > tol
        assert not bad.any(), (l, np.abs(g - r).max(), np.abs(r).max(), int(bad.sum()))


def _tiny():
    return synth.ModelConfig("tiny_score", 2, 32, 8, [4, 3], [16, 12], [0, 0], 50, 16, 3, 1e-12, batch=3, seq=7,
                             cls_id=1)


CONFIGS = [
    ("tiny", _tiny, 3, 7, 0.3),
    ("c2_shape", lambda: synth.config("c2"), 8, 64, 0.02),               # TinyBERT 4L/312/12 heads d=26/1200
    ("c3_unpruned", lambda: synth.config("c3_unpruned"), 4, 64, 0.02),   # distilroberta 6L/768/12/3072
]


@pytest.mark.parametrize("tc", [True, False], ids=["tc_x3", "simt"])
@pytest.mark.parametrize("name,mk,B,S,std", CONFIGS)
def test_scores_match_oracle(name, mk, B, S, std, tc):
    cfg = mk()
    w = synth.make_weights(cfg, std=std)
    batches = [_batch(cfg, B, S, 100 + i) for i in range(2)]
    sc = ffb.Scorer(cfg, w, max_tokens=B * S, tc_linears=tc)
    losses = []
    for ids, mask, labels in batches:
        lg = torch.empty((B, cfg.num_classes), dtype=torch.float32, device="cuda")
        loss = sc.score(*_cuda(ids, mask, labels), logits=lg)
        losses.append(float(loss.item()))
        ref_loss, ref_logits, _, _ = imp.forward_backward(cfg, w, ids, mask, labels)
        assert abs(losses[-1] - ref_loss) <= 1e-5 * max(1.0, abs(ref_loss))
        np.testing.assert_allclose(lg.cpu().numpy(), ref_logits, rtol=0, atol=1e-4)
    hs, fs = sc.scores()
    rh, rf, _ = imp.compute_importance(cfg, w, batches)
    _close(hs, rh)
    _close(fs, rf)


def test_dead_head_exactly_zero_and_padding_inert():
    cfg = synth.config("c2")
    w = synth.make_weights(cfg)
    d = cfg.head_dim
    w["encoder.layer.1.attention.output.dense.weight"][:, 5 * d:6 * d] = 0.0
    ids, mask, labels = _batch(cfg, 6, 48, 7)
    sc = ffb.Scorer(cfg, w, max_tokens=6 * 64)
    sc.score(*_cuda(ids, mask, labels))
    hs, fs = sc.scores()
    assert hs[1][5] == 0.0 and (np.delete(hs[1], 5) > 0).all()
    # the same sequences padded to S = 64: same scores up to fp32 reduction order
    ids2 = np.concatenate([ids, np.full((6, 16), 9, np.int32)], axis=1)
    mask2 = np.concatenate([mask, np.zeros((6, 16), np.int32)], axis=1)
    sc.reset()
    sc.score(*_cuda(ids2, mask2, labels))
    hs2, fs2 = sc.scores()
    _close(hs2, hs)
    _close(fs2, fs)


def test_selection_from_gpu_scores_matches_oracle():
    """Top-k per layer (R25) from GPU scores equals the oracle's, for
    units whose score is not within the fp32 tolerance of the k-th boundary."""
    cfg = synth.config("c2")
    w = synth.make_weights(cfg)
    batches = [_batch(cfg, 8, 64, 300 + i) for i in range(2)]
    sc = ffb.Scorer(cfg, w, max_tokens=8 * 64)
    for b in batches:
        sc.score(*_cuda(*b))
    hs, fs = sc.scores()
    rh, rf, _ = imp.compute_importance(cfg, w, batches)
    for gs, rs, keep in ((hs, rh, 6), (fs, rf, 600)):
        for l in range(cfg.num_layers):
            kept_gpu = set(pruning.select_keep(gs[l], keep))
            kept_ref = set(imp.select_keep(rs[l], keep))
            kth = np.sort(rs[l])[::-1][keep - 1]
            near = {i for i in range(len(rs[l])) if abs(rs[l][i] - kth) <= 1e-4 * kth + 2e-5 * rs[l].max()}
            assert kept_gpu - near == kept_ref - near, l


def test_score_prune_reconnect_encode_end_to_end():
    """P:93 end to end on the GPU: score the unpruned distilroberta shape
    (ff_score_batch), keep 8 of 12 heads and 1536 of 3072 FFN units per layer
    (pruning.prune: the C3 geometry), build the pruned int8 encoder from
    the reconnected weights and check its logits against the C++ oracle of the
    same pruned model (DESIGN §3 drift bound)."""
    import oracle
    cfg = synth.config("c3_unpruned").with_dtype(1)
    w = synth.make_weights(cfg)
    sc = ffb.Scorer(cfg, w, max_tokens=8 * 64)
    for i in range(2):
        sc.score(*_cuda(*_batch(cfg, 8, 64, 900 + i)))
    hs, fs = sc.scores()
    pcfg, pw, kept_h, kept_f = pruning.prune(cfg, w, hs, fs, head_ratio=8 / 12, ffn_ratio=0.5)
    assert pcfg.heads == [8] * 6 and pcfg.ffn_dim == [1536] * 6
    assert all(len(set(k)) == len(k) for k in kept_h + kept_f)
    ids, mask, _ = _batch(pcfg, 6, 128, 950)
    got = ffb.Encoder(pcfg, pw).encode(*_cuda(ids, mask)).cpu().numpy()
    orc = oracle.Oracle(pcfg, pw)
    ref = orc.encode(ids, mask)
    drift = np.abs(orc.encode(ids, mask, acc32=True) - ref).max()
    assert np.abs(got - ref).max() <= max(2 * drift, 1e-3 * np.abs(ref).max())


def test_scorer_flags_invalid_inputs_without_faulting():
    """Token ids outside [0, V), mask[b, 0] = 0 and labels outside [0, C) are
    read as 0 (no out-of-bounds access) and reported by ff_scorer_check."""
    cfg = _tiny()
    w = synth.make_weights(cfg, std=0.3)
    sc = ffb.Scorer(cfg, w, max_tokens=3 * 7)
    ids, mask, labels = _batch(cfg, 3, 7, 5)
    sc.score(*_cuda(ids, mask, labels))
    sc.check_inputs()  # clean batch: no error
    for bad in ("id", "mask", "label"):
        i2, m2, l2 = ids.copy(), mask.copy(), labels.copy()
        if bad == "id":
            i2[1, 2] = cfg.vocab_size + 7
        elif bad == "mask":
            m2[2, 0] = 0
        else:
            l2[0] = cfg.num_classes
        sc.score(*_cuda(i2, m2, l2))
        with pytest.raises(ffb.FFError) as e:
            sc.check_inputs()
        assert e.value.status == ffb.FF_E_INPUT
        sc.check_inputs()  # the flag was cleared


def test_tc_linears_match_simt_linears_on_ragged_tails():
    """The 3xFP16 tcgen05 linears against the SIMT fp32 SGEMM on a shape with
    ragged M / N / K tails in every linear (H = 50: K not a multiple of 4;
    D = 3 x 12, F = 70 / 130: N tails; M = 5 x 29 = 145 rows: an M tail), two
    batches accumulating: scores, loss and logits agree at fp32 level."""
    cfg = synth.ModelConfig("tails", 2, 50, 12, [3, 5], [70, 130], [0, 0], 61, 40, 3, 1e-12, batch=5, seq=29,
                            cls_id=1)
    w = synth.make_weights(cfg, std=0.1)
    batches = [_batch(cfg, 5, 29, 40 + i) for i in range(2)]
    out = []
    for tc in (True, False):
        sc = ffb.Scorer(cfg, w, max_tokens=5 * 29, tc_linears=tc)
        lg = torch.empty((5, cfg.num_classes), dtype=torch.float32, device="cuda")
        losses = [float(sc.score(*_cuda(*b), logits=lg).item()) for b in batches]
        out.append((sc.scores(), losses, lg.cpu().numpy()))
    (hs_t, fs_t), loss_t, lg_t = out[0]
    (hs_s, fs_s), loss_s, lg_s = out[1]
    np.testing.assert_allclose(loss_t, loss_s, rtol=1e-5)
    np.testing.assert_allclose(lg_t, lg_s, rtol=0, atol=1e-5)
    _close(hs_t, hs_s)
    _close(fs_t, fs_s)
    rh, rf, _ = imp.compute_importance(cfg, w, batches)
    _close(hs_t, rh)
    _close(fs_t, rf)


def test_reload_after_finalize_requires_finalize():
    """Loading a tensor after ff_scorer_finalize invalidates the weight splits:
    ff_score_batch refuses (FF_E_STATE) until finalize runs again."""
    import ctypes
    cfg = _tiny()
    w = synth.make_weights(cfg)
    sc = ffb.Scorer(cfg, w, max_tokens=3 * 7)
    L = ffb.lib()
    name = "encoder.layer.0.intermediate.dense.weight"
    a = np.ascontiguousarray(w[name] * 2, dtype=np.float32)
    shape = (ctypes.c_int64 * 2)(*a.shape)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert L.ff_scorer_load_weights(sc.h, name.encode(), ctypes.c_void_p(a.ctypes.data), shape, 2, st) == 0
    ids, mask, labels = _cuda(*_batch(cfg, 3, 7, 5))
    with pytest.raises(ffb.FFError, match="FF_E_STATE"):
        sc.score(ids, mask, labels)
    assert L.ff_scorer_finalize(sc.h, st) == 0
    sc.score(ids, mask, labels)
    w2 = dict(w)
    w2[name] = a
    ref = ffb.Scorer(cfg, w2, max_tokens=3 * 7)
    ref.score(ids, mask, labels)
    torch.cuda.synchronize()
    for g, r in zip(sc.scores(), ref.scores()):
        for x, y in zip(g, r):
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (300, 200, 100), (1, 5, 3), (257, 130, 3072), (4096, 768, 3072)])
def test_gemm_x3_against_fp64(M, N, K):
    """The scorer's 3xFP16 tcgen05 GEMM (ff_debug_gemm_x3) against an fp64
    matmul of the same fp32 inputs: the error is bounded by fp32-level terms,
    |err| <= 2^-20 * sum_k |a_ik b_jk| + 2^-24 |c| (3 products of 11-bit
    halves, ~2^-21 relative each; chunked IEEE accumulation), and within 16x the error of a
    plain fp32 torch matmul (TF32 disabled) on the same inputs."""
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g, dtype=torch.float64)
    B = torch.randn(N, K, generator=g, dtype=torch.float64) * 0.05
    bias = torch.randn(N, generator=g, dtype=torch.float64)
    ref = A @ B.T + bias
    A32, B32, b32 = (t.float().cuda() for t in (A, B, bias))
    got = ffb.gemm_x3(A32, B32, bias=b32).double().cpu()
    bound = 2.0 ** -20 * (A.abs() @ B.abs().T) + 2.0 ** -24 * ref.abs()
    err = (got - ref).abs()
    assert (err <= bound).all(), float((err / bound).max())
    torch.backends.cuda.matmul.allow_tf32 = False
    fp32 = (A32 @ B32.T + b32).double().cpu()
    e32 = (fp32 - ref).abs()
    print("max abs err x3 %.3e fp32 %.3e" % (float(err.max()), float(e32.max())))
    assert err.max() <= 16 * e32.max() + 1e-12, (float(err.max()), float(e32.max()))
    # accumulate: C += A B^T
    c0 = torch.randn(M, N, generator=g, dtype=torch.float64)
    out = c0.float().cuda()
    ffb.gemm_x3(A32, B32, out=out, accumulate=True)
    ref2 = c0.float().double() + A @ B.T
    assert ((out.double().cpu() - ref2).abs() <= bound + 2.0 ** -23 * ref2.abs()).all()


def test_gemm_x3_chunking_reduces_error():
    """One TMEM accumulator over the whole K (kc = K / 64) is less accurate
    than the default 128-wide chunks summed with IEEE adds (the design reason
    for chunking, gemm_x3.cu); both stay within the fp32-level bound's 4x."""
    g = torch.Generator().manual_seed(5)
    M, N, K = 512, 256, 3072
    A = torch.randn(M, K, generator=g, dtype=torch.float64).abs()  # same-sign terms: biased rounding shows
    B = torch.randn(N, K, generator=g, dtype=torch.float64).abs() * 0.05
    ref = A @ B.T
    A32, B32 = A.float().cuda(), B.float().cuda()
    e_chunk = (ffb.gemm_x3(A32, B32, kc=2).double().cpu() - ref).abs().max()
    e_whole = (ffb.gemm_x3(A32, B32, kc=K // 64).double().cpu() - ref).abs().max()
    print("max abs err chunked %.3e whole-K %.3e" % (e_chunk, e_whole))
    assert e_chunk <= e_whole


def test_gemm_x3_row_scaling_handles_wide_dynamic_range():
    """Rows of very different magnitude (1e-30 .. 1e30, and an all-zero row)
    keep fp32-level relative accuracy: each operand row is scaled by its own
    power of two before the fp16 split (gemm_x3.cu)."""
    g = torch.Generator().manual_seed(11)
    M, N, K = 130, 70, 200
    A = torch.randn(M, K, generator=g, dtype=torch.float64)
    A *= torch.logspace(-30, 30, M, dtype=torch.float64)[:, None]
    A[7] = 0.0
    B = torch.randn(N, K, generator=g, dtype=torch.float64) * torch.logspace(-5, 5, N, dtype=torch.float64)[:, None]
    A32, B32 = A.float(), B.float()
    ref = A32.double() @ B32.double().T
    got = ffb.gemm_x3(A32.cuda(), B32.cuda()).double().cpu()
    bound = 2.0 ** -20 * (A32.double().abs() @ B32.double().abs().T)
    assert ((got - ref).abs() <= bound).all()
    assert (got[7] == 0).all()
