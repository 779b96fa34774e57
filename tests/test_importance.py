"""Pins of the importance-scoring oracle (
DESIGN R23-R25) against what the paper and the mathematics fix, plus the
host-side selection / reconnection logic of the product (pruning.py)."""
import dataclasses

import numpy as np
import pytest

import oracle
from oracle import importance as imp
from paper_2010_13382_b200 import pruning, synth


def tiny(act=synth.ACT_GELU):
    return synth.ModelConfig("tiny_score", 2, 32, 8, [4, 3], [16, 12], [0, 0], 50, 16, 3, 1e-12, act=act,
                             batch=3, seq=7, cls_id=1)


def batch(cfg, seed=3, lengths=(7, 4, 2)):
    rng = np.random.default_rng(seed)
    B, S = len(lengths), max(lengths)
    ids = rng.integers(2, cfg.vocab_size, (B, S)).astype(np.int32)
    mask = np.zeros((B, S), np.int32)
    for b, n in enumerate(lengths):
        mask[b, :n] = 1
    labels = rng.integers(0, cfg.num_classes, B).astype(np.int32)
    return ids, mask, labels


def weights(cfg, seed=1234):
    w = synth.make_weights(cfg, seed=seed, std=0.3)  # larger weights: gradients well away from 0
    return w


@pytest.mark.parametrize("act", [synth.ACT_GELU, synth.ACT_GELU_TANH])
def test_mask_gradients_match_central_differences(act):
    """scores match finite differences (here every mask variable, fp64)."""
    cfg = tiny(act)
    w = weights(cfg)
    ids, mask, labels = batch(cfg)
    loss, _, dxi, dnu = imp.forward_backward(cfg, w, ids, mask, labels)
    eps = 1e-6
    for l in range(cfg.num_layers):
        for kind, n, g in (("xi", cfg.heads[l], dxi[l]), ("nu", cfg.ffn_dim[l], dnu[l])):
            for u in range(n):
                def f(delta):
                    xi = [np.ones(a) for a in cfg.heads]
                    nu = [np.ones(f_) for f_ in cfg.ffn_dim]
                    (xi if kind == "xi" else nu)[l][u] += delta
                    return imp.loss_only(cfg, w, ids, mask, labels, xi, nu)
                fd = (f(eps) - f(-eps)) / (2 * eps)
                assert abs(fd - g[u]) <= 1e-7 + 1e-5 * abs(fd), (kind, l, u, fd, g[u])


def test_forward_equals_cpp_oracle_ref64():
    """The scorer's forward is the encoder the C++ oracle defines (ref64 mode)."""
    cfg = tiny()
    w = weights(cfg)
    ids, mask, labels = batch(cfg)
    _, logits, _, _ = imp.forward_backward(cfg, w, ids, mask, labels)
    ref = oracle.Oracle(cfg, w).encode(ids, mask, mode=oracle.MODE_REF64, fp64_logits=True)
    np.testing.assert_allclose(logits, ref, rtol=0, atol=1e-10)


def test_dead_head_scores_exactly_zero():
    """a head whose output-projection columns are zero has score 0."""
    cfg = tiny()
    w = weights(cfg)
    d = cfg.head_dim
    w["encoder.layer.0.attention.output.dense.weight"][:, 2 * d:3 * d] = 0.0
    hs, fs, _ = imp.compute_importance(cfg, w, [batch(cfg, 1), batch(cfg, 2)])
    assert hs[0][2] == 0.0
    assert all(s > 0 for s in hs[0][:2]) and hs[1].min() > 0


def test_identical_heads_score_equally():
    """duplicated head weights -> equal scores."""
    cfg = tiny()
    w = weights(cfg)
    d = cfg.head_dim
    p = "encoder.layer.1.attention."
    for n in ("query", "key", "value"):
        w[p + f"self.{n}.weight"][d:2 * d] = w[p + f"self.{n}.weight"][0:d]
        w[p + f"self.{n}.bias"][d:2 * d] = w[p + f"self.{n}.bias"][0:d]
    w[p + "output.dense.weight"][:, d:2 * d] = w[p + "output.dense.weight"][:, 0:d]
    hs, _, _ = imp.compute_importance(cfg, w, [batch(cfg, 5)])
    assert abs(hs[1][0] - hs[1][1]) <= 1e-12 * max(hs[1][0], 1e-30)


def test_padding_does_not_change_scores():
    """Padded positions carry no gradient: appending padding leaves the scores unchanged."""
    cfg = tiny()
    w = weights(cfg)
    ids, mask, labels = batch(cfg, 9, lengths=(5, 3, 4))
    ids2 = np.concatenate([ids, np.full((3, 2), 7, np.int32)], axis=1)
    mask2 = np.concatenate([mask, np.zeros((3, 2), np.int32)], axis=1)
    a = imp.forward_backward(cfg, w, ids, mask, labels)
    b = imp.forward_backward(cfg, w, ids2, mask2, labels)
    for l in range(cfg.num_layers):
        np.testing.assert_allclose(a[2][l], b[2][l], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(a[3][l], b[3][l], rtol=1e-12, atol=1e-15)


def test_select_keep_spec_examples():
    """SPEC S:330-333 (oracle and the product's host selection)."""
    for sel in (imp.select_keep, pruning.select_keep):
        assert sel([3, 1, 2, 5], 2) == [0, 3]
        assert sel([2, 2, 1], 2) == [0, 1]
        assert sel([0.5, 0.1, 0.9], 3) == [0, 1, 2]


def test_pruned_model_equals_masked_model():
    """P:93 reconnection: slicing away units == zeroing their mask variables
    (loss and logits), and the product's prune keeps max(1, floor(n r)) per layer."""
    cfg = tiny()
    w = weights(cfg)
    ids, mask, labels = batch(cfg, 11)
    hs, fs, _ = imp.compute_importance(cfg, w, [batch(cfg, 12), batch(cfg, 13)])
    pcfg, pw, kept_h, kept_f = pruning.prune(cfg, w, hs, fs, head_ratio=0.5, ffn_ratio=0.5)
    assert pcfg.heads == [2, 1] and pcfg.ffn_dim == [8, 6]
    xi = [np.isin(np.arange(cfg.heads[l]), kept_h[l]).astype(float) for l in range(cfg.num_layers)]
    nu = [np.isin(np.arange(cfg.ffn_dim[l]), kept_f[l]).astype(float) for l in range(cfg.num_layers)]
    la, loga, _, _ = imp.forward_backward(cfg, w, ids, mask, labels, xi, nu)
    lb, logb, _, _ = imp.forward_backward(pcfg, pw, ids, mask, labels)
    assert abs(la - lb) <= 1e-12
    np.testing.assert_allclose(loga, logb, rtol=0, atol=1e-12)
    for l in range(cfg.num_layers):
        assert kept_h[l] == imp.select_keep(hs[l], pcfg.heads[l])
        assert kept_f[l] == imp.select_keep(fs[l], pcfg.ffn_dim[l])
