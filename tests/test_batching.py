"""Dynamic sequence-length batching (SPEC S:420-428,
S:458).  Host planning logic and, through the oracle, the property the
speed-up rests on: padding is inert, so logits do not depend on the batching
mode."""
import numpy as np
import pytest

import oracle
from paper_2010_13382_b200 import batching, synth


def test_spec_examples():
    # lengths [5,3,8], batch_size 3, dynamic -> one batch, S_b = 8
    b = batching.make_batches([5, 3, 8], 3, "dynamic")
    assert len(b) == 1 and b[0].seq == 8 and list(b[0].index) == [0, 1, 2]
    # dynamic_sorted on [8,1,8,1], batch_size 2 -> S_b 1 and 8; order restored
    b = batching.make_batches([8, 1, 8, 1], 2, "dynamic_sorted")
    assert [x.seq for x in b] == [1, 8]
    assert sorted(b[0].index) == [1, 3] and sorted(b[1].index) == [0, 2]
    outs = [np.array([[i] for i in x.index], np.float32) for x in b]
    np.testing.assert_array_equal(batching.unmap(b, outs, 4)[:, 0], [0, 1, 2, 3])


@pytest.mark.parametrize("mode", batching.MODES)
@pytest.mark.parametrize("multiple", [1, 8])
def test_plan_properties(mode, multiple):
    rng = np.random.default_rng(7)
    lengths = rng.integers(1, 129, 203)
    b = batching.make_batches(lengths, 16, mode, fixed_len=128, multiple=multiple)
    idx = np.concatenate([x.index for x in b])
    assert sorted(idx) == list(range(len(lengths)))              # every sequence exactly once
    assert all(len(x.index) <= 16 for x in b)
    for x in b:
        assert x.seq >= lengths[x.index].max() and x.seq <= 128  # covers its longest member
        if mode == "fixed_pad":
            assert x.seq == 128
        else:
            assert x.seq < lengths[x.index].max() + multiple     # no more padding than the bucket
            assert x.seq % multiple == 0 or x.seq == 128
    if mode == "dynamic":
        np.testing.assert_array_equal(idx, np.arange(len(lengths)))
    if mode == "dynamic_sorted":
        assert (np.diff(lengths[idx]) >= 0).all()
        np.testing.assert_array_equal(idx, np.argsort(lengths, kind="stable"))


def test_invalid():
    with pytest.raises(ValueError):
        batching.make_batches([3, 4], 2, "fixed_pad", fixed_len=3)
    with pytest.raises(ValueError):
        batching.make_batches([3, 0], 2, "dynamic")
    with pytest.raises(ValueError):
        batching.make_batches([3], 2, "bogus")


def test_pack():
    corpus = [np.array([101, 7, 8], np.int32), np.array([101, 9], np.int32)]
    ids, mask = batching.pack(corpus, batching.Batch(index=np.array([1, 0]), seq=4))
    np.testing.assert_array_equal(ids, [[101, 9, 1, 1], [101, 7, 8, 1]])
    np.testing.assert_array_equal(mask, [[1, 1, 0, 0], [1, 1, 1, 0]])


def test_mac_ratio_is_exact_arithmetic():
    # S:454 / S:566: the dynamic/fixed MAC ratio is integer arithmetic on the
    # padded shapes: brute force over the per-sequence formula
    cfg = synth.config("c3")
    lengths = batching.ragged_lengths(300, 8, 128, seed=3)
    for mode in batching.MODES:
        b = batching.make_batches(lengths, 32, mode, fixed_len=128)
        brute = 0
        for x in b:
            for _ in x.index:
                S = x.seq
                for A, F in zip(cfg.heads, cfg.ffn_dim):
                    D = A * cfg.head_dim
                    brute += S * (cfg.hidden * 3 * D + D * cfg.hidden + 2 * cfg.hidden * F) + 2 * A * S * S * cfg.head_dim
                brute += cfg.hidden * cfg.hidden + cfg.hidden * cfg.num_classes
        assert batching.macs(cfg, b) == brute
    fixed = batching.macs(cfg, batching.make_batches(lengths, 32, "fixed_pad", fixed_len=128))
    srt = batching.macs(cfg, batching.make_batches(lengths, 32, "dynamic_sorted"))
    assert srt < fixed  # sorting removes padding work


@pytest.mark.parametrize("dtype", [[1, 1], [0, 0], [1, 0]])
def test_logits_independent_of_batching_oracle(dtype):
    """logits under dynamic modes equal those under fixed_pad (padding
    inert) — in the oracle's emulation mode the equality is exact."""
    cfg = synth.config("c1").with_dtype(dtype)
    orc = oracle.Oracle(cfg, synth.make_weights(cfg))
    lengths = batching.ragged_lengths(11, 1, cfg.seq, seed=5)
    corpus = batching.make_corpus(cfg, lengths, seed=9)
    enc = lambda ids, mask: orc.encode(ids, mask)
    ref = batching.classify(enc, corpus, 4, "fixed_pad", fixed_len=cfg.seq)
    for mode in ("dynamic", "dynamic_sorted"):
        got = batching.classify(enc, corpus, 4, mode)
        np.testing.assert_array_equal(got, ref)
    # and one sequence alone, unpadded
    one = orc.encode(corpus[3][None, :], np.ones((1, len(corpus[3])), np.int32))
    np.testing.assert_array_equal(one[0], ref[3])
