"""Dynamic sequence-length batching.

The paper's largest non-model speed-up: "We modify the batch generation to
support dynamic sequence length for each batch" (Table 3 "+ dynamic
sequence length" 3.51x).  Instead of padding every request to
a fixed maximum, each batch is padded only to its own longest sequence;
`dynamic_sorted` first sorts the corpus by length (stable), so neighbours in a
batch have similar lengths, and restores the input order of the outputs.

Host-side batch planning only: every forward runs in the CUDA library.  Padded
positions are inert in the encoder (masked keys get probability exactly 0,
every per-token computation is row-local, per-row int8 scales), so a
sequence's logits do not depend on how it is batched or padded — the tests
check that bit for bit.

Modes:
  fixed_pad       pad every batch to `fixed_len`, input order
  dynamic         input order, each batch padded to its own max length
  dynamic_sorted  stable sort by length, batch, pad to own max; outputs unmapped
`multiple` rounds each batch length up (e.g. 8): length buckets, so a CUDA-graph
cache sees few distinct shapes.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

MODES = ("fixed_pad", "dynamic", "dynamic_sorted")


@dataclass
class Batch:
    index: np.ndarray  # positions of the batch's sequences in the input corpus
    seq: int           # padded length S_b


def make_batches(lengths: Sequence[int], batch_size: int, mode: str, fixed_len: int = None,
                 multiple: int = 1) -> List[Batch]:
    """Plan the batches of a corpus with the given sequence lengths."""
    lengths = np.asarray(lengths, dtype=np.int64)
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    if batch_size < 1 or (lengths < 1).any():
        raise ValueError("batch_size and every length must be >= 1")
    n = len(lengths)
    if mode == "fixed_pad":
        if fixed_len is None or fixed_len < lengths.max(initial=1):
            raise ValueError("fixed_pad needs fixed_len >= the longest sequence")
    order = np.argsort(lengths, kind="stable") if mode == "dynamic_sorted" else np.arange(n)
    batches = []
    for s in range(0, n, batch_size):
        idx = order[s:s + batch_size]
        if mode == "fixed_pad":
            sb = int(fixed_len)
        else:
            sb = int(lengths[idx].max())
            sb = -(-sb // multiple) * multiple
            if fixed_len is not None:
                sb = min(sb, int(fixed_len))
        batches.append(Batch(index=idx, seq=sb))
    return batches


def pack(corpus: Sequence[np.ndarray], batch: Batch):
    """int32 ids / mask [B, S_b] of one batch (pad id 1, mask 0 on padding)."""
    B = len(batch.index)
    ids = np.ones((B, batch.seq), np.int32)
    mask = np.zeros((B, batch.seq), np.int32)
    for r, i in enumerate(batch.index):
        seq = corpus[i]
        ids[r, :len(seq)] = seq
        mask[r, :len(seq)] = 1
    return ids, mask


def unmap(batches: List[Batch], outputs: List[np.ndarray], n: int) -> np.ndarray:
    """Per-batch outputs [B_b, C] -> [n, C] in the corpus's input order."""
    C = outputs[0].shape[1]
    res = np.empty((n, C), outputs[0].dtype)
    for b, o in zip(batches, outputs):
        res[b.index] = o
    return res


def padded_tokens(batches: List[Batch]) -> int:
    return int(sum(len(b.index) * b.seq for b in batches))


def macs(cfg, batches: List[Batch]) -> int:
    """Multiply-accumulates of the padded work (SPEC S:432 `count_macs` with the
    pruned widths): per batch of B sequences of S_b tokens,
    B * sum_l S_b (H 3D_l + D_l H + 2 H F'_l) + B * sum_l 2 A'_l S_b^2 d + B (H^2 + H C)."""
    H, d, C = cfg.hidden, cfg.head_dim, cfg.num_classes
    total = 0
    for b in batches:
        B, S = len(b.index), b.seq
        for A, F in zip(cfg.heads, cfg.ffn_dim):
            D = A * d
            total += B * S * (H * 3 * D + D * H + 2 * H * F) + B * 2 * A * S * S * d
        total += B * (H * H + H * C)
    return int(total)


def ragged_lengths(n: int, lo: int, hi: int, seed: int) -> np.ndarray:
    """Lengths ~ U[lo, hi] (the ragged recipe of DESIGN §4 / SURVEY 8(d))."""
    return np.random.default_rng(seed).integers(lo, hi + 1, n)


def make_corpus(cfg, lengths: Sequence[int], seed: int) -> List[np.ndarray]:
    """Token-id sequences: CLS first, then ids ~ U[5, V)."""
    rng = np.random.default_rng(seed)
    out = []
    for L in lengths:
        s = rng.integers(5, cfg.vocab_size, int(L)).astype(np.int32)
        s[0] = cfg.cls_id
        out.append(s)
    return out


def classify(encode, corpus: Sequence[np.ndarray], batch_size: int, mode: str, fixed_len: int = None,
             multiple: int = 1) -> np.ndarray:
    """Logits [n, C] of a corpus in input order; `encode(ids, mask) -> [B, C]`
    runs one padded batch (the CUDA library through the binding, or the
    oracle in the tests)."""
    lengths = [len(s) for s in corpus]
    batches = make_batches(lengths, batch_size, mode, fixed_len, multiple)
    outs = [np.asarray(encode(*pack(corpus, b))) for b in batches]
    return unmap(batches, outs, len(corpus))
