"""Seeded synthetic workloads shared by the tests, the bench and the oracle.

This module holds NO arithmetic of the method: it only describes model
geometries (BASELINE.json ``configs``) and draws seeded random
weights, token ids and masks.  Both the CUDA path
and the CPU oracle consume what it produces.

Weights: every matrix / embedding ~ N(0, 0.02) (BERT initializer_range),
biases ~ N(0, 0.02) (non-zero on purpose), LayerNorm gamma ~ 1 + N(0, 0.1),
beta ~ N(0, 0.02).  Token ids ~ U[5, V) with position 0 = CLS.  Masks: all
ones (throughput headline) or ragged lengths ~ U[ceil(S/4), S].
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Sequence

import numpy as np

F16, I8 = 0, 1
ACT_GELU, ACT_RELU, ACT_GELU_TANH = 0, 1, 2


@dataclasses.dataclass
class ModelConfig:
    name: str
    num_layers: int
    hidden: int
    head_dim: int
    heads: List[int]
    ffn_dim: List[int]
    dtype: List[int]
    vocab_size: int
    max_positions: int
    num_classes: int
    ln_eps: float
    act: int = ACT_GELU
    batch: int = 1
    seq: int = 128
    cls_id: int = 101

    def with_dtype(self, dt) -> "ModelConfig":
        dts = [dt] * self.num_layers if isinstance(dt, int) else list(dt)
        return dataclasses.replace(self, dtype=dts)

    def with_batch(self, batch: int, seq: int | None = None) -> "ModelConfig":
        return dataclasses.replace(self, batch=batch, seq=self.seq if seq is None else seq)

    def flops_per_seq(self, S: int | None = None) -> float:
        """Algorithmic FLOPs per sequence (SURVEY 8(d) d3 = S:432 count_macs x 2
        with pruned widths): GEMMs + attention + pooler/classifier."""
        S = self.seq if S is None else S
        H, d, C = self.hidden, self.head_dim, self.num_classes
        f = 0.0
        for A, F in zip(self.heads, self.ffn_dim):
            D = A * d
            f += 2.0 * S * (H * 3 * D + D * H + 2 * H * F)
            f += 2.0 * 2 * A * S * S * d
        f += 2.0 * (H * H + H * C)
        return f

    def gemm_flops_per_seq(self, S: int | None = None) -> float:
        S = self.seq if S is None else S
        H, d = self.hidden, self.head_dim
        return sum(2.0 * S * (H * 3 * A * d + A * d * H + 2 * H * F) for A, F in zip(self.heads, self.ffn_dim))


def _uniform(L, v):
    return [v] * L


def config(name: str) -> ModelConfig:
    """BASELINE.json configs (0-based index in the JSON; SURVEY calls them C1..C5)."""
    if name == "c1":  # configs[0]: tiny pruned, 2 layers, hidden 128, heads [2,1], FFN [256,128], B4 S32
        return ModelConfig("c1", 2, 128, 64, [2, 1], [256, 128], [I8, I8], 30522, 512, 2, 1e-12,
                           batch=4, seq=32, cls_id=101)
    if name == "c2":  # configs[1]: TinyBERT 4L/312, 12 heads (d=26), FFN 1200, B64 S128
        return ModelConfig("c2", 4, 312, 26, _uniform(4, 12), _uniform(4, 1200), _uniform(4, I8), 30522, 512, 2,
                           1e-12, batch=64, seq=128, cls_id=101)
    if name in ("c2_9_900", "c2_8_600"):  # Table 3 pruned TinyBERT students (DESIGN R20)
        A, F = (9, 900) if name == "c2_9_900" else (8, 600)
        return ModelConfig(name, 4, 312, 26, _uniform(4, A), _uniform(4, F), _uniform(4, I8), 30522, 512, 2,
                           1e-12, batch=64, seq=128, cls_id=101)
    if name == "c3":  # configs[2]: distilroberta 6L/768, heads 12->8, FFN 3072->1536, int8, B256 S128
        return ModelConfig("c3", 6, 768, 64, _uniform(6, 8), _uniform(6, 1536), _uniform(6, I8), 50265, 514, 2,
                           1e-5, batch=256, seq=128, cls_id=0)
    if name == "c3_unpruned":  # pruning speed-up reference (D2)
        return ModelConfig("c3_unpruned", 6, 768, 64, _uniform(6, 12), _uniform(6, 3072), _uniform(6, I8), 50265,
                           514, 2, 1e-5, batch=256, seq=128, cls_id=0)
    if name == "c4":  # configs[3]: BERT-base 12L unpruned fp16, B128 S512
        return ModelConfig("c4", 12, 768, 64, _uniform(12, 12), _uniform(12, 3072), _uniform(12, F16), 30522, 512, 2,
                           1e-12, batch=128, seq=512, cls_id=101)
    if name == "c5":  # configs[4]: RoBERTa-large shape 24L/1024/16 heads/4096 fp16, B64 S256
        return ModelConfig("c5", 24, 1024, 64, _uniform(24, 16), _uniform(24, 4096), _uniform(24, F16), 50265, 514,
                           2, 1e-5, batch=64, seq=256, cls_id=0)
    raise KeyError(name)


def tensor_shapes(cfg: ModelConfig) -> Dict[str, tuple]:
    """HF BERT state_dict names -> shapes for a (pruned) geometry."""
    H, d = cfg.hidden, cfg.head_dim
    s = {
        "embeddings.word_embeddings.weight": (cfg.vocab_size, H),
        "embeddings.position_embeddings.weight": (cfg.max_positions, H),
        "embeddings.token_type_embeddings.weight": (2, H),
        "embeddings.LayerNorm.weight": (H,),
        "embeddings.LayerNorm.bias": (H,),
    }
    for l in range(cfg.num_layers):
        D, F = cfg.heads[l] * d, cfg.ffn_dim[l]
        p = f"encoder.layer.{l}."
        for w in ("query", "key", "value"):
            s[p + f"attention.self.{w}.weight"] = (D, H)
            s[p + f"attention.self.{w}.bias"] = (D,)
        s[p + "attention.output.dense.weight"] = (H, D)
        s[p + "attention.output.dense.bias"] = (H,)
        s[p + "attention.output.LayerNorm.weight"] = (H,)
        s[p + "attention.output.LayerNorm.bias"] = (H,)
        s[p + "intermediate.dense.weight"] = (F, H)
        s[p + "intermediate.dense.bias"] = (F,)
        s[p + "output.dense.weight"] = (H, F)
        s[p + "output.dense.bias"] = (H,)
        s[p + "output.LayerNorm.weight"] = (H,)
        s[p + "output.LayerNorm.bias"] = (H,)
    s["pooler.dense.weight"] = (H, H)
    s["pooler.dense.bias"] = (H,)
    s["classifier.weight"] = (cfg.num_classes, H)
    s["classifier.bias"] = (cfg.num_classes,)
    return s


def make_weights(cfg: ModelConfig, seed: int = 1234, std: float = 0.02) -> Dict[str, np.ndarray]:
    """Seeded random-init weights (fp32) for the geometry in ``cfg``."""
    out = {}
    for i, (name, shape) in enumerate(tensor_shapes(cfg).items()):
        rng = np.random.Generator(np.random.PCG64([seed, i]))
        if name.endswith("LayerNorm.weight"):
            a = 1.0 + 0.1 * rng.standard_normal(shape, dtype=np.float32)
        else:
            a = std * rng.standard_normal(shape, dtype=np.float32)
        out[name] = a.astype(np.float32)
    return out


def make_inputs(cfg: ModelConfig, B: int | None = None, S: int | None = None, seed: int = 1000,
                ragged: bool = False, lengths: Sequence[int] | None = None):
    """Token ids [B,S] int32 (id 0 of each row = CLS) and a 0/1 mask [B,S] int32."""
    B = cfg.batch if B is None else B
    S = cfg.seq if S is None else S
    rng = np.random.Generator(np.random.PCG64(seed))
    ids = rng.integers(5, cfg.vocab_size, size=(B, S), dtype=np.int64).astype(np.int32)
    ids[:, 0] = cfg.cls_id
    mask = np.ones((B, S), np.int32)
    if lengths is not None:
        for b, n in enumerate(lengths):
            mask[b, n:] = 0
    elif ragged:
        lo = max(1, math.ceil(S / 4))
        lens = rng.integers(lo, S + 1, size=B)
        for b, n in enumerate(lens):
            mask[b, n:] = 0
    return ids, mask


# ------------------------------------------------------------- pruning utils
# Structured pruning "re-group and reconnect" as pure index
# selection: keep the listed heads / FFN units of each layer.
def prune_slice(cfg: ModelConfig, w: Dict[str, np.ndarray], keep_heads, keep_ffn):
    """Return (pruned cfg, pruned weights) keeping heads keep_heads[l] and FFN units keep_ffn[l]."""
    d = cfg.head_dim
    nw = dict(w)
    heads, ffn = [], []
    for l in range(cfg.num_layers):
        p = f"encoder.layer.{l}."
        kh = list(keep_heads[l])
        kf = np.asarray(list(keep_ffn[l]), dtype=np.int64)
        cols = np.concatenate([np.arange(h * d, (h + 1) * d) for h in kh])
        for t in ("query", "key", "value"):
            nw[p + f"attention.self.{t}.weight"] = w[p + f"attention.self.{t}.weight"][cols].copy()
            nw[p + f"attention.self.{t}.bias"] = w[p + f"attention.self.{t}.bias"][cols].copy()
        nw[p + "attention.output.dense.weight"] = w[p + "attention.output.dense.weight"][:, cols].copy()
        nw[p + "intermediate.dense.weight"] = w[p + "intermediate.dense.weight"][kf].copy()
        nw[p + "intermediate.dense.bias"] = w[p + "intermediate.dense.bias"][kf].copy()
        nw[p + "output.dense.weight"] = w[p + "output.dense.weight"][:, kf].copy()
        heads.append(len(kh))
        ffn.append(len(kf))
    return dataclasses.replace(cfg, heads=heads, ffn_dim=ffn), nw


def prune_zero(cfg: ModelConfig, w: Dict[str, np.ndarray], keep_heads, keep_ffn):
    """Same model as prune_slice but unpruned geometry with removed parts zeroed."""
    d = cfg.head_dim
    nw = {k: v.copy() for k, v in w.items()}
    for l in range(cfg.num_layers):
        p = f"encoder.layer.{l}."
        drop_h = [h for h in range(cfg.heads[l]) if h not in set(keep_heads[l])]
        drop_f = np.asarray([f for f in range(cfg.ffn_dim[l]) if f not in set(keep_ffn[l])], dtype=np.int64)
        for h in drop_h:
            cols = slice(h * d, (h + 1) * d)
            for t in ("query", "key", "value"):
                nw[p + f"attention.self.{t}.weight"][cols] = 0.0
                nw[p + f"attention.self.{t}.bias"][cols] = 0.0
            nw[p + "attention.output.dense.weight"][:, cols] = 0.0
        if drop_f.size:
            nw[p + "intermediate.dense.weight"][drop_f] = 0.0
            nw[p + "intermediate.dense.bias"][drop_f] = 0.0
            nw[p + "output.dense.weight"][:, drop_f] = 0.0
    return nw
