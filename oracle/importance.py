"""CPU oracle for structured-pruning importance scores -- TEST INFRASTRUCTURE ONLY.

SURVEY 8(f) NEXT-3.  Only ``tests/`` and ``bench.py`` may import this module;
it shares no code with the CUDA library.  Plain numpy in fp64, no blocking or
fusion: the encoder forward written out, then its reverse-mode derivative
step by step (the "backward pass" of PAPER.md P:93).

Paper: "we add a mask variable to each attention head for the gradient
computation of the heads.  Next, we run forward and backward passes of the
model on the entire validation data set, then the absolute values of the
gradients are accumulated.  These accumulated values are used as importance
scores which we use to sort the importance of the heads and the intermediate
hidden states.  Based on the target model size, we select a given number of
top heads and top hidden states from the network. ... we re-group and
reconnect the remaining heads and hidden states which result in a smaller
sized model. ... we use the same pruning ratio across different layers."

Readings (R23-R25):
* R23 mask variables: xi[l, h] multiplies head h's context rows before the
  output projection; nu[l, f] multiplies FFN unit f after the activation,
  before the second FFN linear.  Both are 1 when scoring.
* R24 loss: the task loss, mean cross-entropy of the classifier logits over
  the batch's sequences (SPEC S:295 default; the paper does not say).  Per
  batch, the mask gradient is summed over the batch, its absolute value is
  taken, and added to the running score ("absolute values taken
  per batch before accumulation").
* R25 selection: per layer keep max(1, floor(n * ratio)) of n units, the top
  scores, ties to the lower index, kept indices ascending;
  the same ratio in every layer.
The forward is the ref64 encoder of ``oracle.cpp`` (post-LN BERT, DESIGN R1-R4,
R10, R16): masked keys get probability 0, 1/sqrt(d) multiplies Q K^T, position
ids 0..S-1, token-type row 0, tanh pooler on position 0, GELU-erf / ReLU /
GELU-tanh.

Pins (tests/test_importance.py, -m "not gpu"): central finite differences of
the loss w.r.t. every mask variable on a tiny model; the forward logits equal
the C++ oracle's ref64 logits; a head whose output-projection columns are
zero scores exactly 0; two identical heads score equally; the pruned model's
loss equals the masked model's; SPEC's select_keep examples.
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence, Tuple

import numpy as np
from scipy.special import erf

SQRT1_2 = 1.0 / math.sqrt(2.0)


def _w(weights, name):
    for pre in ("", "bert.", "roberta."):
        if pre + name in weights:
            return np.asarray(weights[pre + name], dtype=np.float64)
    raise KeyError(name)


def _act(u, act):
    if act == 0:  # GELU-erf
        return 0.5 * u * (1.0 + erf(u * SQRT1_2))
    if act == 1:  # ReLU
        return np.maximum(u, 0.0)
    return 0.5 * u * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (u + 0.044715 * u ** 3)))


def _act_grad(u, act):
    """d act(u) / du."""
    if act == 0:
        return 0.5 * (1.0 + erf(u * SQRT1_2)) + u * np.exp(-0.5 * u * u) / math.sqrt(2.0 * math.pi)
    if act == 1:
        return (u > 0.0).astype(np.float64)
    c = math.sqrt(2.0 / math.pi)
    t = np.tanh(c * (u + 0.044715 * u ** 3))
    return 0.5 * (1.0 + t) + 0.5 * u * (1.0 - t * t) * c * (1.0 + 3 * 0.044715 * u * u)


def _ln(x, g, b, eps):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xh = (x - mu) * rstd
    return xh * g + b, xh, rstd


def _ln_back(dy, g, xh, rstd):
    """LayerNorm input gradient: rstd * (dxh - mean(dxh) - xh * mean(dxh * xh))."""
    dxh = dy * g
    return rstd * (dxh - dxh.mean(axis=-1, keepdims=True) - xh * (dxh * xh).mean(axis=-1, keepdims=True))


def forward_backward(cfg, weights: Dict[str, np.ndarray], ids, mask, labels, xi=None, nu=None):
    """One batch: loss (mean CE), logits, dL/dxi [L][A_l], dL/dnu [L][F_l].

    ids, mask: [B, S] ints; labels: [B].  xi / nu default to all ones."""
    ids = np.asarray(ids)
    mask = np.asarray(mask)
    labels = np.asarray(labels)
    B, S = ids.shape
    L, H, d = cfg.num_layers, cfg.hidden, cfg.head_dim
    xi = [np.ones(cfg.heads[l]) for l in range(L)] if xi is None else [np.asarray(v, np.float64) for v in xi]
    nu = [np.ones(cfg.ffn_dim[l]) for l in range(L)] if nu is None else [np.asarray(v, np.float64) for v in nu]
    keyok = mask.astype(bool)  # [B, S]

    # embeddings + LayerNorm (R16)
    x = _w(weights, "embeddings.word_embeddings.weight")[ids] + \
        _w(weights, "embeddings.position_embeddings.weight")[np.arange(S)][None] + \
        _w(weights, "embeddings.token_type_embeddings.weight")[0][None, None]
    x, _, _ = _ln(x, _w(weights, "embeddings.LayerNorm.weight"), _w(weights, "embeddings.LayerNorm.bias"), cfg.ln_eps)

    saved = []
    for l in range(L):
        p = f"encoder.layer.{l}."
        A = cfg.heads[l]
        wq, wk, wv = (_w(weights, p + f"attention.self.{n}.weight") for n in ("query", "key", "value"))
        bq, bk, bv = (_w(weights, p + f"attention.self.{n}.bias") for n in ("query", "key", "value"))
        q = (x @ wq.T + bq).reshape(B, S, A, d).transpose(0, 2, 1, 3)  # [B, A, S, d]
        k = (x @ wk.T + bk).reshape(B, S, A, d).transpose(0, 2, 1, 3)
        v = (x @ wv.T + bv).reshape(B, S, A, d).transpose(0, 2, 1, 3)
        s = np.einsum("bhid,bhjd->bhij", q, k) * (1.0 / math.sqrt(d))
        s = np.where(keyok[:, None, None, :], s, -np.inf)  # masked keys: probability 0 (R4)
        e = np.exp(s - s.max(axis=-1, keepdims=True))
        P = e / e.sum(axis=-1, keepdims=True)
        c = np.einsum("bhij,bhjd->bhid", P, v)  # [B, A, S, d]
        cm = c * xi[l][None, :, None, None]  # head mask (R23)
        cflat = cm.transpose(0, 2, 1, 3).reshape(B, S, A * d)
        o = cflat @ _w(weights, p + "attention.output.dense.weight").T + _w(weights, p + "attention.output.dense.bias")
        g1 = _w(weights, p + "attention.output.LayerNorm.weight")
        y1, xh1, r1 = _ln(o + x, g1, _w(weights, p + "attention.output.LayerNorm.bias"), cfg.ln_eps)
        u = y1 @ _w(weights, p + "intermediate.dense.weight").T + _w(weights, p + "intermediate.dense.bias")
        a = _act(u, cfg.act)
        am = a * nu[l]  # FFN-unit mask (R23)
        o2 = am @ _w(weights, p + "output.dense.weight").T + _w(weights, p + "output.dense.bias")
        g2 = _w(weights, p + "output.LayerNorm.weight")
        y2, xh2, r2 = _ln(o2 + y1, g2, _w(weights, p + "output.LayerNorm.bias"), cfg.ln_eps)
        saved.append(dict(x=x, q=q, k=k, v=v, P=P, c=c, g1=g1, xh1=xh1, r1=r1, u=u, a=a, g2=g2, xh2=xh2, r2=r2))
        x = y2

    wp, bp = _pool_weights(weights)
    wc, bc = _cls_weights(weights)
    pool = np.tanh(x[:, 0, :] @ wp.T + bp)  # [B, H]
    logits = pool @ wc.T + bc  # [B, C]
    z = logits - logits.max(axis=1, keepdims=True)
    lse = np.log(np.exp(z).sum(axis=1))
    loss = float(np.mean(lse - z[np.arange(B), labels]))  # R24

    # ---- backward
    prob = np.exp(z - lse[:, None])
    dlogits = prob.copy()
    dlogits[np.arange(B), labels] -= 1.0
    dlogits /= B
    dpool = dlogits @ wc
    dpre = dpool * (1.0 - pool * pool)
    dx = np.zeros_like(x)
    dx[:, 0, :] = dpre @ wp
    dxi = [None] * L
    dnu = [None] * L
    for l in reversed(range(L)):
        p = f"encoder.layer.{l}."
        A = cfg.heads[l]
        sv = saved[l]
        dz2 = _ln_back(dx, sv["g2"], sv["xh2"], sv["r2"])  # d(o2 + y1)
        dam = dz2 @ _w(weights, p + "output.dense.weight")  # [B, S, F]
        dnu[l] = np.einsum("bsf,bsf->f", sv["a"], dam)
        du = dam * nu[l] * _act_grad(sv["u"], cfg.act)
        dy1 = dz2 + du @ _w(weights, p + "intermediate.dense.weight")
        dz1 = _ln_back(dy1, sv["g1"], sv["xh1"], sv["r1"])  # d(o + x)
        dcflat = dz1 @ _w(weights, p + "attention.output.dense.weight")  # [B, S, A d]
        dcm = dcflat.reshape(B, S, A, d).transpose(0, 2, 1, 3)
        dxi[l] = np.einsum("bhid,bhid->h", sv["c"], dcm)
        dc = dcm * xi[l][None, :, None, None]
        dP = np.einsum("bhid,bhjd->bhij", dc, sv["v"])
        dv = np.einsum("bhij,bhid->bhjd", sv["P"], dc)
        ds = sv["P"] * (dP - (dP * sv["P"]).sum(axis=-1, keepdims=True)) * (1.0 / math.sqrt(d))
        dq = np.einsum("bhij,bhjd->bhid", ds, sv["k"])
        dk = np.einsum("bhij,bhid->bhjd", ds, sv["q"])
        back = lambda t: t.transpose(0, 2, 1, 3).reshape(B, S, A * d)
        dx = dz1 + back(dq) @ _w(weights, p + "attention.self.query.weight") + \
            back(dk) @ _w(weights, p + "attention.self.key.weight") + \
            back(dv) @ _w(weights, p + "attention.self.value.weight")
    return loss, logits, dxi, dnu


def _pool_weights(weights):
    try:
        return _w(weights, "pooler.dense.weight"), _w(weights, "pooler.dense.bias")
    except KeyError:
        return _w(weights, "classifier.dense.weight"), _w(weights, "classifier.dense.bias")


def _cls_weights(weights):
    try:
        return _w(weights, "classifier.weight"), _w(weights, "classifier.bias")
    except KeyError:
        return _w(weights, "classifier.out_proj.weight"), _w(weights, "classifier.out_proj.bias")


def loss_only(cfg, weights, ids, mask, labels, xi=None, nu=None) -> float:
    return forward_backward(cfg, weights, ids, mask, labels, xi, nu)[0]


def compute_importance(cfg, weights, batches: Sequence[Tuple[np.ndarray, np.ndarray, np.ndarray]]):
    """Accumulate |dL/dxi| and |dL/dnu| over batches (R24).
    Returns (head_scores [L][A_l], ffn_scores [L][F_l], losses)."""
    hs = [np.zeros(cfg.heads[l]) for l in range(cfg.num_layers)]
    fs = [np.zeros(cfg.ffn_dim[l]) for l in range(cfg.num_layers)]
    losses = []
    for ids, mask, labels in batches:
        loss, _, dxi, dnu = forward_backward(cfg, weights, ids, mask, labels)
        for l in range(cfg.num_layers):
            hs[l] += np.abs(dxi[l])
            fs[l] += np.abs(dnu[l])
        losses.append(loss)
    return hs, fs, losses


def select_keep(scores: Sequence[float], keep: int) -> List[int]:
    """Indices of the `keep` largest scores, ties to the lower index, ascending (R25)."""
    order = sorted(range(len(scores)), key=lambda i: (-scores[i], i))
    return sorted(order[:keep])
