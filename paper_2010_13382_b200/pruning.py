"""Structured pruning, host side.

The importance scores come from the GPU scorer (``fastformers.Scorer``, C-ABI
``ff_score_batch``): accumulated |dL/dxi| per head and |dL/dnu| per FFN unit.
This module does the two host steps after it, which are index bookkeeping and
weight slicing only:

* ``select_keep`` -- "we select a given number of top heads and top hidden
  states": per layer the top-k scores, ties to the lower index, kept
  indices ascending (DESIGN R25);
* ``prune`` -- "we re-group and reconnect the remaining heads and hidden states
  which result in a smaller sized model" with "the same pruning ratio across
  different layers": slices Q/K/V rows and output-projection columns of
  the kept heads, FFN1 rows / FFN2 columns of the kept units, and returns the
  pruned geometry that ``ff_model_create`` takes (per-layer heads / ffn_dim).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Sequence, Tuple

import numpy as np


def select_keep(scores: Sequence[float], keep: int) -> List[int]:
    """Indices of the `keep` highest scores (ties -> lower index), ascending."""
    s = np.asarray(scores, dtype=np.float64)
    order = np.lexsort((np.arange(len(s)), -s))  # primary: score descending, then index ascending
    return sorted(int(i) for i in order[:keep])


def keep_count(n: int, ratio: float) -> int:
    """max(1, floor(n * ratio)) units of n."""
    if not 0.0 < ratio <= 1.0:
        raise ValueError("keep ratio must be in (0, 1]")
    return max(1, int(math.floor(n * ratio + 1e-12)))


def _name(weights, name):
    for pre in ("", "bert.", "roberta."):
        if pre + name in weights:
            return pre + name
    raise KeyError(name)


def prune(cfg, weights: Dict[str, np.ndarray], head_scores, ffn_scores, head_ratio: float, ffn_ratio: float
          ) -> Tuple[object, Dict[str, np.ndarray], List[List[int]], List[List[int]]]:
    """Reconnect the model to its top heads / FFN units.  Returns (pruned cfg,
    pruned weights, kept head indices per layer, kept unit indices per layer)."""
    d = cfg.head_dim
    out = dict(weights)
    kept_h, kept_f = [], []
    for l in range(cfg.num_layers):
        kh = select_keep(head_scores[l][:cfg.heads[l]], keep_count(cfg.heads[l], head_ratio))
        kf = select_keep(ffn_scores[l][:cfg.ffn_dim[l]], keep_count(cfg.ffn_dim[l], ffn_ratio))
        kept_h.append(kh)
        kept_f.append(kf)
        cols = np.concatenate([np.arange(h * d, (h + 1) * d) for h in kh])
        p = f"encoder.layer.{l}."
        for n in ("query", "key", "value"):
            wn, bn = _name(weights, p + f"attention.self.{n}.weight"), _name(weights, p + f"attention.self.{n}.bias")
            out[wn] = np.ascontiguousarray(weights[wn][cols])
            out[bn] = np.ascontiguousarray(weights[bn][cols])
        on = _name(weights, p + "attention.output.dense.weight")
        out[on] = np.ascontiguousarray(weights[on][:, cols])
        i_w, i_b = _name(weights, p + "intermediate.dense.weight"), _name(weights, p + "intermediate.dense.bias")
        out[i_w] = np.ascontiguousarray(weights[i_w][kf])
        out[i_b] = np.ascontiguousarray(weights[i_b][kf])
        o_w = _name(weights, p + "output.dense.weight")
        out[o_w] = np.ascontiguousarray(weights[o_w][:, kf])
    pcfg = dataclasses.replace(cfg, heads=[len(k) for k in kept_h], ffn_dim=[len(k) for k in kept_f])
    return pcfg, out, kept_h, kept_f
