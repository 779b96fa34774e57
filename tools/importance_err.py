"""Max |gpu - oracle| of the importance scores relative to each layer's max
score, per config (the numbers quoted in DESIGN §3 for NEXT-3)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

from oracle import importance as imp
from test_gpu_importance import CONFIGS, _batch, _cuda
from paper_2010_13382_b200 import fastformers as ffb
from paper_2010_13382_b200 import synth

names = sys.argv[1:] or [c[0] for c in CONFIGS]
for name, mk, B, S, std in CONFIGS:
    if name not in names:
        continue
    cfg = mk()
    w = synth.make_weights(cfg, std=std)
    batches = [_batch(cfg, B, S, 100 + i) for i in range(2)]
    sc = ffb.Scorer(cfg, w, max_tokens=B * S)
    for b in batches:
        sc.score(*_cuda(*b))
    hs, fs = sc.scores()
    rh, rf, _ = imp.compute_importance(cfg, w, batches)
    eh = max(float(np.abs(g - r).max() / np.abs(r).max()) for g, r in zip(hs, rh))
    ef = max(float(np.abs(g - r).max() / np.abs(r).max()) for g, r in zip(fs, rf))
    print(f"{name}: max |gpu-ref| / layer max: heads {eh:.2e}  ffn units {ef:.2e}", flush=True)
