"""Run a few importance-scoring batches (for ncu): python tools/prof_score.py [iters]
C3-unpruned shape, B 32 x S 128 (the bench's importance_scoring variant)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2010_13382_b200 import synth
from paper_2010_13382_b200.fastformers import Scorer

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = synth.config("c3_unpruned")
sc = Scorer(cfg, synth.make_weights(cfg), max_tokens=32 * 128)
ids, mask = synth.make_inputs(cfg, 32, 128, seed=5000)
labels = np.random.default_rng(77).integers(0, 2, 32).astype(np.int32)
ids, mask, labels = (torch.from_numpy(a).cuda() for a in (ids, mask, labels))
for _ in range(iters):
    sc.score(ids, mask, labels)
torch.cuda.synchronize()
print("done")
