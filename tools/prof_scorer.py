"""One importance-scoring batch (C3-unpruned, B 32 x S 128) for ncu launch lists:

  ncu --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/prof_scorer.py [tc=1] [B] [S]

Runs one warm-up batch, then one batch inside cudaProfilerStart/Stop (use
ncu --profile-from-start off to capture only that batch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2010_13382_b200 import synth
from paper_2010_13382_b200.fastformers import Scorer

tc = int(sys.argv[1]) if len(sys.argv) > 1 else 1
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
S = int(sys.argv[3]) if len(sys.argv) > 3 else 128
cfg = synth.config("c3_unpruned")
sc = Scorer(cfg, synth.make_weights(cfg), max_tokens=B * S, tc_linears=bool(tc))
ids, mask = synth.make_inputs(cfg, B, S, seed=1)
labels = np.random.default_rng(2).integers(0, cfg.num_classes, B).astype(np.int32)
args = [torch.from_numpy(a).cuda() for a in (ids, mask, labels)]
sc.score(*args)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
sc.score(*args)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
