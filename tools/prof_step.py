"""Run a few C3 forwards (for ncu): python tools/prof_step.py [config] [i8|f16] [iters] [fusion]
fusion: default (library default, FF_OPT_FUSED_MASK 2) | fused (all, 7) | unfused (0) | a mask 0..7"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2010_13382_b200 import synth
from paper_2010_13382_b200.fastformers import Encoder

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
dt = 1 if (len(sys.argv) <= 2 or sys.argv[2] == "i8") else 0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
arg = sys.argv[4] if len(sys.argv) > 4 else "default"
fused = {"default": None, "fused": True, "unfused": False}.get(arg, None if not arg.isdigit() else int(arg))
cfg = synth.config(name).with_dtype(dt)
enc = Encoder(cfg, synth.make_weights(cfg), use_graphs=False, fused=fused)
ids, mask = synth.make_inputs(cfg, seed=1000)
ids, mask = torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda()
for _ in range(iters):
    enc.encode(ids, mask)
torch.cuda.synchronize()
print("done")
