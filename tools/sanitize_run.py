"""Small forwards of every kernel variant for compute-sanitizer (memcheck /
racecheck / synccheck):

  compute-sanitizer --tool racecheck python tools/sanitize_run.py

C1 (int8, fp16, mixed; every fusion mask), a C3-shaped int8 / fp16 batch of 8
sequences (CTA-pair GEMMs, cluster row-reduction epilogues, tcgen05 attention
with fused requant), C2-shaped d = 26 attention (manual cp.async producer),
C4-shaped S = 512 / 256 attention (attention_long), and the importance scorer.
Un-graphed launches so each kernel is checked where it is launched.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2010_13382_b200 import synth
from paper_2010_13382_b200.fastformers import Encoder, Scorer


def run(name, dt, B, S, **kw):
    cfg = synth.config(name).with_dtype(dt).with_batch(B, S)
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, B=B, S=S, ragged=True, seed=3)
    enc = Encoder(cfg, w, max_tokens=B * S, use_graphs=False, **kw)
    out = enc.encode(torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda())
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    print(f"ok {name} dtype={dt} B={B} S={S} {kw}", flush=True)


def main():
    # --no-cluster-exchange: only configurations without multi-CTA row-reduction
    # clusters (memcheck reports their DSMEM bulk copies, see profiles/r02_sanitizers.md)
    nox = "--no-cluster-exchange" in sys.argv
    fms = (0,) if nox else (0, 2, 7)
    for dt in ([1, 1], [0, 0], [1, 0]):
        for fm in fms:
            run("c1", dt, 4, 32, fused=fm)
    run("c1", [1, 1], 4, 32, act_quant=1)
    run("c3", 1, 8, 128, **({"fused": 0} if nox else {}))
    run("c3", 0, 8, 128, **({"fused": 0} if nox else {}))
    run("c3", 1, 8, 128, fused=0)
    run("c2", 1, 4, 128, **({"fused": 0} if nox else {}))
    run("c4", 0, 2, 512, **({"fused": 0} if nox else {}))
    run("c5", 0, 2, 256, **({"fused": 0} if nox else {}))
    cfg = synth.config("c1")
    sc = Scorer(cfg, synth.make_weights(cfg), max_tokens=4 * 32)
    ids, mask = synth.make_inputs(cfg, B=4, S=32, ragged=True, seed=4)
    labels = np.array([0, 1, 1, 0], np.int32)
    sc.score(*(torch.from_numpy(a).cuda() for a in (ids, mask, labels)))
    torch.cuda.synchronize()
    print("ok scorer", flush=True)


if __name__ == "__main__":
    main()
