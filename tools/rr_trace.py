"""Timeline of the fused row-reduction GEMMs (layer 0 of a C3 int8 forward,
fused epilogues on).  python tools/rr_trace.py [which=1|2|3]
Events: 0 acc free (MMA), 1 first operands, 2 committed, 3 tfull seen by
epilogue warp 0, 8 before stats exchange, 9 after it, 10 LN / act pass done,
11 after the amax exchange, 5 tile done."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2010_13382_b200 import fastformers as ffb, synth

which = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = synth.config("c3").with_dtype(1)
enc = ffb.Encoder(cfg, synth.make_weights(cfg), use_graphs=False, fused=True)
ids, mask = synth.make_inputs(cfg, seed=1000)
ids, mask = torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda()
enc.encode(ids, mask)
torch.cuda.synchronize()
trace = torch.zeros(148, 64, 24, dtype=torch.int64, device="cuda")
ffb.set_gemm_trace(trace, which)
enc.encode(ids, mask)
torch.cuda.synchronize()
ffb.set_gemm_trace(None, 0)
t = trace.cpu().numpy().astype(np.int64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, -1000) / 1000.0
print("span", t.max())
for c in [0, 1, 2]:
    print(f"CTA {c}")
    for i in range(8):
        row = t[c, i]
        if (row < 0).all():
            break
        print("  tile %d " % i + " ".join("%7.2f" % row[e] for e in (0, 1, 2, 3, 8, 9, 10, 11, 5)))
def med(a, b):
    x = t[:, :, b] - t[:, :, a]
    ok = (t[:, :, a] >= 0) & (t[:, :, b] >= 0)
    return np.median(x[ok]) if ok.any() else float("nan")
for nm, a, b in [("MMA span 1->2", 1, 2), ("commit->epi 2->3", 2, 3), ("pass1 (+M2) 3->8", 3, 8),
                 ("stats exchange 8->9", 8, 9), ("LN pass 9->10", 9, 10), ("act pass 3->10", 3, 10),
                 ("amax exchange 10->11", 10, 11), ("quant ch0 11->12", 11, 12), ("quant ch1 12->13", 12, 13), ("quant tail 13->5", 13, 5), ("epi total 3->5", 3, 5)]:
    print(f"{nm:24s} {med(a, b):7.3f} us")
