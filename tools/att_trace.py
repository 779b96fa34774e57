"""Timeline of the tcgen05 attention pipeline (per-CTA per-head events).

python tools/att_trace.py [B] [S] [A]
Events: 0 load issued, 1 kv_full seen (MMA), 2 S MMA issued, 3 s_full seen
(softmax), 4 P published, 5 p_full seen (MMA), 6 o_full seen (epilogue),
7 epilogue done (events 3, 4, 6, 7 of softmax group 0 only: even heads).  Prints per-head intervals (us) for a few CTAs and medians.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2010_13382_b200 import fastformers as ffb

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
S = int(sys.argv[2]) if len(sys.argv) > 2 else 128
A = int(sys.argv[3]) if len(sys.argv) > 3 else 8
d = 64
g = torch.Generator().manual_seed(0)
qkv = (torch.randn(B * S, 3 * A * d, generator=g) * 1.5).half().cuda()
mask = torch.ones(B, S, dtype=torch.int32).cuda()
grid = min(B, 148)
trace = torch.zeros(grid, 32, 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    ffb.attention_q8(qkv, mask, A, d, with_ctx16=False)
# flush L2 so QKV comes from HBM (ATT_NOFLUSH=1: leave it warm)
junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
if not os.environ.get("ATT_NOFLUSH"):
    junk.fill_(1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ffb.attention_q8(qkv, mask, A, d, with_ctx16=False)
e1.record()
torch.cuda.synchronize()
print("untraced launch %.1f us" % (e0.elapsed_time(e1) * 1e3))
if not os.environ.get("ATT_NOFLUSH"):
    junk.fill_(1)
ffb.attention_q8(qkv, mask, A, d, with_ctx16=False, trace=trace)
torch.cuda.synchronize()
t = trace.cpu().numpy().astype(np.int64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, -1) / 1000.0
nh = (B * A + grid - 1) // grid
for c in [0, 1, 100, 147]:
    if c >= grid:
        continue
    print(f"CTA {c}")
    for n in range(min(nh + 1, 32)):
        row = t[c, n]
        if (row < 0).all():
            break
        print("  head %2d " % n + " ".join("%7.2f" % x for x in row))
end = t[:, :, 7].max()
print("kernel span (us, from first event):", end)
v = t[:, :nh]
ok = (v >= 0).all(axis=2)
def med(a, b):
    x = (v[:, :, b] - v[:, :, a]); x = x[(v[:, :, a] >= 0) & (v[:, :, b] >= 0)]
    return np.median(x), np.percentile(x, 90)
import os as _os
if _os.environ.get("ATT_SUB"):
    for name, a, b in [("S seen -> S in regs 3->0", 3, 0), ("mask/max + pair 0->1", 0, 1), ("exp/sum + pair 1->2", 1, 2),
                       ("normalize + P store 2->4", 2, 4)]:
        m, p9 = med(a, b)
        print(f"{name:28s} median {m:7.3f} us  p90 {p9:7.3f}")
for name, a, b in [("load latency 0->1", 0, 1), ("S wait 1->2", 1, 2), ("S ready->seen 2->3", 2, 3),
                   ("softmax 3->4", 3, 4), ("P->MMA seen 4->5", 4, 5), ("P->O seen 4->6", 4, 6),
                   ("epilogue 6->7", 6, 7)]:
    m, p9 = med(a, b)
    print(f"{name:24s} median {m:7.3f} us  p90 {p9:7.3f}")
d3 = np.diff(t[:, :nh, 3], axis=1).ravel()
print("head period (s_full to s_full) median %.3f us p90 %.3f" % (np.median(d3), np.percentile(d3, 90)))
