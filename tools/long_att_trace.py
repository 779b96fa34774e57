"""Timeline of the S > 128 tcgen05 attention (attention_long.cu) on a C4-shaped
problem through ff_debug_attention: python tools/long_att_trace.py [B] [S] [A]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2010_13382_b200 import fastformers as ffb

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
S = int(sys.argv[2]) if len(sys.argv) > 2 else 512
A = int(sys.argv[3]) if len(sys.argv) > 3 else 12
d = 64
g = torch.Generator().manual_seed(0)
qkv = (torch.randn(B * S, 3 * A * d, generator=g) * 1.5).half().cuda()
mask = torch.ones(B, S, dtype=torch.int32).cuda()
for _ in range(3):
    ffb.attention(qkv, mask, A, d, impl=2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ffb.attention(qkv, mask, A, d, impl=2)
e1.record()
torch.cuda.synchronize()
print("launch %.1f us" % (e0.elapsed_time(e1) * 1e3))
trace = torch.zeros(148, 32, 8, dtype=torch.int64, device="cuda")
ffb.set_gemm_trace(trace, 4)
ffb.attention(qkv, mask, A, d, impl=2)
torch.cuda.synchronize()
ffb.set_gemm_trace(None, 0)
t = trace.cpu().numpy().astype(np.int64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, -1) / 1000.0
for c in (0, 77):
    print(f"CTA {c}")
    for k in range(8):
        print("  unit %2d " % k + " ".join("%7.2f" % x for x in t[c, k]))
v = t[:, :30]
def med(a, b):
    x = v[:, :, b] - v[:, :, a]
    x = x[(v[:, :, a] >= 0) & (v[:, :, b] >= 0)]
    return np.median(x)
for name, a, b in [("t_free -> S committed", 1, 2), ("S committed -> softmax", 2, 3), ("pass 1", 3, 4),
                   ("pass 2", 4, 5), ("pass 3", 5, 6), ("P -> O read", 6, 7), ("O read -> next t_free seen", 7, 1)]:
    print(f"{name:28s} {med(a, b):7.3f} us")
per = np.diff(v[:, :, 3], axis=1)
print("unit period (s_full to s_full) median %.3f us" % np.median(per[per > 0]))
