"""Timeline of the tcgen05 GEMM pipeline (per-CTA per-tile events) for one C3
GEMM shape through the debug entry.

python tools/gemm_trace.py [M] [N] [K] [act]   (act: -1 none, 0 GELU)
Events (us from the first): 0 acc free seen by MMA, 1 first operands seen,
2 accumulator committed, 3 tfull seen by epilogue, 4 acc released,
5 epilogue done, 6 first load issued; per epilogue chunk i: 8+3i TMEM load
landed, 9+3i staging buffer free, 10+3i store issued.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2010_13382_b200 import fastformers as ffb

M = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1536
K = int(sys.argv[3]) if len(sys.argv) > 3 else 768
act = int(sys.argv[4]) if len(sys.argv) > 4 else -1
g = torch.Generator().manual_seed(0)
A = torch.randint(-127, 128, (M, K), generator=g, dtype=torch.int8).cuda()
W = torch.randint(-127, 128, (N, K), generator=g, dtype=torch.int8).cuda()
sx = torch.rand(M, generator=g).cuda() * 1e-3
sw = torch.rand(N, generator=g).cuda() * 1e-3
bias = torch.randn(N, generator=g).cuda()
out = torch.empty(M, N, dtype=torch.float16, device="cuda")
for _ in range(3):
    ffb.gemm(A, W, 1, bias=bias, sx=sx, sw=sw, act=act, out=out)
torch.cuda.synchronize()
trace = torch.zeros(148, 64, 24, dtype=torch.int64, device="cuda")
ffb.set_gemm_trace(trace)
junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
junk.fill_(1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ffb.gemm(A, W, 1, bias=bias, sx=sx, sw=sw, act=act, out=out)
e1.record()
torch.cuda.synchronize()
ffb.set_gemm_trace(None)
print(f"M {M} N {N} K {K} act {act}: {e0.elapsed_time(e1) * 1e3:.1f} us ({2 * M * N * K / e0.elapsed_time(e1) / 1e9:.0f} TOP/s)")
t = trace.cpu().numpy().astype(np.int64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, -1000) / 1000.0
for c in [0, 1, 2, 147]:
    print(f"CTA {c}")
    for i in range(64):
        row = t[c, i]
        if (row < 0).all():
            break
        print("  tile %2d " % i + " ".join("%7.2f" % x for x in row[:7]) + " | chunks " + " ".join("%6.2f" % x for x in row[8:20]))
def med(a, b):
    x = (t[:, :, b] - t[:, :, a])
    ok = (t[:, :, a] >= 0) & (t[:, :, b] >= 0)
    return np.median(x[ok]), np.percentile(x[ok], 90)
for name, a, b in [("load issue->operands 6->1", 6, 1), ("MMA span 1->2", 1, 2), ("commit->epi seen 2->3", 2, 3),
                   ("epi TMEM drain 3->4", 3, 4), ("epi total 3->5", 3, 5), ("acc free->operands 0->1", 0, 1)]:
    m, p9 = med(a, b)
    print(f"{name:28s} median {m:7.3f} us  p90 {p9:7.3f}")
for i in range(4):
    for a, b, nm in [(3 if i == 0 else 10 + 3 * (i - 1), 8 + 3 * i, "ld landed"), (8 + 3 * i, 9 + 3 * i, "buf free"), (9 + 3 * i, 10 + 3 * i, "sts+store")]:
        m, p9 = med(a, b)
        print(f"chunk {i} {nm:10s} median {m:7.3f} us  p90 {p9:7.3f}")
for i in range(4):
    m, p9 = med(8 + 3 * i, 20 + i)
    print(f"chunk {i} math only  median {m:7.3f} us  p90 {p9:7.3f}")
