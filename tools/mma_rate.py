"""MMA-rate probe of the production GEMM kernel (ff_debug_gemm bit 6 skips
the operand TMA loads, so the tile time is MMA issue + epilogue only).
Compares loaded vs no-load launches per shape: if no-load is much faster the
mainloop is operand-feed bound, otherwise MMA / epilogue bound.

python tools/mma_rate.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2010_13382_b200 import fastformers as ffb


def run(M, N, K, i8, noload, act=-1):
    g = torch.Generator().manual_seed(0)
    if i8:
        A = torch.randint(-127, 128, (M, K), generator=g, dtype=torch.int8).cuda()
        W = torch.randint(-127, 128, (N, K), generator=g, dtype=torch.int8).cuda()
    else:
        A = torch.randn(M, K, generator=g).half().cuda()
        W = (torch.randn(N, K, generator=g) * 0.05).half().cuda()
    sx = torch.rand(M, generator=g).cuda() * 1e-3
    sw = torch.rand(N, generator=g).cuda() * 1e-3
    bias = torch.randn(N, generator=g).cuda()
    out = torch.empty(M, N, dtype=torch.float16, device="cuda")
    mode = 1 | 16 | (64 if noload else 0)
    ts = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for i in range(25):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ffb.gemm(A, W, mode, bias=bias, sx=sx if i8 else None, sw=sw if i8 else None, act=act, out=out)
        e1.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    return ms * 1e3, 2 * M * N * K / ms / 1e9


for (M, N, K, i8, act) in [(32768, 1536, 768, True, -1), (32768, 768, 1536, True, -1), (32768, 768, 512, True, -1),
                           (32768, 1536, 768, True, 0), (32768, 1536, 6144, True, -1), (32768, 1536, 768, False, -1),
                           (32768, 1536, 6144, False, -1)]:
    r = [run(M, N, K, i8, nl, act) for nl in (False, True)]
    print(f"{'i8 ' if i8 else 'f16'} M{M} N{N} K{K} act{act}: loaded {r[0][0]:6.1f} us {r[0][1]:6.0f} TOP/s | "
          f"no-load {r[1][0]:6.1f} us {r[1][1]:6.0f} TOP/s", flush=True)
