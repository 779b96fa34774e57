"""Sweep FF_OPT_ROW_DIRS on the C3 int8 step (graph replay, L2 flushed before
each step, median of 40): python tools/dirs_sweep.py [masks...]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2010_13382_b200 import synth  # noqa: E402
from paper_2010_13382_b200 import fastformers as ffb  # noqa: E402

masks = [int(x, 0) for x in sys.argv[1:]] or [0b01010, 0, 0b01000, 0b01011, 0b01001, 0b11010, 0b01110]
cfg = synth.config("c3").with_dtype(1)
enc = ffb.Encoder(cfg, synth.make_weights(cfg), device=0)
ids, mask = synth.make_inputs(cfg)
ids, mask = torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for rep in range(2):
    for m in masks:
        ffb.check(ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_ROW_DIRS, m))
        for _ in range(8):
            enc.encode(ids, mask)
        ts = []
        for _ in range(40):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            enc.encode(ids, mask)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        print(f"dirs={m:05b}: {ms:.4f} ms/step {ids.shape[0] / ms:.1f}K seq/s", flush=True)
