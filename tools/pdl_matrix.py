"""Graph-replayed C3 int8 step time with PDL disabled for one kernel kind at a
time (FF_OPT_PDL_KINDS), default fusion mask; median of 30, L2 flushed."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2010_13382_b200 import fastformers as ffb  # noqa: E402
from paper_2010_13382_b200 import synth  # noqa: E402


def main():
    cfg = synth.config("c3").with_dtype(1 if (sys.argv[1] if len(sys.argv) > 1 else "i8") == "i8" else 0)
    enc = ffb.Encoder(cfg, synth.make_weights(cfg), device=0)
    ids, mask = synth.make_inputs(cfg)
    ids, mask = torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    cases = [("all", 0xFFFF)] + [(f"no_{k}", 0xFFFF & ~(1 << i)) for i, k in enumerate(ffb.KERNEL_KINDS)] + \
            [("none", 0)]
    for rep in range(2):
        for name, m in cases:
            ffb.check(ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_PDL_KINDS, m))
            for _ in range(5):
                enc.encode(ids, mask)
            ts = []
            for _ in range(30):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                enc.encode(ids, mask)
                e1.record(st)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[15]
            print(f"{name:16s}: {ms:.4f} ms/step {256 / ms:.1f}K seq/s", flush=True)
    ffb.check(ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_PDL_KINDS, 0xFFFF))


if __name__ == "__main__":
    main()
