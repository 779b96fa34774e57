"""Graph-replayed C3 step time for every FF_OPT_FUSED_MASK value with PDL on
and off (median of 30, L2 flushed before each step)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2010_13382_b200 import fastformers as ffb  # noqa: E402
from paper_2010_13382_b200 import synth  # noqa: E402


def main():
    cfg = synth.config("c3").with_dtype(1)
    enc = ffb.Encoder(cfg, synth.make_weights(cfg), device=0)
    ids, mask = synth.make_inputs(cfg)
    ids, mask = torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for pdl, pdl_rr in ((1, 1), (1, 0), (0, 0)):
        ffb.check(ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_PDL, pdl))
        ffb.check(ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_PDL_RR, pdl_rr))
        for m in range(8):
            enc.set_fused(m)
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
            print(f"pdl={pdl} pdl_rr={pdl_rr} mask={m}: {ms:.4f} ms/step {256 / ms:.1f}K seq/s", flush=True)
    ffb.check(ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_PDL, 1))
    ffb.check(ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_PDL_RR, 1))


if __name__ == "__main__":
    main()
