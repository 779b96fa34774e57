"""A/B probe of a per-model kernel option on the C3 forward: device time per
step (graph replay, L2 flushed before each step, median of 30) and the
per-launch GEMM times of one profiled forward (first layer's four GEMMs).

python tools/ab_probe.py [option_name] [dtype i8|f16]   (default fused7 i8)
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2010_13382_b200 import synth  # noqa: E402
from paper_2010_13382_b200 import fastformers as ffb  # noqa: E402

OPTS = {"pdl": lambda enc, on: ffb.check(ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_PDL, 1 if on else 0)),
        "pdl_rr": lambda enc, on: ffb.check(ffb.lib().ff_set_option(enc.h, ffb.FF_OPT_PDL_RR, 1 if on else 0))}
for _m in range(1, 8):  # FF_OPT_FUSED_MASK bits: 1 out-proj+LN1, 2 FFN1+requant, 4 FFN2+LN2
    OPTS[f"fused{_m}"] = (lambda m: lambda enc, on: enc.set_fused(m if on else 0))(_m)


def main():
    opt = sys.argv[1] if len(sys.argv) > 1 else "fused7"
    dtype = 1 if (sys.argv[2] if len(sys.argv) > 2 else "i8") == "i8" else 0
    cfg = synth.config("c3").with_dtype(dtype)
    w = synth.make_weights(cfg)
    enc = ffb.Encoder(cfg, w, device=0)
    ids, mask = synth.make_inputs(cfg)
    ids, mask = torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    res = {}
    for rep in range(2):
        for on in (False, True):
            OPTS[opt](enc, on)
            ref = enc.encode(ids, mask).clone()
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
            ms = sorted(ts)[len(ts) // 2]
            prof = enc.profile(ids, mask)
            gem = [round(t * 1e3, 1) for k, t in prof][:9]
            gsum = sum(t for k, t in prof if k.startswith("gemm")) * 1e3
            res.setdefault(on, []).append(ms)
            print(f"{opt}={int(on)} {'i8' if dtype else 'f16'}: {ms:.4f} ms/step {256 / ms:.1f}K seq/s; "
                  f"GEMMs total {gsum:.0f} us, first launches {gem}", flush=True)
            if on:
                print(f"  max |logits(on) - logits(off)| = {float((ref - res_ref).abs().max()):.3e}", flush=True)
            else:
                res_ref = ref
    OPTS[opt](enc, False)


if __name__ == "__main__":
    main()
