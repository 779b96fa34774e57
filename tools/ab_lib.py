"""A/B of two builds of the library on the C3 int8 step, in one process per
build, alternating: python tools/ab_lib.py LIB_A LIB_B [rounds]
Each run: device time per step (graph replay, L2 flushed before each step,
median of 40) and the per-launch times of one profiled forward by kernel role.
"""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import torch

    sys.path.insert(0, ".")
    from paper_2010_13382_b200 import synth  # noqa: E402
    from paper_2010_13382_b200 import fastformers as ffb  # noqa: E402

    cfg = synth.config(os.environ.get("AB_CONFIG", "c3")).with_dtype(1)
    enc = ffb.Encoder(cfg, synth.make_weights(cfg), device=0)
    ids, mask = synth.make_inputs(cfg)
    ids, mask = torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(10):
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
    prof = enc.profile(ids, mask)
    by = {}
    for k, t in prof:
        by.setdefault(k, []).append(t * 1e3)
    roles = " ".join(f"{k}={sum(v) / len(v):.1f}" for k, v in by.items())
    print(f"{os.environ.get('FF_LIB_PATH', 'default')}: {ms:.4f} ms/step {ids.shape[0] / ms:.1f}K seq/s | {roles}",
          flush=True)
    sys.exit(0)

libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
for r in range(rounds):
    for lb in libs:
        env = dict(os.environ, FF_LIB_PATH=os.path.abspath(lb))
        subprocess.run([sys.executable, __file__, "--one"], env=env, check=True)
