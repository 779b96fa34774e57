"""Print per-stage lockstep statistics (GPU vs oracle fed the GPU's stage input)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_model import build_case, dev, f32
import oracle
from oracle import Oracle
from paper_2010_13382_b200.fastformers import Encoder

names = sys.argv[1:] or ["c1_f16", "c2_i8", "c3_i8", "c3_f16"]
for name in names:
    cfg, w, ids, mask = build_case(name)
    enc, orc = Encoder(cfg, w), Oracle(cfg, w)
    B, S = ids.shape
    for l in [0, cfg.num_layers - 1]:
        t = {k: f32(v) for k, v in enc.trace(dev(ids), dev(mask), l).items()}
        for key, st, a, b in [("qkv", oracle.ST_QKV, t["x_in"], None), ("ctx", oracle.ST_ATTN, t["qkv"], None),
                              ("o", oracle.ST_OPROJ, t["ctx"], None), ("h1", oracle.ST_LN1, t["o"], t["x_in"]),
                              ("i", oracle.ST_FFN1, t["h1"], None), ("y", oracle.ST_FFN2, t["i"], None),
                              ("x_out", oracle.ST_LN2, t["y"], t["h1"])]:
            ref = orc.stage(l, st, a, b, mask=mask, B=B, S=S)
            got = t[key]
            d = np.abs(got.astype(np.float64) - ref)
            nd = int((d > 0).sum())
            rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
            big = d > (np.abs(ref) * 2.0 ** -10 + 2.0 ** -14)
            where = np.argwhere(d == d.max())[0] if nd else None
            print(f"{name} L{l} {key:6s} ndiff={nd:7d}/{d.size} maxabs={d.max():.3e} rel={rel:.2e} big={int(big.sum())}"
                  f" at={where} got={got[tuple(where)] if nd else ''} ref={ref[tuple(where)] if nd else ''}", flush=True)
