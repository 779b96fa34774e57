"""GPU-vs-oracle logit error against the oracle's own fp32-vs-fp64 drift,
row by row, on full-size int8 configs (DESIGN §3 tolerance calibration).

python tools/drift_ratio.py [config] [n_rows] [fused_mask]   (default c3 64 library default)

For each sampled row r: err[r] = max |gpu - oracle| and drift[r] = max
|oracle(acc32) - oracle|; prints the distributions and the ratio of the maxima
over random subsets of 4 and 8 rows (what the tests compare).
"""
import concurrent.futures as cf
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import Oracle  # noqa: E402
from paper_2010_13382_b200 import synth  # noqa: E402
from paper_2010_13382_b200.fastformers import Encoder  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    kw = {"fused": int(sys.argv[3])} if len(sys.argv) > 3 else {}
    cfg = synth.config(name).with_dtype(1)
    w = synth.make_weights(cfg)
    ids, mask = synth.make_inputs(cfg, seed=1000)
    got = Encoder(cfg, w, **kw).encode(torch.from_numpy(ids).cuda(), torch.from_numpy(mask).cuda()).cpu().numpy()
    orc = Oracle(cfg, w)
    rows = np.linspace(0, cfg.batch - 1, n).astype(int)

    def one(r, acc32):
        return orc.encode(ids[r:r + 1], mask[r:r + 1], acc32=acc32)[0]

    with cf.ThreadPoolExecutor(os.cpu_count()) as ex:
        ref = np.stack(list(ex.map(lambda r: one(r, False), rows)))
        d32 = np.stack(list(ex.map(lambda r: one(r, True), rows)))
    err = np.abs(got[rows] - ref).max(1)
    drift = np.abs(d32 - ref).max(1)
    print(f"{name} {kw or 'default'}: {n} rows, max|logit| {np.abs(ref).max():.3f}")
    print(f"  gpu err   : max {err.max():.3e} mean {err.mean():.3e} median {np.median(err):.3e} zero-rows {int((err == 0).sum())}")
    print(f"  drift     : max {drift.max():.3e} mean {drift.mean():.3e} median {np.median(drift):.3e}")
    print(f"  max ratio over all rows: {err.max() / drift.max():.3f}")
    rng = np.random.default_rng(0)
    for k in (4, 8):
        rs = []
        for _ in range(2000):
            sub = rng.choice(n, k, replace=False)
            rs.append(err[sub].max() / max(drift[sub].max(), 1e-30))
        rs = np.array(rs)
        print(f"  subsets of {k}: ratio median {np.median(rs):.2f} p95 {np.percentile(rs, 95):.2f} "
              f"P(ratio > 2) {np.mean(rs > 2):.3f}")
    print(f"  argmax agreement {np.mean(got[rows].argmax(1) == ref.argmax(1)):.4f}")


if __name__ == "__main__":
    main()
