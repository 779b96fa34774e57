"""Warp-stall samples and executed instructions aggregated per CUDA source
line of one kernel in an ncu report (sass+cuda source view):
python tools/ncu_lines.py REP.ncu-rep [n] [kernel-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
want = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
for block in out.split('"File Path",')[1:]:
    lines = block.split("\n")
    fname = lines[0]
    func = lines[1]
    if want and want not in func:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[2:]))))
    h = rows[0]
    iss = h.index("Warp Stall Sampling (All Samples)")
    iex = h.index("Instructions Executed")
    ist = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    agg = {}
    cur = None
    for r in rows[1:]:
        if len(r) <= iss:
            continue
        if r[0].strip():
            cur = (r[0], r[1].strip()[:80])
        if cur is None:
            continue
        s = int(r[iss]) if r[iss].isdigit() else 0
        e = int(r[iex]) if r[iex].isdigit() else 0
        a = agg.setdefault(cur, [0, 0, {}])
        a[0] += s
        a[1] += e
        for i, c in ist:
            if len(r) > i and r[i].isdigit():
                a[2][c] = a[2].get(c, 0) + int(r[i])
    tot = sum(v[0] for v in agg.values()) or 1
    print(f"== {fname[:60]} {func[:100]} samples {tot}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
        why = ",".join(f"{c}:{n}" for c, n in sorted(v[2].items(), key=lambda x: -x[1])[:3] if n)
        print(f"  {v[0] / tot:6.1%} {v[1]:>10d}  L{k[0]}: {k[1][:60]:60s} {why}")
