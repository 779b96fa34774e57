"""Top stalled SASS instructions per kernel of an ncu report (--page source):
python tools/ncu_hot_sass.py REP.ncu-rep [kernel-substring] [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name",')
for b in blocks[1:]:
    name, rest = b.split("\n", 1)
    if want and want not in name:
        continue
    rows = list(csv.reader(io.StringIO(rest)))
    h = rows[0]
    ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[iss]) for r in rows[1:] if len(r) > iss and r[iss].isdigit())
    top = sorted((r for r in rows[1:] if len(r) > iss and r[iss].isdigit()), key=lambda r: -int(r[iss]))[:n]
    print(f"== {name[:110]}  total samples {tot}")
    for r in top:
        print(f"  {int(r[iss]) / max(tot, 1):6.1%}  {r[isrc].strip()[:90]}")


def by_opcode(rep, want):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    for b in out.split('"Kernel Name",')[1:]:
        name, rest = b.split("\n", 1)
        if want and want not in name:
            continue
        rows = list(csv.reader(io.StringIO(rest)))
        h = rows[0]
        isrc, iss, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        agg, ex = {}, {}
        for r in rows[1:]:
            if len(r) <= iss or not r[iss].isdigit():
                continue
            toks = r[isrc].split()
            op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
            op = op.split(".")[0]
            agg[op] = agg.get(op, 0) + int(r[iss])
            ex[op] = ex.get(op, 0) + int(r[iex] or 0)
        tot = sum(agg.values())
        print(f"-- by opcode: {name[:80]}")
        for op, v in sorted(agg.items(), key=lambda kv: -kv[1])[:22]:
            print(f"  {v / tot:6.1%} samples  {ex[op]:>10d} warp-instr  {op}")


if len(sys.argv) > 4 and sys.argv[4] == "op":
    by_opcode(rep, want)
