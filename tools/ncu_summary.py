"""Summarise ncu output into a markdown file for profiles/.

  python tools/ncu_summary.py OUT.md --launches launches.csv [--rep a.ncu-rep ...]

* launches.csv: `ncu --metrics gpu__time_duration.sum[,...] --csv --log-file`
  of tools/prof_step.py (un-graphed forwards); the second forward is kept.
* each .ncu-rep (`--set full`): duration, tensor-pipe %, DRAM bytes, L2 %,
  registers, top stall reasons per profiled launch.
"""
import argparse
import csv
import io
import subprocess
import sys


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[hi + 1:]:
        d = per.setdefault(int(r[ii]), {"name": r[ki].split("(")[0].replace("void ", "").replace("ff::", "")})
        try:
            d[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            d[r[mi]] = r[vi]
    seq = [per[i] for i in sorted(per)]
    starts = [i for i, x in enumerate(seq) if "embed_ln" in x["name"]]
    return seq[starts[-1]:] if starts else seq[len(seq) // 2:]  # the last (warm) forward


def rep_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    res = []
    for v in r[2:]:
        d = dict(zip(h, v))
        stalls = []
        for k, val in d.items():
            if "pcsamp_warps_issue_stalled" in k and "not_issued" not in k:
                try:
                    stalls.append((float(val.replace(",", "")), k.split("stalled_")[-1]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        res.append((d, stalls[:4]))
    return res


def f(d, k, scale=1.0, fmt="{:.1f}"):
    try:
        return fmt.format(float(str(d.get(k, "nan")).replace(",", "")) * scale)
    except ValueError:
        return "-"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--launches")
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.launches:
        L = read_launches(a.launches)
        tot = sum(x.get("gpu__time_duration.sum", 0) for x in L)
        lines += [f"Launch list of one warm forward (`{a.launches}`; cold-cache, serialised by ncu: compare shares).",
                  "", "| # | kernel | us | share | extra metrics |", "|---|---|---|---|---|"]
        agg = {}
        for i, x in enumerate(L):
            t = x.get("gpu__time_duration.sum", 0)
            agg[x["name"]] = agg.get(x["name"], 0) + t
            extra = ", ".join(f"{k.split('.')[0].split('__')[-1]}={v:.3g}" for k, v in x.items()
                              if k not in ("name", "gpu__time_duration.sum") and isinstance(v, float))
            lines.append(f"| {i} | {x['name']} | {t / 1e3:.1f} | {t / tot:.1%} | {extra} |")
        lines += ["", f"Total {tot / 1e3:.1f} us.", "", "| kernel | total us | share |", "|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
            lines.append(f"| {k} | {v / 1e3:.1f} | {v / tot:.1%} |")
        lines.append("")
    for rp in a.rep:
        lines += [f"## `{rp}` (ncu --set full)", "",
                  "| kernel | grid | regs | us | tensor pipe % | DRAM read MB | DRAM write MB | L2 % | DRAM % | top stalls |",
                  "|---|---|---|---|---|---|---|---|---|---|"]
        for d, st in rep_rows(rp):
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").replace("ff::", "")
            lines.append("| {} | {} | {} | {} | {} | {} | {} | {} | {} | {} |".format(
                name, d.get("launch__grid_size", "?"), d.get("launch__registers_per_thread", "?"),
                f(d, "gpu__time_duration.sum", 1e-3 if float(str(d.get("gpu__time_duration.sum", "0")).replace(",", "")) > 1e4 else 1.0),
                f(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum"),
                f(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                f(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                ", ".join(f"{n} {v:.0f}" for v, n in st)))
        lines.append("")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
