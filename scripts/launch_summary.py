"""Summarise an ncu --csv launch list (one step): per kernel time share and,
when captured, DRAM bytes per launch.

usage: python scripts/launch_summary.py launches.csv [--md out.md] [--json out.json]
"""
import csv
import json
import sys
from collections import OrderedDict, defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("ID"))
    gi = h.index("Grid Size") if "Grid Size" in h else None
    launches = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        d = launches.setdefault(r[ii], {"kernel": r[ki], "grid": r[gi] if gi is not None else ""})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return list(launches.values())


def short(name):
    n = name.split("(")[0]
    return n.replace("void ", "").replace("quantc::kern::", "").replace("(anonymous namespace)::", "")


def main():
    args = sys.argv[1:]
    path = args[0]
    L = load(path)
    tot = sum(x.get("gpu__time_duration.sum", 0.0) for x in L)
    by = defaultdict(lambda: [0.0, 0, 0.0])
    for x in L:
        k = short(x["kernel"])
        by[k][0] += x.get("gpu__time_duration.sum", 0.0)
        by[k][1] += 1
        by[k][2] += x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)
    lines = [f"total {tot / 1e3:.1f} us over {len(L)} launches"]
    for k, (t, n, b) in sorted(by.items(), key=lambda kv: -kv[1][0]):
        extra = f"  dram {b / n / 1e6:8.1f} MB/launch" if b else ""
        lines.append(f"  {t / 1e3:8.1f} us {100 * t / tot:5.1f}% n={n:3d} {k}{extra}")
    print("\n".join(lines))
    if "--md" in args:
        out = args[args.index("--md") + 1]
        with open(out, "w") as f:
            f.write("| # | kernel | grid | time (us) | DRAM read (MB) | DRAM write (MB) |\n")
            f.write("|---|---|---|---|---|---|\n")
            for i, x in enumerate(L):
                f.write(f"| {i} | {short(x['kernel'])} | {x['grid']} | "
                        f"{x.get('gpu__time_duration.sum', 0) / 1e3:.1f} | "
                        f"{x.get('dram__bytes_read.sum', 0) / 1e6:.1f} | "
                        f"{x.get('dram__bytes_write.sum', 0) / 1e6:.1f} |\n")
            f.write("\n```\n" + "\n".join(lines) + "\n```\n")
    if "--json" in args:
        out = args[args.index("--json") + 1]
        tc = [x for x in L if "tc_conv_kernel" in x["kernel"]]
        d = {"total_us": tot / 1e3, "launches": len(L),
             "tc_conv_launches": len(tc),
             "tc_conv_us": sum(x.get("gpu__time_duration.sum", 0) for x in tc) / 1e3,
             "tc_conv_dram_bytes_per_launch": (sum(x.get("dram__bytes_read.sum", 0) +
                                                   x.get("dram__bytes_write.sum", 0) for x in tc)
                                               / max(1, len(tc)))}
        json.dump(d, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
