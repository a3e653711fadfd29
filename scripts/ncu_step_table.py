"""Summarise an `ncu --csv --metrics ...` launch list of one step: per launch
time, instructions, issue / tensor-pipe activity, DRAM and L2 bytes."""
import csv
import re
import sys

TIME = {"usecond": 1, "us": 1, "nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}
BYTES = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3,
         "MB": 1, "GB": 1e3}


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    I, N, M, V, U = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value",
                                          "Metric Unit"))
    per, names = {}, {}
    for r in rows[1:]:
        per.setdefault(r[I], {})[r[M]] = (float(r[V].replace(",", "")), r[U])
        names[r[I]] = r[N]
    return per, names


def main(path):
    per, names = load(path)
    tot = 0.0
    print("| # | kernel | us | inst (M) | issue % | tensor % | DRAM MB | L2 MB |")
    print("|---|---|---|---|---|---|---|---|")
    agg = {}
    for i in sorted(per, key=int):
        d = per[i]
        t = d["gpu__time_duration.sum"]
        us = t[0] * TIME[t[1]]
        tot += us
        nm = re.sub(r"void quantc::kern::(\(anonymous namespace\)::)?", "", names[i])
        nm = re.sub(r"\(.*", "", nm)[:44]
        mb = lambda k: d[k][0] * BYTES[d[k][1]] if k in d else 0.0
        g = lambda k: d[k][0] if k in d else float("nan")
        print(f"| {i} | {nm} | {us:.1f} | {g('sm__inst_executed.sum') / 1e6:.2f} | "
              f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f} | "
              f"{g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.0f} | "
              f"{mb('dram__bytes_read.sum') + mb('dram__bytes_write.sum'):.1f} | "
              f"{mb('lts__t_bytes.sum'):.1f} |")
        a = agg.setdefault(nm, [0, 0.0])
        a[0] += 1
        a[1] += us
    print(f"\ntotal {tot:.1f} us over {len(per)} launches")
    for nm, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {us:8.1f} us {100 * us / tot:5.1f}% n={n:3d} {nm}")


if __name__ == "__main__":
    main(sys.argv[1])
