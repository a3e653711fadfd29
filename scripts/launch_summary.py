"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0, []])
    tot = 0.0
    for d in data:
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"])
        u = d["Metric Unit"]
        ns = v * 1e3 if u == "usecond" else (v * 1e6 if u == "msecond" else v)
        agg[name][0] += 1
        agg[name][1] += ns
        agg[name][2].append((ns, d.get("Grid Size", "")))
        tot += ns
    print(f"total {tot/1e6:.3f} ms over {len(data)} launches")
    for k, (n, t, lst) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t/1e6:8.3f} ms {100*t/tot:5.1f}% n={n:4d} {k}")
    return agg


if __name__ == "__main__":
    main(sys.argv[1])
