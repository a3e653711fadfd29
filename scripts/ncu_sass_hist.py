"""Opcode histogram (executed warp instructions and stall samples) of one
kernel's `ncu --page source --csv --print-source sass` export."""
import csv
import sys
from collections import Counter


def main(path, top=45):
    rows = list(csv.reader(open(path)))
    h = next(r for r in rows if "Address" in r and "Source" in r)
    iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), \
        h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows:
        if len(r) <= iE or not r[iE].isdigit():
            continue
        data.append((r[iS].strip(), int(r[iE]), int(r[iW] or 0)))
    tot = sum(d[1] for d in data)
    totw = sum(d[2] for d in data)
    c, cw = Counter(), Counter()
    for s, e, w in data:
        toks = s.split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        c[op] += e
        cw[op] += w
    print(f"total warp instructions {tot}  stall samples {totw}")
    for op, n in c.most_common(top):
        print(f"{op:12s} {n:12d} {100 * n / tot:5.1f}%   samples {cw[op]:7d} ({100 * cw[op] / max(1, totw):4.1f}%)")


if __name__ == "__main__":
    main(sys.argv[1])
