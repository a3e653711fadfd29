"""Summarise an ncu --set full report's SASS source page: stall reasons per
code region (address buckets) and the top stalled instructions.
usage: python scripts/ncu_stalls.py report.ncu-rep [lo_hex hi_hex]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = rows[2:]
ad, src = h.index("Address"), h.index("Source")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
base = int(data[0][ad], 16)
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
tot = defaultdict(int)
for r in data:
    off = int(r[ad], 16) - base
    if lo <= off < hi:
        for c in reasons:
            tot[c] += int(r[h.index(c)] or 0)
s = sum(tot.values()) or 1
print("stall reasons in [%x, %x):" % (lo, min(hi, 1 << 32)))
for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print("  %-24s %6d  %5.1f%%" % (c, v, 100.0 * v / s))
