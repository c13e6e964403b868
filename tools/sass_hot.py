"""Summarise an ncu --page source --csv --print-source sass dump: top stall lines + op mix."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
tot = sum(int(r[iS] or 0) for r in data)
print("samples", tot, "instructions", sum(int(r[iE] or 0) for r in data))
for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{int(r[iS]):6d} {int(r[iE] or 0):10d} {r[0][-5:]} {r[1][:100]}")
c = collections.Counter()
for r in data:
    op = r[1].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    c[o] += int(r[iE] or 0)
print("op mix:", ", ".join(f"{k}:{v}" for k, v in c.most_common(22)))
