"""SASS-level view of an ncu capture: opcode histogram and the hottest basic blocks (run here):
python tools/ncu_sass.py gpurun_out/x.ncu-rep"""
import csv
import io
import subprocess
import sys
from collections import Counter

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(int(r[iE]) for r in data)
print("warp instructions", tot, "samples", sum(int(r[iW]) for r in data))
c = Counter()
for r in data:
    t = r[iS].split()
    op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0]
    c[op] += int(r[iE])
print(" ".join(f"{op}:{n / tot * 100:.1f}%" for op, n in c.most_common(16)))
runs, start = [], 0
for k in range(1, len(data) + 1):
    if k == len(data) or data[k][iE] != data[start][iE]:
        runs.append((int(data[start][iE]) * (k - start), start, k))
        start = k
runs.sort(reverse=True)
for n, a, b in runs[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    ops = Counter()
    for j in range(a, b):
        t = data[j][iS].split()
        ops[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += 1
    st = Counter()
    for j in range(a, b):
        for r in reasons:
            st[r[6:]] += int(data[j][h.index(r)])
    print(f"{n / tot * 100:5.1f}% rows {a}-{b} x{data[a][iE]} len {b - a}: {dict(ops.most_common(6))} stalls {dict(st.most_common(5))}")
