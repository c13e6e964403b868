"""Attribute ncu source-page (SASS) samples of a warp-specialised kernel to code regions.
python tools/ncu_roles.py rep.ncu-rep [kernel-regex]  -- prints sample totals per contiguous region
between 'landmark' instructions and the top stalled instructions."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "dwpw"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# first block only
starts = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')]
blk = lines[starts[0] + 1:(starts[1] if len(starts) > 1 else len(lines))]
rows = list(csv.reader(io.StringIO("\n".join(blk))))
h = rows[0]
data = rows[1:]
iS = h.index("Warp Stall Sampling (All Samples)")
iN = h.index("Warp Stall Sampling (Not-issued Samples)")
iE = h.index("Instructions Executed")
tot = sum(int(r[iS] or 0) for r in data)
print("total samples", tot, "instructions", sum(int(r[iE] or 0) for r in data))
# regions: split at instructions that mark roles
marks = ("UTMALDG", "UTCHMMA", "UTCQMMA", "UTCIMMA", "LDTM", "FFMA2", "UTMASTG", "FHFMA", "STS", "LDS")
reg = collections.OrderedDict()
cur = None
for r in data:
    op = r[1].split()
    o = (op[1] if op and op[0].startswith("@") else (op[0] if op else ""))
    key = r[0][-5:]
    if cur is None:
        cur = key
        reg[cur] = [0, 0, 0, set()]
    s, n, e = int(r[iS] or 0), int(r[iN] or 0), int(r[iE] or 0)
    reg[cur][0] += s; reg[cur][1] += n; reg[cur][2] += e
    for m in marks:
        if o.startswith(m):
            reg[cur][3].add(m)
    if o.startswith("EXIT") or o == "BRA" and e == 0:
        cur = None
# print top regions by samples
for k, (s, n, e, m) in sorted(reg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{k} samples {s:6d} ({100*s/max(tot,1):5.1f}%) notissued {n:6d} instr {e:10d} marks {sorted(m)}")
