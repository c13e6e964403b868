"""View FCM_TRACE stamps of a PWDW_R launch (CTA 0, first tiles): python tools/trace_pwdw.py trace.txt [rows]"""
import sys

blocks, cur = [], None
for ln in open(sys.argv[1]):
    if ln.startswith("#"):
        cur = [ln.strip()]
        blocks.append(cur)
    elif cur is not None and ln.strip():
        cur.append([int(x) for x in ln.split()])
tag, *rows = [b for b in blocks if "pwdw" in b[0]][-1]
rows = [r for r in rows if any(r)]
t0 = min(x for r in rows for x in r if x)
names = {8: "tma", 0: "mma_te", 1: "mma_X", 2: "mma_cmt", 3: "tp_tfull", 4: "tp_Tempty", 5: "tp_done",
         6: "dw_Tfull", 7: "dw_done"}
order = [8, 0, 1, 2, 3, 4, 5, 6, 7]
print(tag)
print("tile " + " ".join(f"{names[e]:>9s}" for e in order))
for i, r in enumerate(rows[:int(sys.argv[2]) if len(sys.argv) > 2 else 24]):
    print(f"{i:4d} " + " ".join(f"{r[e] - t0:9d}" if r[e] else f"{'-':>9s}" for e in order))
