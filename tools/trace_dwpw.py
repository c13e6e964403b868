"""View FCM_TRACE stamps of a DWPW launch (CTA 0, first tiles): python tools/trace_dwpw.py trace.txt"""
import sys

blocks, cur = [], None
for ln in open(sys.argv[1]):
    if ln.startswith("#"):
        cur = [ln.strip()]
        blocks.append(cur)
    elif cur is not None and ln.strip():
        cur.append([int(x) for x in ln.split()])
tag, *rows = blocks[-1]
rows = [r for r in rows if any(r)]
t0 = min(x for r in rows for x in r if x)
names = {8: "tx_k0", 9: "tx_kN", 10: "dw_beg", 6: "dw_X0", 11: "dw_A0", 7: "dw_done", 0: "mma_te", 1: "mma_A0",
         2: "mma_cmt", 3: "epi_tf", 5: "epi_done"}
order = [8, 9, 10, 6, 11, 7, 0, 1, 2, 3, 5]
print(tag)
print("tile " + " ".join(f"{names[e]:>9s}" for e in order))
for i, r in enumerate(rows[:int(sys.argv[2]) if len(sys.argv) > 2 else 24]):
    print(f"{i:4d} " + " ".join(f"{r[e] - t0:9d}" if r[e] else f"{'-':>9s}" for e in order))
