"""View chunk-level FCM_TRACE stamps of a DWPW launch (libfcm built with -DFCM_TRACE_STAMPS -DFCM_TRACE_CHUNK)."""
import sys

rows, cur = [], None
for ln in open(sys.argv[1]):
    if ln.startswith("#"):
        rows = []
        continue
    if ln.strip():
        rows.append([int(x) for x in ln.split()])
rows = [r for r in rows if any(r)]
t0 = min(x for r in rows for x in r if x)
names = {8: "tx", 0: "rl_X", 1: "rl_A", 2: "dw_bar", 3: "dw_go", 4: "dw0_end", 5: "dw7_end", 6: "mma_A", 7: "mma_cmt"}
order = [8, 0, 1, 2, 3, 4, 5, 6, 7]
print("chunk " + " ".join(f"{names[e]:>8s}" for e in order))
for i, r in enumerate(rows[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]):
    print(f"{i:5d} " + " ".join(f"{r[e] - t0:8d}" if r[e] else f"{'-':>8s}" for e in order))
