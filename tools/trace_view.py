import sys
lines=[l.split() for l in open(sys.argv[1]) if not l.startswith('#')]
rows=[[int(x) for x in l] for l in lines if l and int(l[0])>0][-64:]
t0=min(r[0] for r in rows)
names=["mma_tempty","mma_full","mma_commit","T_tfull","T_Tempty","T_done","DW_Tfull","DW_done","tma_empty"]
print("tile " + " ".join(f"{n:>10s}" for n in names))
for i,r in enumerate(rows[:40]):
    print(f"{i:4d} " + " ".join(f"{(x-t0):10d}" if x else f"{'-':>10s}" for x in r[:9]))
