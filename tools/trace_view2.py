import sys
blocks=[];cur=None
for l in open(sys.argv[1]):
    if l.startswith('#'): cur=[];blocks.append((l.strip(),cur));continue
    cur.append([int(x) for x in l.split()])
tag,rows=blocks[-1]
rows=[r for r in rows if r[0]>0]
t0=min(min(x for x in r if x) for r in rows)
names=["mma_tempty","mma_full","mma_commit","epi_tfull","epi_bufok","epi_done","epi_ld","epi_math","tma_first"]
print(tag); print("tile " + " ".join(f"{n:>10s}" for n in names))
for i,r in enumerate(rows[:20]):
    print(f"{i:4d} " + " ".join(f"{(x-t0):10d}" if x else f"{'-':>10s}" for x in r[:9]))
