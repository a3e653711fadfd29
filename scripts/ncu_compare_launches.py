import csv, sys
def load(p):
    rows=[r for r in csv.reader(open(p)) if len(r)>10]
    h=rows[0]; iid=h.index("ID"); inm=h.index("Kernel Name"); imn=h.index("Metric Name"); iv=h.index("Metric Value"); iu=h.index("Metric Unit")
    d={}
    for r in rows[1:]:
        if r[imn]!="gpu__time_duration.sum": continue
        v=float(r[iv].replace(",",""))*{"nsecond":1e-3,"usecond":1,"msecond":1e3}.get(r[iu],1)
        d[int(r[iid])]=(r[inm][:40],v)
    return d
base=load(sys.argv[1]); others=[load(p) for p in sys.argv[2:]]
print("total", sum(v for _,v in base.values()), [sum(v for _,v in o.values()) for o in others])
for i in sorted(base):
    nm,v=base[i]
    print(i, nm, "%.1f"%v, " ".join("%.1f"%o[i][1] if i in o else "-" for o in others))
