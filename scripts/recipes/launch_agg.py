import csv,sys,collections
f=sys.argv[1]; start=sys.argv[2] if len(sys.argv)>2 else "k_ctl_init"
rows=list(csv.reader(l for l in open(f) if not l.startswith("==")))
h=rows[0]; ix={n:i for i,n in enumerate(h)}
L=[(r[ix["Kernel Name"]].split("(")[0].replace("void ","").replace("sg::<unnamed>::","").replace("sg::",""), float(r[ix["Metric Value"]].replace(",",""))/(1000 if r[ix["Metric Unit"]]=="ns" else (1 if r[ix["Metric Unit"]]=="us" else 1e-3))) for r in rows[1:] if r[ix["Metric Name"]]=="gpu__time_duration.sum"]
idx=[i for i,x in enumerate(L) if start in x[0]]
run=L[idx[-1]:]
agg=collections.OrderedDict()
for k,t in run:
    a=agg.setdefault(k,[0,0.0]); a[0]+=1; a[1]+=t
for k,(n,t) in agg.items(): print(f"{k[:60]:<60} {n:5d} {t:10.1f} us")
print("total", round(sum(t for _,t in run),1), "launches", len(run))
