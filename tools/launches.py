import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; out=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            out.append((int(d['ID']), d['Kernel Name'], float(d['Metric Value'])))
bins=[i for i,(id_,k,v) in enumerate(out) if 'k_bin' in k]
seg=out[bins[-1]:]
agg=collections.OrderedDict()
for id_,k,v in seg:
    name=k[:k.index('(')] if '(' in k else k
    agg.setdefault(name,[0,0.0]); agg[name][0]+=1; agg[name][1]+=v
tot=sum(v for _,_,v in seg)
for k,(c,v) in sorted(agg.items(), key=lambda x:-x[1][1]):
    print(f"{v/1e6:8.3f} ms {100*v/tot:5.1f}%  x{c:3d}  {k[-100:]}")
print("total", tot/1e6)
