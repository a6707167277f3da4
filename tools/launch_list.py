import csv, sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; out=[]
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            out.append((d['Kernel Name'].split('(')[0][:40], float(d['Metric Value']), d.get('Grid Size','')))
tot=sum(v for _,v,_ in out)
agg=defaultdict(float); cnt=defaultdict(int)
for k,v,_ in out: agg[k]+=v; cnt[k]+=1
for k,v in sorted(agg.items(), key=lambda x:-x[1]): print(f"{v/1e3:9.1f} us {100*v/tot:5.1f}% x{cnt[k]:3d} {k}")
print('total us', tot/1e3, 'launches', len(out))
if len(sys.argv)>2:
    for k,v,g in out: print(f"{v/1e3:8.1f} {k} {g}")
