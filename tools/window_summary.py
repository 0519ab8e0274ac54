import csv, sys
from collections import defaultdict
path, first, title = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows=[r for r in csv.reader(l for l in open(path) if l.startswith('"')) if len(r)>10]
h=rows[0]; data=[dict(zip(h,r)) for r in rows[1:]]
starts=[i for i,d in enumerate(data) if 'k_zero_flags' in d['Kernel Name']]
U={"ns":1e-3,"nsecond":1e-3,"us":1.0,"usecond":1.0,"ms":1e3,"msecond":1e3}
def nm(d):
    n=d['Kernel Name'].split('(')[0].replace('void ','').replace('mrlbm_b200::','')
    return 'k_stream_collide'+n[n.find('<'):] if 'k_stream_collide' in n else n.split('<')[0]
acc=defaultdict(float); cnt=defaultdict(int); per=[]
for si,a in enumerate(starts):
    b=starts[si+1] if si+1<len(starts) else len(data)
    t=0
    for d in data[a:b]:
        us=float(d['Metric Value'].replace(',',''))*U[d['Metric Unit']]
        acc[nm(d)]+=us; cnt[nm(d)]+=1; t+=us
    per.append((b-a,t))
print(title)
print("ncu --metrics gpu__time_duration.sum --clock-control none; cold caches, serialised: read shares, not absolutes.")
for i,(n,t) in enumerate(per): print(f"step {first+i}: {n} launches, {t:8.1f} us")
tot=sum(acc.values())
print(f"total {tot:.1f} us = {tot/len(per):.1f} us/step")
for k,v in sorted(acc.items(), key=lambda kv:-kv[1]):
    print(f"{v/len(per):9.1f} us/step {100*v/tot:5.1f}%  x{cnt[k]//len(per):3d}/step  {k}")
