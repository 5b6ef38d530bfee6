import csv, collections, re, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
agg=collections.defaultdict(lambda:[0,0.0])
for d in data:
    short=re.sub(r'\(.*','',d['Kernel Name'])[:60]
    key=short+" "+d['Grid Size'] if 'gemm_tc' in short else short
    agg[key][0]+=1; agg[key][1]+=float(d['Metric Value'])
tot=sum(v[1] for v in agg.values())
for k,(c,v) in sorted(agg.items(), key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 30]:
    print(f"{v/1e3:9.1f} us {100*v/tot:5.1f}% n={c:4d} avg={v/c/1e3:8.1f}us  {k}")
