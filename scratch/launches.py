import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
def us(d):
    v=float(d['Metric Value'].replace(',','')); u=d['Metric Unit']
    return v/1000 if u=='nsecond' else (v if u=='usecond' else v*1000)
agg=collections.defaultdict(lambda:[0,0.0])
for d in data:
    name=d['Kernel Name'].split('(')[0]
    agg[name][0]+=1; agg[name][1]+=us(d)
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1]):
    print("%-60s n=%4d total=%9.1f us avg=%8.2f us share=%5.1f%%"%(k[:60],v[0],v[1],v[1]/v[0],100*v[1]/tot))
print("total us", tot)
if len(sys.argv)>2:
    for d in data:
        if sys.argv[2] in d['Kernel Name']: print(d['Kernel Name'][:70], d['Grid Size'], "%.1f"%us(d))
