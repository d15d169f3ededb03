"""Summarise an ncu --csv launch list (gpu__time_duration.sum): kernels > 8 us and the small-kernel total."""
import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
tot=sum(float(d['Metric Value']) for d in data)
print(len(data),"launches, total us %.1f"%(tot/1e3))
for j,d in enumerate(data):
    t=float(d['Metric Value'])
    if t>8000: print(j, "%7.1f us"%(t/1e3), d['Grid Size'], d['Kernel Name'][:60])
small=[float(d['Metric Value']) for d in data if float(d['Metric Value'])<=8000]
print("small kernels", len(small), "%.1f us"%(sum(small)/1e3))
