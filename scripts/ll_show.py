import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
for i,r in enumerate(rows):
    if r and r[0]=='ID': hdr=i;break
h=rows[hdr]; data=rows[hdr+1:]
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size')
out=[(r[ki][:50], float(r[vi]), r[gi]) for r in data]
idx=[i for i,(k,v,g) in enumerate(out) if 'distribution' in k]
end=idx[0]
first=sys.argv[2]
starts=[i for i,(k,v,g) in enumerate(out[:end]) if first in k]
step=out[starts[-1]:end]
tot=sum(v for k,v,g in step); lay=0
thr=float(sys.argv[3]) if len(sys.argv)>3 else 0
for k,v,g in step:
    if 'umma' not in k: lay+=v
    if v>=thr: print(f"{v/1000:9.3f} us {g:>14} {k}")
print("total", tot/1e6, "ms; non-umma", lay/1e6, "launches", len(step))
