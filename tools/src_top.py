import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
# multiple kernels may be concatenated; take first block
blocks=[]; cur=None
for r in rows:
    if r and r[0]=="Kernel Name": cur={'name':r[1],'rows':[]}; blocks.append(cur); continue
    if r and r[0]=="Address": cur['hdr']=r; continue
    if cur is not None and r: cur['rows'].append(r)
from collections import Counter
for b in blocks[:int(sys.argv[2]) if len(sys.argv)>2 else 1]:
    hdr=b['hdr']; data=b['rows']
    si=hdr.index("Warp Stall Sampling (All Samples)"); src=hdr.index("Source")
    def f(x):
        try: return float(x)
        except: return 0.0
    tot=sum(f(r[si]) for r in data)
    print(b['name'][:60], "samples", tot)
    c=Counter()
    for r in data:
        parts=r[src].split()
        if not parts: continue
        op=parts[1] if parts[0].startswith('@') else parts[0]
        c[op.split('.')[0]]+=f(r[si])
    print('  '+', '.join("%s %.1f%%"%(op,100*v/tot) for op,v in c.most_common(14)))
    for r in sorted(data,key=lambda r:-f(r[si]))[:int(sys.argv[3]) if len(sys.argv)>3 else 20]:
        print("  %5.2f%% %s"%(100*f(r[si])/tot, r[src][:100]))
