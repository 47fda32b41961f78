import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
tot=collections.defaultdict(float); cnt=collections.Counter()
for r in rows[hdr+1:]:
    if len(r)<=vi: continue
    try: v=float(r[vi].replace(',',''))
    except: continue
    k=r[ki][:50]; tot[k]+=v; cnt[k]+=1
div=float(sys.argv[2]) if len(sys.argv)>2 else 1
for k,v in sorted(tot.items(), key=lambda x:-x[1]): print(f"{v/1e3/div:9.1f} us/call  {cnt[k]/div:5.1f}/call  {v/1e3/cnt[k]:8.1f} us/launch  {k}")
print("total us/call", sum(tot.values())/1e3/div)
