import csv,collections,sys
for f in sys.argv[1:]:
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value'); ui=hdr.index('Metric Unit')
    d=collections.defaultdict(list)
    for r in rows[1:]:
        d[r[ki][:40]].append(float(r[vi].replace(',','')))
    print(f, rows[1][ui])
    for k,v in d.items(): print('  %-42s n=%d mean=%.1f min=%.1f'%(k,len(v),sum(v)/len(v),min(v)))
