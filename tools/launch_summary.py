import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
agg = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0]; v = float(r[vi].replace(',', ''))
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += v
tot = sum(a[1] for a in agg.values())
print("| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("| %s | %d | %.3f | %.1f%% |" % (k, c, t / 1e6, 100 * t / tot))
