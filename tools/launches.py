import csv, collections, sys
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
    h = rows[hi]; data = rows[hi + 1:]
    ki = h.index('Kernel Name'); vi = h.index('Metric Value')
    agg = collections.OrderedDict()
    for r in data:
        agg.setdefault(r[ki][:60], []).append(float(r[vi].replace(',', '')))
    print("==", f)
    for k, v in agg.items():
        if 'native::' in k or 'spin_kernel' in k:
            continue
        print(f"  {k:60s} n={len(v):3d} mean={sum(v)/len(v)/1e3:8.2f} us  min={min(v)/1e3:.2f}")
