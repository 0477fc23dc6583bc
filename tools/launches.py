"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]
ki, mi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
for r in rows[hdr + 1:]:
    if len(r) <= mi:
        continue
    name = r[ki].split('(')[0][:70]
    agg[name][0] += 1
    agg[name][1] += float(r[mi].replace(',', '')) * scale.get(r[ui], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"total {tot/1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{v[1]/1e3:9.3f} ms {100*v[1]/tot:5.1f}% n={v[0]:5d} avg={v[1]/v[0]:9.2f} us  {k}")
