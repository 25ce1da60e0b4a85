"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name (microseconds)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.defaultdict(lambda: [0, 0.0])
scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3, 'second': 1e6, 's': 1e6}
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['Metric Name'] != 'gpu__time_duration.sum': continue
        v = float(d['Metric Value'].replace(',', '')) * scale[d['Metric Unit']]
        k = d['Kernel Name'][:80]
        agg[k][0] += 1; agg[k][1] += v
tot = sum(a[1] for a in agg.values())
print(f'total {tot/1e3:.2f} ms')
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{t/1e3:9.3f} ms {n:5d}  {k}")
