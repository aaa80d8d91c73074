"""Summarise an ncu --csv launch list (gpu__time_duration per launch) by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    k = d['Kernel Name'].split('(')[0][:48]; v = float(d['Metric Value'].replace(',', ''))
    agg[k][0] += 1; agg[k][1] += v
tot = sum(t for _, t in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:6d} launches {t/1e6:10.3f} ms  share {100*t/tot:5.1f}%  avg {t/c/1e3:9.2f} us  {k}")
