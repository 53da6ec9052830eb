"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (csv) by kernel and grid."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
by = collections.defaultdict(list)
for d in data:
    name = d['Kernel Name'].split('(')[0]
    by[(name, d['Grid Size'])].append(float(d['Metric Value'].replace(',', '')) *
                                      scale.get(d['Metric Unit'], 1.0))
tot = sum(sum(v) for v in by.values())
print(f"launches {len(data)}  total {tot:.1f} us (serialised, cold)")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1]))[:n]:
    print(f"{sum(v):9.1f} us {100*sum(v)/tot:5.1f}%  n={len(v):4d} avg={sum(v)/len(v):7.2f}  "
          f"grid={k[1]:>14}  {k[0][:72]}")
