"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel totals of the second half."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
hdr, data = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
start = int(len(data) * (1 - frac))
for d in data[start:]:
    v = float(d['Metric Value'].replace(',', ''))
    unit = d['Metric Unit']
    us = v / 1000.0 if unit in ('nsecond', 'ns') else (v if unit in ('usecond', 'us') else v * 1000.0)
    agg[d['Kernel Name'][:60]][0] += 1
    agg[d['Kernel Name'][:60]][1] += us
tot = sum(v[1] for v in agg.values())
print(f"{len(data) - start} launches, {tot / 1e3:.2f} ms kernel time")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 16]:
    print(f"{v[1] / 1e3:9.3f} ms {v[0]:6d} calls {v[1] / v[0]:9.2f} us/call  {k}")
