#!/usr/bin/env python3
"""Per-kernel totals of an ncu launch list (gpu__time_duration.sum csv): python tools/launch_table.py <csv>"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, d = None, collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        if x['Metric Name'] == 'gpu__time_duration.sum':
            d[x['Kernel Name'][:70]].append(float(x['Metric Value']))
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:70s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:8.2f}us share={sum(v) / tot:.3f}")
