#!/usr/bin/env python3
"""Mean / min duration per kernel of an ncu launch list: python tools/launch_means.py gpurun_out/launches_<tag>.csv"""
import csv, io, re, sys
from collections import defaultdict
for path in sys.argv[1:]:
    txt = open(path).read()
    rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    t = defaultdict(list)
    for r in rows[1:]:
        if len(r) > vi:
            n = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("<unnamed>::", "")
            t[n].append(float(r[vi]) / 1e3)
    print(path)
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
        print(f"  {k[:48]:48s} n={len(v):3d} mean={sum(v) / len(v):7.2f} min={min(v):7.2f}")
