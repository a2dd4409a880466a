#!/usr/bin/env python
"""Per-kernel mean duration and launch count from an ncu --metrics gpu__time_duration.sum CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            unit = d.get("Metric Unit", "ns")
            v = float(d["Metric Value"].replace(",", ""))
            v = v / 1e3 if unit == "ns" else v if unit == "us" else v * 1e3 if unit == "ms" else v
            a = agg.setdefault(d["Kernel Name"][:100], [0, 0.0])
            a[0] += 1
            a[1] += v
for k, (n, v) in agg.items():
    print("%4d %10.2f us  %s" % (n, v / n, k))
