#!/usr/bin/env python3
"""Print an ncu --csv launch list (one line per launch, metrics as columns)."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    H = rows[h]
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        d = dict(zip(H, r))
        try:
            v = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        agg.setdefault((d["ID"], d["Kernel Name"][:28]), {})[d["Metric Name"]] = v
    print("#", path)
    for (i, k), m in agg.items():
        print(i, k, " ".join(f"{n.split('__')[1][:22]}={v:.4g}" for n, v in m.items()))
