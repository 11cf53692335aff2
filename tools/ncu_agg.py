"""Aggregate an ncu --metrics CSV launch list per kernel (sums; pct metrics averaged)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
idx = {h: j for j, h in enumerate(rows[start])}
agg = collections.defaultdict(lambda: collections.defaultdict(float)); cnt = collections.Counter()
for r in rows[start + 1:]:
    k = r[idx['Kernel Name']][:36]; m = r[idx['Metric Name']]
    agg[k][m] += float(r[idx['Metric Value']].replace(',', ''))
    if m == 'gpu__time_duration.sum': cnt[k] += 1
for k in agg:
    d = {m: (v / cnt[k] if ('pct' in m or 'rate' in m) else v) for m, v in agg[k].items()}
    print(f"{k:38s} n={cnt[k]:3d} " + " ".join(f"{m.split('.')[0].replace('__','.')}={v:.4g}" for m, v in d.items()))
