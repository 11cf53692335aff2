"""Aggregate an ncu `--page source --print-source cuda,sass --csv` dump per
CUDA source line: instructions executed and warp-stall samples."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
file = None
hdr = None
agg = defaultdict(lambda: [0, 0, ""])
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        i_inst = hdr.index("Instructions Executed")
        i_samp = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None:
        continue
    if r[0]:
        cur = (file, int(r[0]))
        agg[cur][2] = r[1].strip()[:90]
    if len(r) > i_inst and r[2]:
        try:
            agg[cur][0] += int(float(r[i_inst] or 0))
            agg[cur][1] += int(float(r[i_samp] or 0))
        except ValueError:
            pass
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {tot_i:,}  stall samples {tot_s:,}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:<5} inst {v[0]:>12,} ({100*v[0]/tot_i:5.1f}%)  samp {100*v[1]/tot_s:5.1f}%  {v[2]}")
