"""Aggregate an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel name.
python tools/launch_table.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[h]
ix = {k: i for i, k in enumerate(hdr)}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows[h + 1:]:
    if len(r) < len(hdr):
        continue
    name = r[ix["Kernel Name"]][:90]
    met = r[ix["Metric Name"]]
    val = float(r[ix["Metric Value"]].replace(",", ""))
    if met == "gpu__time_duration.sum":
        agg[name][0] += 1
        agg[name][1] += val
    elif "dram" in met:
        agg[name][2] += val
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:5d} {v[1] / 1e6:9.3f} ms {100 * v[1] / tot:5.1f}% {v[2] / 1e9:8.2f} GB  {k}")
