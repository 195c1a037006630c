"""Per-kernel device times of one bench-workload step (from an ncu csv written
with --metrics gpu__time_duration.sum --csv): python tools/ktimes.py file.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
acc = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            acc[d["Kernel Name"].split("(")[0][:50]].append(float(d["Metric Value"]) / 1e3)
tot = 0
for k, v in acc.items():
    print(f"{k:50s} n={len(v):3d} mean={sum(v)/len(v):8.1f} us  sum={sum(v):8.1f}")
    tot += sum(v)
print(f"total {tot:.1f} us")
