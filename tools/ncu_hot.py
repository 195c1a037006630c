"""Print the hottest SASS instructions (by warp-stall samples) of an ncu report,
one kernel at a time: python tools/ncu_hot.py report.ncu-rep [kernel-regex] [N]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else "."
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
blocks = re.split(r'(?m)^"Kernel Name",', out)
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if not re.search(pat, name):
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    h = rows[0]
    si = h.index("Warp Stall Sampling (All Samples)")
    src = h.index("Source")
    ex = h.index("Instructions Executed")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    data = []
    tot = 0
    for r in rows[1:]:
        try:
            s = float(r[si] or 0)
        except ValueError:
            continue
        tot += s
        top = sorted(((float(r[i] or 0), h[i]) for i in stall_cols), reverse=True)[:2]
        data.append((s, r[0], r[src], r[ex], top))
    print(f"=== {name[:80]}  total samples {tot:.0f}")
    for s, addr, sass, ex_, top in sorted(data, reverse=True)[:N]:
        print(f"{100*s/tot:5.1f}% {addr} {sass[:60]:60s} exec={ex_} {[(t[1], int(t[0])) for t in top]}")
