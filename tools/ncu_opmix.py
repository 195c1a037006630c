"""Executed-instruction mix of one kernel in an ncu report, by SASS opcode,
weighted by execution count: python tools/ncu_opmix.py report.ncu-rep kernel-regex"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
for b in re.split(r'(?m)^"Kernel Name",', out)[1:]:
    name = b.split("\n", 1)[0]
    if not re.search(pat, name):
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    h = rows[0]
    src, ex = h.index("Source"), h.index("Instructions Executed")
    mix = collections.Counter()
    tot = 0
    for r in rows[1:]:
        try:
            n = float(r[ex] or 0)
        except ValueError:
            continue
        op = r[src].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", op).split(" ")[0].split(".")[0]
        mix[op] += n
        tot += n
    print(name[:90], f"total warp-instr {tot:.4g}")
    for op, n in mix.most_common(30):
        print(f"  {op:10s} {n:12.4g} {100 * n / tot:5.1f}%")
    break
