"""Warp-stall samples per CUDA source line of one kernel (ncu report captured with
--import-source on, code built with -lineinfo):
    python tools/ncu_stall_lines.py report.ncu-rep kernel-regex [N]"""
import collections
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", f"regex:{pat}", "--launch-count", "1"], capture_output=True, text=True).stdout
cur_file, head = None, None
acc, text, inst = collections.Counter(), {}, collections.Counter()
stall = collections.defaultdict(collections.Counter)
tot = 0.0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        head = r
        continue
    if head is None or len(r) < 8 or r[2] != "-":   # source-line rows carry the aggregated metrics
        continue
    try:
        s = float(r[4] or 0)
        ie = float(r[7] or 0)
    except ValueError:
        continue
    key = (cur_file, int(r[0]))
    text[key] = r[1].strip()[:72]
    acc[key] += s
    inst[key] += ie
    tot += s
    for i, c in enumerate(head):
        if c.startswith("stall_") and i < len(r):
            try:
                stall[key][c] += float(r[i] or 0)
            except ValueError:
                pass
print(f"total stall samples {tot:.0f}")
for k, n in acc.most_common(N):
    top = ", ".join(f"{c[6:]}={int(v)}" for c, v in stall[k].most_common(2) if v)
    print(f"{100 * n / max(tot, 1):5.1f}% {k[0]}:{k[1]:<4d} inst={inst[k]:9.3g} {text.get(k, ''):72s} {top}")
