"""Executed warp-instructions per CUDA source line of one kernel (from an ncu
report captured with --import-source on / -lineinfo):
    python tools/ncu_lines.py report.ncu-rep kernel-regex [N]"""
import collections
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", f"regex:{pat}", "--launch-count", "1"], capture_output=True, text=True).stdout
cur_file, cur = None, None
acc = collections.Counter()
text = {}
tot = 0.0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if len(r) > 7 and r[0] and r[2] == "-":  # a source line with its aggregated metrics
        cur = (cur_file, int(r[0]))
        text[cur] = r[1].strip()[:70]
        try:
            n = float(r[7] or 0)
        except ValueError:
            continue
        acc[cur] += n
        tot += n
print(f"total warp-instr {tot:.4g}")
for k, n in acc.most_common(N):
    print(f"{100 * n / tot:5.1f}%  {k[0]}:{k[1]:<5d} {text.get(k, '')}")
