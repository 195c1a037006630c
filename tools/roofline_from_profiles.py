"""Recomputes bench.py's roofline rows from a committed capture round:
profiles/<tag>_bench.json (counts, CUDA-event stage times, clocks) and, for the
ncu view, profiles/<tag>_launches.md (cold-cache, serialised per-kernel times).

    python tools/roofline_from_profiles.py r2c
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r2c"
b = json.load(open(os.path.join(ROOT, "profiles", f"{tag}_bench.json")))
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
c, s = b["counts"], b["stages_ms"]
mhz = b["clocks"]["sm_mhz"] or 1965.0
alu = 148 * 128 * mhz * 1e6 / 1e12
P, V, K = c["particles"], c["visible"], 16
s1 = 48 * P + (12 * K + 56) * V + 4 * (P - V)
ncu = {}
p = os.path.join(ROOT, "profiles", f"{tag}_launches.md")
if os.path.exists(p):
    for ln in open(p):
        m = re.match(r"\| `([^`]+)` \| 1 \| ([\d.]+) \|", ln)
        if m:
            ncu[m.group(1)] = float(m.group(2)) / 1e3
rows = [
    ("render_bwd_tiles (K7)", 45 * c["sum_n_contrib"] / 1e12, alu, s["render_bwd_tiles"], "render_bwd_kernel<4, 0>"),
    ("render_fwd (K6)", 15 * c["evals_fwd"] / 1e12, alu, s["render_fwd"], "render_fwd_kernel<2, 0, 0>"),
    ("preprocess (K1)", s1 / 1e9, peaks["hbm_gbs"], s["preprocess"], "preprocess_tma_kernel<16>"),
]
print(f"{'row':24s} {'work':>10s} {'event ms':>9s} {'frac':>6s} {'ncu ms':>7s} {'frac(ncu)':>9s}")
for name, work, peak, ms, kern in rows:
    nm = ncu.get(kern)
    f = work / (ms / 1e3) / peak
    fn = work / (nm / 1e3) / peak if nm else float("nan")
    print(f"{name:24s} {work:10.4g} {ms:9.4f} {f:6.3f} {nm if nm else float('nan'):7.4f} {fn:9.3f}")
print("bench line:", {k: round(v["frac"], 3) for k, v in b["roofline"]["all"].items()})
