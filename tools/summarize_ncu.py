"""Summaries of ncu outputs for profiles/ (markdown).

    python tools/summarize_ncu.py launches <launches.csv>      # per-kernel device time
    python tools/summarize_ncu.py full <report.ncu-rep>        # key metrics per captured kernel
    python tools/summarize_ncu.py traffic <report.ncu-rep>...  # JSON: DRAM bytes per launch per kernel
"""
import json
import re
import collections
import os
import csv
import io
import subprocess
import sys


# launches of each kernel in one bench step
STEP = {"preprocess_tma_kernel<16>": 1, "depth_sort_kernel": 1, "bin_rows_kernel<2>": 1, "bin_cols_count_kernel<3>": 1,
        "bin_cols_kernel<3>": 1, "render_fwd_kernel<2, 0, 0>": 1, "render_bwd_kernel<4, 0>": 1,
        "particle_bwd_tma_kernel<16>": 1}


def share(path):
    """Per-step share of each kernel from the launch list (median x launches per step)."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in data:
        k = r[ki].split("(")[0].replace("void ", "").replace("ges::", "")
        agg[k].append(float(r[vi]) / 1000.0)
    tot = 0.0
    out = []
    for k, n in STEP.items():
        v = sorted(agg.get(k, [0.0]))
        t = v[len(v) // 2] * n
        out.append((k, n, t))
        tot += t
    print("| kernel | per step | us per step (median x n) | share |")
    print("|---|---|---|---|")
    for k, n, t in out:
        print(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    print(f"| total | | {tot:.1f} | |")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    order, agg = [], collections.defaultdict(list)
    for r in data:
        k = r[ki].split("(")[0]
        if k not in agg:
            order.append(k)
        agg[k].append(float(r[vi]) / 1000.0)
    print("| kernel | launches | median us | min us | max us |")
    print("|---|---|---|---|---|")
    for k in order:
        v = sorted(agg[k])
        print(f"| `{k}` | {len(v)} | {v[len(v) // 2]:.1f} | {v[0]:.1f} | {v[-1]:.1f} |")


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
        "Executed Ipc Active", "Achieved Occupancy", "Registers Per Thread", "L2 Hit Rate"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"]


def full(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[ii], r[ki].split("(")[0])
        if r[mi] in WANT:
            per.setdefault(key, {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hr = rr[0]
    units = rr[1]
    rawv = {}
    for row in rr[2:]:
        key = (row[hr.index("ID")], row[hr.index("Kernel Name")].split("(")[0])
        rawv[key] = {m: f"{row[hr.index(m)]} {units[hr.index(m)]}" for m in RAW if m in hr}
    cols = WANT + RAW
    print("| id | kernel | " + " | ".join(cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    for key, d in per.items():
        d.update(rawv.get(key, {}))
        print(f"| {key[0]} | `{key[1]}` | " + " | ".join(d.get(c, "") for c in cols) + " |")


def _bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return float(v.replace(",", "")) * scale.get(unit.strip(), 1.0)


def traffic(*paths):
    """dram__bytes_read.sum + dram__bytes_write.sum per captured launch, keyed by the
    kernel's base name (template arguments dropped): what bench.py reports as
    roofline.traffic for its dominant kernel."""
    out = {}
    for path in paths:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(io.StringIO(raw)))
        hr, units = rr[0], rr[1]
        for row in rr[2:]:
            name = row[hr.index("Kernel Name")].split("(")[0]
            base = re.sub(r"<.*", "", name.replace("void ", "")).split("::")[-1]
            rd = _bytes(row[hr.index("dram__bytes_read.sum")], units[hr.index("dram__bytes_read.sum")])
            wr = _bytes(row[hr.index("dram__bytes_write.sum")], units[hr.index("dram__bytes_write.sum")])
            dur = row[hr.index("gpu__time_duration.sum")] if "gpu__time_duration.sum" in hr else ""
            out[base] = {"kernel": name, "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
                         "duration": f"{dur} {units[hr.index('gpu__time_duration.sum')]}" if dur else None,
                         "report": os.path.basename(path)}
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    {"launches": launches, "share": share, "full": full, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
