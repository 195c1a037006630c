"""Pipe / issue / atomic counters per kernel from an `ncu --set full` report, for profiles/.

    python tools/pipes.py <report.ncu-rep> [--json out.json] [--md out.md]

SURVEY.md §8(d) names the evidence for the compositing kernels (K6/K7): FP32 (FMA) and ALU
pipe utilisation, MUFU (XU), issue-slot use, divergence (threads per instruction), shared-memory
bank conflicts, and the L2 reduction (red.global) traffic of S5a's atomics; for the HBM-bound
kernels, DRAM bytes.  One row per captured launch; kernels captured several times are listed
once per launch.
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("us", "gpu__time_duration.sum", 1e-3),
    ("fma_pipe_%", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("fmaheavy_%", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    ("alu_pipe_%", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("xu_inst_%", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    ("shared_pipe_%", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("issue_%", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("thr/inst", "smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    ("warp_inst", "smsp__inst_executed.sum", 1),
    ("thread_inst", "smsp__thread_inst_executed.sum", 1),
    ("occupancy_%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    ("l2_red_requests", "lts__t_requests_srcunit_tex_op_red.sum", 1),
    ("l2_red_sectors", "lts__t_sectors_srcunit_tex_op_red.sum", 1),
    ("l2_red_%", "lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed", 1),
    ("dram_read_B", "dram__bytes_read.sum", 1),
    ("dram_write_B", "dram__bytes_write.sum", 1),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
]


def _num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def read(report):
    raw = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head = rows[0]
    col = {n: i for i, n in enumerate(head)}
    units = rows[1]
    out = []
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("ges::", "")
        d = {"kernel": name}
        for key, metric, scale in METRICS:
            i = col.get(metric)
            v = _num(r[i]) if i is not None else None
            if v is not None and key == "us":
                u = units[i]
                v = v * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
            elif v is not None and key.endswith("_B"):
                u = units[i]
                v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
            d[key] = v
        out.append(d)
    return out


def markdown(rows):
    keys = [k for k, _, _ in METRICS]
    lines = ["| kernel | " + " | ".join(keys) + " |", "|---" * (len(keys) + 1) + "|"]
    for d in rows:
        cells = []
        for k in keys:
            v = d.get(k)
            if v is None:
                cells.append("—")
            elif abs(v) >= 1e5:
                cells.append(f"{v:.4g}")
            else:
                cells.append(f"{v:.3g}")
        lines.append(f"| `{d['kernel']}` | " + " | ".join(cells) + " |")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--json")
    ap.add_argument("--md")
    a = ap.parse_args()
    rows = read(a.report)
    md = markdown(rows)
    print(md)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"report": a.report, "metrics": {k: m for k, m, _ in METRICS}, "launches": rows}, f, indent=1)
    if a.md:
        with open(a.md, "w") as f:
            f.write(f"Counters from `{a.report}` (tools/pipes.py)\n\n" + md + "\n")


if __name__ == "__main__":
    sys.exit(main())
