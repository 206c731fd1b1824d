#!/usr/bin/env python
"""Summarise ncu reports / launch lists into markdown for profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py report.ncu-rep [...]     # --set full captures
    python scripts/ncu_summary.py --launches launches.csv  # gpu__time_duration launch list
"""
import argparse
import csv
import io
import subprocess
import sys
from collections import OrderedDict, defaultdict

METRICS = OrderedDict([
    ("gpu__time_duration.sum", "duration"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp-instr"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (occupancy) %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thread-instr"),
    ("sm__sass_thread_inst_executed_op_ffma2_pred_on.sum", "FFMA2 thread-instr"),
    ("sm__sass_thread_inst_executed_op_fadd_pred_on.sum", "FADD thread-instr"),
    ("sm__sass_thread_inst_executed_op_fadd2_pred_on.sum", "FADD2 thread-instr"),
    ("sm__sass_thread_inst_executed_op_fmul_pred_on.sum", "FMUL thread-instr"),
    ("sm__sass_thread_inst_executed_op_fmul2_pred_on.sum", "FMUL2 thread-instr"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("launch__registers_per_thread", "registers"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short scoreboard"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math throttle"),
    ("smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio", "stall branch"),
])


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def fp32_flops(get):
    """Measured FP32 flops from predicated-on thread instruction counts."""
    try:
        return (2 * get("sm__sass_thread_inst_executed_op_ffma_pred_on.sum") +
                get("sm__sass_thread_inst_executed_op_fadd_pred_on.sum") +
                get("sm__sass_thread_inst_executed_op_fmul_pred_on.sum") +
                4 * get("sm__sass_thread_inst_executed_op_ffma2_pred_on.sum") +
                2 * get("sm__sass_thread_inst_executed_op_fadd2_pred_on.sum") +
                2 * get("sm__sass_thread_inst_executed_op_fmul2_pred_on.sum"))
    except (KeyError, ValueError):
        return None


def summarise(rep):
    hdr, units, data = raw(rep)
    ki = hdr.index("Kernel Name")
    lines = [f"### {rep}", "", "| kernel | " + " | ".join(METRICS.values()) + " | measured FP32 TFLOP/s |",
             "|---|" + "---|" * (len(METRICS) + 1)]
    for r in data:
        def get(m):
            return float(r[hdr.index(m)].replace(",", ""))
        cells = []
        for m in METRICS:
            if m in hdr:
                v = r[hdr.index(m)]
                u = units[hdr.index(m)]
                cells.append(f"{v} {u}".strip())
            else:
                cells.append("-")
        fl = fp32_flops(get)
        t = None
        try:
            t = get("gpu__time_duration.sum")
            tu = units[hdr.index("gpu__time_duration.sum")]
            t = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(tu, 1e-9)
        except (KeyError, ValueError):
            pass
        tf = f"{fl / t / 1e12:.2f}" if fl and t else "-"
        lines.append(f"| {r[ki][:60]} | " + " | ".join(cells) + f" | {tf} |")
    return "\n".join(lines)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    t = defaultdict(list)
    unit = None
    for r in rows[hdr + 1:]:
        if len(r) > vi and (mi is None or r[mi] == "gpu__time_duration.sum"):
            t[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
            unit = r[ui]
    total = sum(sum(v) for v in t.values())
    out = [f"### launch list {path} (gpu__time_duration, cold-cache, serialised)", "",
           f"| kernel | launches | mean ({unit}) | total share |", "|---|---|---|---|"]
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / total:.1f} % |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--launches", nargs="*", default=[])
    a = ap.parse_args()
    for r in a.reports:
        print(summarise(r))
        print()
    for l in a.launches:
        print(launches(l))
        print()


if __name__ == "__main__":
    sys.exit(main())
