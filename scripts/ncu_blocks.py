"""Profiling helper: key metrics, stall breakdown and hot SASS blocks of an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


r = csv.reader(io.StringIO(ncu("--page", "details", "--csv")))
h = next(r)
want = {"Duration", "Issue Slots Busy", "Issued Instructions", "Achieved Active Warps Per SM",
        "Avg. Active Threads Per Warp", "No Eligible", "L1/TEX Hit Rate", "DRAM Throughput", "Registers Per Thread"}
for row in r:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(d["Kernel Name"][:30], d["Metric Name"].ljust(32), d["Metric Value"], d["Metric Unit"])
rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
stalls = [(k, float(x)) for k, x in zip(rows[0], rows[2]) if "pcsamp_warps_issue_stalled" in k and
          not k.endswith("not_issued") and x.replace(".", "").isdigit()]
tot = sum(x for _, x in stalls) or 1
print("stalls:", ", ".join(f"{k.split('stalled_')[1]} {100 * x / tot:.0f}%" for k, x in sorted(stalls, key=lambda t: -t[1])[:8]))
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
out = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    out.append((int(r[ix["Address"]], 16), int(r[ix["Instructions Executed"]] or 0), r[ix["Source"]],
                int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
base = out[0][0]
blocks, prev = [], None
for a, n, s, st in out:
    if n != prev:
        blocks.append([a - base, 0, n, s, 0])
        prev = n
    blocks[-1][1] += 1
    blocks[-1][4] += st
ti = sum(o[1] for o in out) or 1
ts = sum(o[3] for o in out) or 1
print("total instr", ti)
for off, c, n, s, st in blocks:
    if n * c > ti * thr or st > ts * thr * 1.5:
        print(f"{off:#7x} x{c:3d} n={n:>10} instr={100 * n * c / ti:5.2f}% stall={100 * st / ts:5.2f}%  {s.strip()[:60]}")
