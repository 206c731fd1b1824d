"""Summarise an `ncu --page source --print-source sass --csv` export: instructions executed
per SASS line, grouped into contiguous hot regions (profiling helper, not product code)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: k for k, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    data.append((r[ix["Address"]], r[ix["Source"]], n, r[ix["Warp Stall Sampling (All Samples)"]]))
tot = sum(d[2] for d in data)
print("total warp instructions", tot)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
for a, s, n, st in sorted(data, key=lambda d: -d[2])[:top]:
    print(f"{a:>6} {100.0 * n / tot:6.2f}% {n:>12} stall={st:>6}  {s[:90]}")
