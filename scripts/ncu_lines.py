"""Profiling helper: per-source-line instruction counts and stall samples of one kernel.

usage: python scripts/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_SUBSTR [top]
Maps the report's SASS view (ncu --page source --print-source sass) to source lines with
nvdisasm -g on the library's cubin (build with -lineinfo).  The library must be the one
the report was captured with."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout

addr_line = {}
cur = None
infn = False
for ln in sass.splitlines():
    if ln.startswith("//---") and ".text." in ln:
        infn = kname in ln
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        addr_line[int(m.group(1), 16)] = cur

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, h = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        blocks.append([r[1], None, []])
    elif r and r[0] == "Address":
        blocks[-1][1] = r
    elif blocks and blocks[-1][1] is not None and r:
        blocks[-1][2].append(r)
blk = [b for b in blocks if kname in b[0].replace("(bool)0", "ILb0").replace("(bool)1", "ILb1") or kname in b[0]]
name, h, data = (blk or blocks)[int(os.environ.get("NCU_BLOCK", "0"))]
ci, cs = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
byline = collections.defaultdict(lambda: [0, 0])
tot_i = tot_s = 0
base = int(data[0][0], 16)               # the report's addresses are absolute
for r in data:
    a = int(r[0], 16) - base
    ni = int(r[ci].replace(",", "") or 0)
    ns = int(r[cs].replace(",", "") or 0)
    tot_i += ni
    tot_s += ns
    key = addr_line.get(a, ("?", 0))
    byline[key][0] += ni
    byline[key][1] += ns
print(f"{name[:80]}  instructions {tot_i}  stall samples {tot_s}")
for (f, l), (ni, ns) in sorted(byline.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{l:<5d} instr {100.0 * ni / tot_i:5.1f}%  samples {100.0 * ns / max(tot_s, 1):5.1f}%")
