"""Profiling helper: aggregate scripts/ncu_lines.py output of k_density_v4 into code regions.
usage: python scripts/ncu_lines.py REP LIB k_density_v4ILb0 100000 > lines.txt
       python scripts/ncu_regions.py lines.txt"""
import collections
import re
import sys

SRC = "paper_1804_06231_b200/csrc/density_v4.cuh"
src = open(SRC).read().splitlines()


def line_of(pat):
    for k, l in enumerate(src, 1):
        if pat in l:
            return k
    raise SystemExit(f"pattern not found: {pat}")


marks = [("global-memory tiles", "void v4_particle_global("), ("M4 interaction (math)", "void interact_pair("),
         ("window searches", "float v4_dot("), ("particle setup", "void v4_particle_staged("),
         ("hit drains", "auto drain = "), ("drain checks", "auto drain_check"), ("self-cell sweep", "auto step4 = "),
         ("window sweeps", "auto step4pair"), ("self loop", "// the self cell"), ("direction loop", "int pos = lpos"),
         ("final drain + finalise", "PH_T0(tf0)"), ("staging / tile loop", "struct TileGeom {")]
bounds = sorted((line_of(p), n) for n, p in marks)
agg = collections.defaultdict(lambda: [0.0, 0.0])
for ln in open(sys.argv[1]).read().splitlines()[1:]:
    m = re.match(r"(\S+):(\d+)\s+instr\s+([\d.]+)%\s+samples\s+([\d.]+)%", ln)
    if not m:
        continue
    f, l, i, s = m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4))
    if f == "density_v4.cuh":
        key = "tile list / records" if l < bounds[0][0] else [n for b, n in bounds if b <= l][-1]
    elif f in ("sm_100_rt.hpp", "packed.cuh"):
        key = "FFMA2/FMUL2/FADD2 + smem helpers (packed.cuh)"
    elif f == "density.cuh":
        key = "global-memory tiles"
    else:
        key = f
    agg[key][0] += i
    agg[key][1] += s
print("| region | instructions | stall samples |\n|---|---|---|")
for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if i >= 0.1 or s >= 0.1:
        print(f"| {k} | {i:.1f} % | {s:.1f} % |")
