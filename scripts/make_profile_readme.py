"""Refresh profiles/r1 from one scripts/round_profile.sh TAG run (here, no GPU needed).

usage: python scripts/make_profile_readme.py TAG [history-line ...]
Copies gpurun_out/TAG_bench_{c5,c3,c4}.json and TAG_launches_c5.csv into profiles/r1/, writes
the raw metrics of the k_density_v4 capture as CSV, and regenerates profiles/r1/README.md's
measured sections (bench table, launch list, ncu summary, hot blocks, per-region breakdown).
The library (paper_1804_06231_b200/libpvsph.so) must be the one the capture ran."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
out = os.path.join(ROOT, "profiles", "r1")
go = os.path.join(ROOT, "gpurun_out")


def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True, cwd=ROOT).stdout


for c in ("c5", "c3", "c4"):
    shutil.copy(os.path.join(go, f"{tag}_bench_{c}.json"), os.path.join(out, f"bench_{c}.json"))
shutil.copy(os.path.join(go, f"{tag}_launches_c5.csv"), os.path.join(out, "launches_c5.csv"))
rep = os.path.join(go, f"{tag}_prof_c5.ncu-rep")
with open(os.path.join(out, "ncu_density_c5_raw.csv"), "w") as f:
    f.write(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)

rows = []
for c in ("c5", "c3", "c4"):
    d = json.loads(open(os.path.join(out, f"bench_{c}.json")).read().strip().splitlines()[-1])
    st, e, cb, r, ck = d["stage_ms"], d.get("e2e") or {}, d.get("cpu_baseline") or {}, d["roofline"], d["clocks"]
    cpu = "%.3e (%d cores)" % (cb["value"], cb["cores"]) if cb.get("value") else "-"
    rows.append(f"| {c} | {d['config']['n_particles']:,} | {d['ms_per_step']:.2f} | {st['build']:.2f} / {st['sort']:.2f} / "
                f"{st['density']:.2f} | {d['value']:.3e} | {e.get('value', float('nan')):.3e} "
                f"({e.get('ms_per_step', float('nan')):.1f} ms) | {r['achieved']:.2f} TFLOP/s = {100 * r['frac']:.2f} % | "
                f"{cpu} | {ck.get('sm_mhz')} MHz, {ck.get('samples')} samples, reasons {ck.get('reasons')} |")
launch = run("scripts/ncu_summary.py", "--launches", os.path.join(out, "launches_c5.csv"))
summ = run("scripts/ncu_summary.py", rep)
blocks = run("scripts/ncu_blocks.py", rep, "0.02")
lines = run("scripts/ncu_lines.py", rep, "paper_1804_06231_b200/libpvsph.so", "k_density_v4ILb0", "100000")
tmp = os.path.join(go, f"{tag}_lines.txt")
open(tmp, "w").write(lines)
regions = run("scripts/ncu_regions.py", tmp)

readme = open(os.path.join(out, "README.md")).read()
head = readme[:readme.index("## bench.py lines")]
tail = readme[readme.index("Reading:"):] if "Reading:" in readme else ""
hist = readme[readme.index("History at c5"):readme.index("## launch list")] if "History at c5" in readme else ""
body = f"""## bench.py lines (`scripts/round_profile.sh {tag}`)

| config | particles | ms/step | build / sort / density (ms) | interactions/s | e2e (host buffers, pipelined) | roofline (useful FP32, k_density_v4) | cpu_baseline (fp64 oracle) | clocks (NVML, timed region) |
|---|---|---|---|---|---|---|---|---|
{chr(10).join(rows)}

{hist}## launch list (c5, `ncu --metrics gpu__time_duration.sum`, cold-cache, serialised)

{launch}
(`k_density_v4<1>` is the counting variant bench.py runs once, outside the timed region, for
the candidate/hit statistics.)

## k_density_v4 at c5 (`ncu --set full`, one launch)

{summ}
### hot SASS blocks

```
{blocks}```

### instructions and stall samples by code region (`scripts/ncu_lines.py` + `scripts/ncu_regions.py`)

{regions}
"""
open(os.path.join(out, "README.md"), "w").write(head + body + tail)
print("profiles/r1 refreshed from", tag)
