"""Build profiles/r2/ from one scripts/round2_measure.sh TAG run (here, no GPU needed).

usage: python scripts/make_profile_r2.py TAG
Copies the bench lines, launch lists, test27cells and calibration results into profiles/r2/,
regenerates profiles/r2/ncu_fp32.json (bench.py's measured-FP32 source) from the ncu counter
logs, writes the raw metrics of the --set full capture as CSV and writes profiles/r2/README.md:
every table cell is a measured number or an explicit 'n/a (why)'."""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import parse_fp32  # noqa: E402

tag = sys.argv[1]
out = os.path.join(ROOT, "profiles", "r2")
go = os.path.join(ROOT, "gpurun_out")
os.makedirs(out, exist_ok=True)
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
HBM = PEAK["hbm_gbs"]


def last_json(path):
    for line in reversed(open(path).read().strip().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    raise ValueError(f"no JSON line in {path}")


def g(path):
    return os.path.join(go, f"{tag}_{path}")


benches = OrderedDict()
for name in ("bench_c5", "bench_c3", "bench_c4", "bench_reuse_c5", "bench_sym_c3", "bench_ref_c5"):
    src = g(name + ".json")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(out, name + ".json"))
        benches[name] = last_json(src)
for name, dst in (("test27cells.json", "test27cells.json"), ("calib.json", "calib.json"),
                  ("cpu_baselines.json", "cpu_baselines.json"),
                  ("launches_c5.csv", "launches_c5.csv"), ("launches_c4.csv", "launches_c4.csv")):
    if os.path.exists(g(name)):
        shutil.copy(g(name), os.path.join(out, dst))

# measured FP32 counters -> ncu_fp32.json (bench.py reads it)
fp32 = OrderedDict()
for c in ("c3", "c4", "c5"):
    p = os.path.join(go, f"{tag}_fp32_{c}.csv")
    if os.path.exists(p):
        fp32[c] = parse_fp32.parse(p)
        fp32[c]["source"] = os.path.basename(p)
        shutil.copy(p, os.path.join(out, f"{tag}_fp32_{c}.csv"))
if fp32:
    json.dump(fp32, open(os.path.join(out, "ncu_fp32.json"), "w"), indent=1)
symfp = None
for tg in (tag, "r2s"):
    sp = os.path.join(go, f"{tg}_sym_fp32_c3.csv")
    if os.path.exists(sp):
        symfp = parse_fp32.parse_multi(sp)
        symfp["source"] = os.path.basename(sp)
        shutil.copy(sp, os.path.join(out, os.path.basename(sp)))
        json.dump(symfp, open(os.path.join(out, "ncu_sym_c3.json"), "w"), indent=1)
        break

rep = g("prof_c5.ncu-rep")
summ = ""
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    open(os.path.join(out, "ncu_density_c5_raw.csv"), "w").write(raw)
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                          capture_output=True, text=True).stdout
    # the per-op FP32 counters are not part of --set full: they are in the counter table above
    summ = summ.replace("| - |", "| n/a (counter table above) |").replace("| - |", "| n/a (counter table above) |")
    summ = summ.replace(f"### {rep}", "### " + os.path.basename(rep))


def launches(path):
    """Per-kernel totals of one step (the last quarter of the launch list is not reliable, so
    the whole list is divided by the number of bench steps it covers: 1 timed + 3 warm-up +
    the stats pass)."""
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[h]
    ki, vi, mi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("ID")
    per = OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        per.setdefault(r[ii], {"k": r[ki].split("(")[0]})[r[mi]] = float(r[vi].replace(",", ""))
    tot = OrderedDict()
    for x in per.values():
        k = x["k"].replace("void ", "").replace("pvsph::", "")
        t = tot.setdefault(k, [0, 0.0, 0.0])
        t[0] += 1
        t[1] += x.get("gpu__time_duration.sum", 0.0)
        t[2] += x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)
    return tot


def launch_table(path, title):
    tot = launches(path)
    allt = sum(v[1] for v in tot.values())
    lines = [f"### {title}", "",
             "| kernel | launches | mean time (ms) | share of listed time | DRAM bytes / launch (GB) | DRAM GB/s | "
             "fraction of measured HBM (%.0f GB/s) |" % HBM, "|---|---|---|---|---|---|---|"]
    for k, (n, t, b) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        if t / allt < 0.001:
            continue
        ms = t / n / 1e6
        gbs = b / t if t else 0.0          # bytes / ns = GB/s
        lines.append(f"| {k[:60]} | {n} | {ms:.3f} | {100 * t / allt:.1f} % | {b / n / 1e9:.3f} | {gbs:.0f} | "
                     f"{gbs / HBM:.3f} |")
    return "\n".join(lines) + "\n"


def f3(x, fmt="%.3g"):
    return fmt % x if isinstance(x, (int, float)) else str(x)


rows = []
for name, d in benches.items():
    if name == "bench_ref_c5":
        continue
    st, e, cb, r, ck = d.get("stage_ms") or {}, d.get("e2e") or {}, d.get("cpu_baseline") or {}, \
        d.get("roofline") or {}, d["clocks"]
    cpu = ("%.3e %s (%d cores, %s)" % (cb["value"], cb["unit"], cb["cores"], cb.get("sample", "")[:60])
           if cb.get("value") else "n/a (not run on this line; see c3/c4/c5)")
    e2e = ("%.3e (%.1f ms/step)" % (e["value"], e.get("ms_per_step", float("nan"))) if e.get("value")
           else "n/a (not measured on this line; see c3/c4/c5)")
    cfg = name.replace("bench_", "")
    fp = fp32.get(cfg) if cfg in ("c3", "c4", "c5") else (symfp if cfg == "sym_c3" else None)
    why = ("n/a (39 colour-phase launches per pass: no single-launch counter form)" if "sym" in name else
           "n/a (see the c5 line: same kernel)" if "reuse" in name else "n/a (no ncu counters)")
    if r.get("measured_frac"):
        meas = "%.3f (%.2f TFLOP/s)" % (r["measured_frac"], r["measured_tflops"])
    elif fp:
        meas = "%.3f (%.2f TFLOP/s; %s)" % (fp["measured_frac"], fp["fp32_tflops_measured"],
                                            "ncu_sym_c3.json, 78 launches summed" if cfg == "sym_c3" else "ncu_fp32.json")
    else:
        meas = why
    hbmf = ("%.3f" % r["hbm_frac"] if r.get("hbm_frac") is not None else
            "%.3f" % (fp["hbm_gbs"] / HBM) if fp else why)
    weff = ("%.3f" % r["warp_efficiency"] if r.get("warp_efficiency") is not None else
            "%.3f" % fp["warp_efficiency"] if fp and "warp_efficiency" in fp else
            "n/a (not in the summed counter set)" if fp else why)
    if "build" in st and "fused" in str((d.get("config") or {}).get("step", "")):
        stages = f"{st['build']:.2f} (build + sort, one fused call) / {st['density']:.2f}"
    elif "build" in st:
        stages = f"{st['build']:.2f} / {st['sort']:.2f} / {st['density']:.2f}"
    elif "density" in st:
        stages = f"density {st['density']:.2f}, drift + rebuilds {st['drift_and_rebuilds']:.2f}"
    else:
        stages = "n/a (this capture timed the whole reuse step only)"
    useful = (f"{r['achieved']:.2f} TFLOP/s = {r['frac']:.4f}" if r.get("achieved")
              else "n/a (this capture timed the whole reuse step only)")
    rows.append(f"| {name.replace('bench_', '')} | {d['config']['n_particles']:,} | {d['ms_per_step']:.2f} | "
                f"{stages} | {d['value']:.3e} | "
                f"{e2e} | {useful} | {meas} | {hbmf} | {weff} | "
                f"{d.get('gpu_launches', 'n/a (not counted in this capture)')} | {cpu} | {ck.get('sm_mhz')} MHz, "
                f"{ck.get('samples')} samples, reasons {ck.get('reasons')} |")

fp_rows = []
for c, v in fp32.items():
    b = benches.get(f"bench_{c}")
    useful = b["roofline"]["achieved"] if b else float("nan")
    fp_rows.append(f"| {c} | {v['kernel'].replace('void ', '').replace('pvsph::', '')} | {v['duration_ms']:.3f} | "
                   f"{v['fp32_flops_executed']:.3e} | {v['fp32_tflops_measured']:.2f} | {v['fp32_peak_tflops_ncu']:.2f} | "
                   f"{v['measured_frac']:.4f} | {useful:.2f} | {v['dram_bytes'] / 1e9:.3f} | {v['hbm_gbs']:.0f} | "
                   f"{v['hbm_gbs'] / HBM:.4f} | {v['warp_efficiency']:.3f} | {v['fma_pipe_active_pct']:.1f} | "
                   f"{v['issue_active_pct']:.1f} | {v['warps_active_pct']:.1f} | {v['warp_instructions']:.3e} | "
                   f"{v['registers']:.0f} |")

ref = benches.get("bench_ref_c5")
ref_txt = ("`bench.py --impl reference` (the fp64 oracle on the host, bounded sample): %s %s, %s" %
           (f3(ref["value"], "%.4g"), ref["unit"], json.dumps(ref.get("cpu_baseline"))) if ref else
           "reference arm: not run in this capture")
t27 = ""
if os.path.exists(os.path.join(out, "test27cells.json")):
    d = last_json(os.path.join(out, "test27cells.json"))
    o = d["orientations"]
    t27 = ["| orientation | GPU us per symmetric pair (two gathers) | sym kernel us per pair | interactions per pair | "
           "candidates per pair (sym) | paper AVX us per pair (context) |", "|---|---|---|---|---|---|"]
    for k in ("face", "edge", "corner"):
        x = o[k]
        t27.append(f"| {k} | {x['us_per_symmetric_pair']:.4f} | {x['sym_kernel_us_per_symmetric_pair']:.4f} | "
                   f"{x['interactions_per_symmetric_pair']:.1f} | {x['sym_kernel_candidates_per_pair']:.1f} | "
                   f"{x['paper_avx_us_per_pair']} |")
    t27 = "\n".join(t27) + "\n\n(self cells: %.4f us per cell, %.0f interactions per cell.)\n" % (
        o["self"]["us_per_cell"], o["self"]["interactions_per_cell"])
cal = ""
if os.path.exists(os.path.join(out, "calib.json")):
    cal = "```\n" + json.dumps(last_json(os.path.join(out, "calib.json")), indent=1) + "\n```\n"

cpub = ""
if os.path.exists(os.path.join(out, "cpu_baselines.json")):
    cb = last_json(os.path.join(out, "cpu_baselines.json"))
    cpub = [f"Host: {cb['cpu_model']}, {cb['host_threads']} hardware threads; {cb['protocol']}.", "",
            "| config | variant | threads | sample | seconds median (min, max) | reps | interactions | interactions/s |",
            "|---|---|---|---|---|---|---|---|"]
    for r in cb["runs"]:
        sc = r["seconds"]
        cpub.append(f"| {r['config']} | {r['variant']} | {r['threads']} | {r['sample']} | {sc['median']:.4g} "
                    f"({sc['min']:.4g}, {sc['max']:.4g}) | {r['reps']} | {r['interactions']:,} | "
                    f"{r['interactions_per_s']:.3e} |")
    cpub = "\n".join(cpub) + "\n"

body = f"""# Round 2 profiles (B200, sm_100a, 1 GPU)

Production engine: density v5 (`csrc/density_v5.cuh`, DESIGN.md §4.4), radix-sorted cluster
cells (`k_sort_radix`), warp-per-pair symmetric whole pass (`sph_density_all_sym`, §4.7).
All numbers come from one `gpurun` call (`scripts/round2_measure.sh {tag}`), summarised here by
`scripts/make_profile_r2.py {tag}`.  Files: `bench_*.json` (bench.py lines), `ncu_fp32.json`
(the measured-FP32 counters bench.py quotes as `roofline.measured_frac`), `{tag}_fp32_c*.csv`
(raw ncu logs), `launches_c5.csv` / `launches_c4.csv` (ncu launch lists with DRAM bytes),
`ncu_density_c5_raw.csv` (every metric of one `--set full` capture of `k_density_v5<0>` at c5),
`test27cells.json`, `calib.json`.

Reproduce (one B200): `gpurun -- 'bash scripts/round2_measure.sh TAG'`, then here
`python scripts/make_profile_r2.py TAG`.  The measurement script runs the GPU tests and smoke
(unless `notests`), every bench line, test27cells, the calibration, the CPU baselines, the
ncu counter captures (`scripts/ncu_fp32.sh`), the launch lists and one `--set full` capture;
each ncu command only after the same command exited 0 without ncu.

## bench.py lines

Roofline columns: `useful` = algorithmic flops (8 per candidate + 48 per interaction, SURVEY
§8(d)) / the kernel's event-timed launch / 74.45 TFLOP/s; `measured` = executed FP32 flops
(2 FFMA + FADD + FMUL + 4 FFMA2 + 2 FADD2 + 2 FMUL2) / ncu duration / ncu's FFMA peak; HBM =
ncu DRAM bytes / duration / {HBM:.0f} GB/s (MEASURED_PEAKS.json); warp efficiency = active
threads per issued warp instruction / 32.

| line | particles | ms/step | build / sort / density (ms) | interactions/s | e2e interactions/s (host buffers) | useful FP32 (frac) | measured FP32 frac | HBM frac | warp eff | launches/step | cpu_baseline | clocks (timed region) |
|---|---|---|---|---|---|---|---|---|---|---|---|---|
{chr(10).join(rows)}

{ref_txt}

## density kernel, measured roofline (ncu counters, one launch per config)

| config | kernel | ms | FP32 flops executed | measured TFLOP/s | ncu FP32 peak | measured frac | useful TFLOP/s (bench) | DRAM GB | DRAM GB/s | HBM frac | warp eff | FMA pipe % | issue active % | warps active % | warp instr | regs |
|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|
{chr(10).join(fp_rows)}

## launch lists (ncu, cold-cache, serialised: shares, not absolute step times)

{launch_table(os.path.join(out, 'launches_c5.csv'), 'c5 (1 timed + 3 warm-up steps + the stats pass)') if os.path.exists(os.path.join(out, 'launches_c5.csv')) else ''}
{launch_table(os.path.join(out, 'launches_c4.csv'), 'c4, three level grids') if os.path.exists(os.path.join(out, 'launches_c4.csv')) else ''}
Algorithmic bytes (DESIGN.md §4.1): build 72 B/particle (k_bin + k_scatter_rec + k_stable_*),
sort 42 B/particle, density output 36 B/particle.  The build and sort kernels run near the
DRAM bandwidth on the bytes they move (k_stable_small, k_unpermute ~5.5 TB/s) but move 3-4x
the algorithmic bytes (random 64-byte records, DESIGN.md §4.1); the sort's rank loop is
issue-bound.

## k_density_v5 at c5 (`ncu --set full`, one launch)

{summ}
## test27cells (SURVEY §8(f) #4, `bench_test27cells.py`)

{t27}
## CPU baselines (`scripts/cpu_baselines.py`: SURVEY §8(d) one-thread O2 for c1-c3, O1 brute force for c1/c2)

{cpub}
## calibration (`scripts/calibrate.py`: FFMA / FFMA2 peaks and the production interaction rate)

{cal}"""
open(os.path.join(out, "README.md"), "w").write(body)
print("profiles/r2 written from", tag)
