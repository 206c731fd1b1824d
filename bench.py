#!/usr/bin/env python
"""Benchmark of the pseudo-Verlet SPH density pass on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

One step = one pass of the whole hot path over the config's particle set:
sph_build_cells -> sph_sort_cells -> sph_density_all (+ the x-slab ghost
exchange when N > 1).  Inputs are resident in HBM when the timed region
starts (`value`); the `e2e` figure repeats the step through the public API
with pinned HOST buffers, the H2D copy of the inputs and the D2H copy of all
outputs inside the timed region.  Rank 0 prints one JSON line.

Metric: in-range pair interactions per second (sum_i nngb_i per step / step
time), whole job.  `--impl reference` times the fp64 CPU oracle (the only
reference this tier has) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "in-range pair interactions/sec (whole job)"
UNIT = "interactions/s"
FLOP_CAND, FLOP_HIT = 8, 48                  # algorithmic flops
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.45, SMs x FP32 lanes x FMA x max clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--levels", type=int, default=0,
                    help="level passes (DESIGN.md §4.5); 0 = auto: 3 for the clustered c4, else 1")
    ap.add_argument("--engine", default="gather", choices=["gather", "sym"],
                    help="density pass: the gather engine (sph_density_all, default) or the coloured symmetric "
                         "whole pass (sph_density_all_sym, SURVEY §8(f) #1)")
    ap.add_argument("--reuse", action="store_true",
                    help="list-reuse time loop (P:102 max_dx; ReuseLoop): drift + density per step, cells and "
                         "lists rebuilt only when the skin would be exceeded (1 GPU)")
    ap.add_argument("--skin-frac", type=float, default=0.01, help="--reuse: skin / C_l")
    ap.add_argument("--rebuild-every", type=int, default=4, help="--reuse: dt chosen so the skin lasts this many steps")
    ap.add_argument("--balance", type=int, default=-1,
                    help="N > 1: x-slab cuts by estimated work (1) or equal planes (0); -1 = auto: on for c4")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock and clock-event reasons during the timed region: NVML polled every 2 ms in a
    thread (short regions such as c3's ~10 ms still get samples), else nvidia-smi -lms 100."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clock-event reason bits -> names (nvml.h: SwPowerCap 0x4, HwSlowdown 0x8,
    # SwThermalSlowdown 0x20, HwThermalSlowdown 0x40)
    BITS = ((0x8, "hw_slowdown"), (0x40, "hw_thermal_slowdown"), (0x20, "sw_thermal_slowdown"), (0x4, "sw_power_cap"))

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.nvml = (pynvml, h)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                row = [str(self.gpu), str(sm), str(mx), "", hex(rs)] + \
                    ["Active" if rs & b else "Not Active" for b, _ in self.BITS]
                self.rows.append(row)
            except Exception:
                return
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            self.t.join(timeout=1)
            try:
                self.nvml[0].nvmlShutdown()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 5 + k and r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _profile_ncu(config: str):
    """The committed ncu capture of the density kernel at this config (profiles/r2/ncu_fp32.json,
    written by scripts/ncu_fp32.sh + scripts/parse_fp32.py): the measured FP32 form, DRAM bytes,
    warp efficiency and FMA-pipe activity of one launch.  None when absent."""
    path = os.path.join(ROOT, "profiles", "r2", "ncu_fp32.json")
    try:
        with open(path) as f:
            return json.load(f).get(config)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# CPU baseline: the oracle's cell list on a bounded sample
# ---------------------------------------------------------------------------
def _oracle_rate(p, seconds: float, rng):
    """Time oracle_celllist on two bounded random target samples of p.  Each call bins all
    N particles once (a fixed cost) and then evaluates its targets; the difference of the
    two calls gives the per-target cost, the rest is the binning.  The rate is that of a
    full pass (binning once + all N targets).  Returns (interactions/s, n_targets, text)."""
    import oracle
    if p.n <= 1_000_000:                       # small sets: one full pass
        t0 = time.perf_counter()
        r = oracle.celllist(p.xyzh, p.vm, p.nc)
        dt = time.perf_counter() - t0
        return (float(r["nngb"].sum()) / dt, p.n,
                f"oracle_celllist (fp64, OpenMP), one full pass over {p.name} (N={p.n}): {dt:.2f} s")
    n_a = 50_000
    ta = np.sort(rng.choice(p.n, n_a, replace=False))
    t0 = time.perf_counter()
    oracle.celllist(p.xyzh, p.vm, p.nc, targets=ta)
    d_a = time.perf_counter() - t0
    # second sample: about `seconds` of target work, from a rough per-target estimate, capped
    rough = max(d_a / n_a, 2e-7) if p.n <= 4 * n_a else 2e-6
    n_b = int(min(p.n, max(4 * n_a, seconds / rough)))
    tb = np.sort(rng.choice(p.n, n_b, replace=False))
    t0 = time.perf_counter()
    rb = oracle.celllist(p.xyzh, p.vm, p.nc, targets=tb)
    d_b = time.perf_counter() - t0
    per_target = max(d_b - d_a, 1e-9) / max(n_b - n_a, 1)
    t_bin = max(0.0, d_a - n_a * per_target)
    inter_per_target = float(rb["nngb"].sum()) / n_b
    rate = inter_per_target * p.n / (t_bin + per_target * p.n)
    desc = (f"oracle_celllist (fp64, OpenMP) timed on {n_a} and {n_b} random targets of {p.name} (N={p.n}); "
            f"per-target {per_target * 1e6:.2f} us, binning {t_bin:.2f} s, extrapolated to a full pass over all N")
    return rate, n_b, desc


def cpu_baseline(p, seconds: float):
    import oracle
    rate, n_s, desc = _oracle_rate(p, seconds, np.random.default_rng(123))
    return {"value": rate, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle", "sample": desc}


# ---------------------------------------------------------------------------
# reference arm: the oracle, timed on the host cores
# ---------------------------------------------------------------------------
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import synth
    p = synth.make(args.config)
    per_step = max(5.0, 90.0 / max(1, args.steps + args.warmup))
    rng = np.random.default_rng(7)
    # one-off cost of a call (binning all N) and the per-target cost, from two bounded calls
    # (small sets: every step is a full pass)
    n_a = min(p.n, 50_000)
    t0 = time.perf_counter()
    oracle.celllist(p.xyzh, p.vm, p.nc, targets=np.sort(rng.choice(p.n, n_a, replace=False)))
    d_a = time.perf_counter() - t0
    n_b = min(p.n, 20 * n_a)
    t0 = time.perf_counter()
    oracle.celllist(p.xyzh, p.vm, p.nc, targets=np.sort(rng.choice(p.n, n_b, replace=False)))
    d_b = time.perf_counter() - t0
    slope = max(d_b - d_a, 1e-9) / max(n_b - n_a, 1)
    t_bin = max(0.0, d_a - n_a * slope)
    n_s = int(min(p.n, max(n_a, per_step / slope)))
    if n_b >= p.n:
        n_s, t_bin = p.n, 0.0
    times, rates = [], []
    for s in range(args.warmup + args.steps):
        tgt = np.sort(rng.choice(p.n, n_s, replace=False))
        t0 = time.perf_counter()
        r = oracle.celllist(p.xyzh, p.vm, p.nc, targets=tgt)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            per_target = max(dt - t_bin, 1e-9) / n_s
            times.append(dt)
            # a full pass bins once and evaluates all N targets
            rates.append(float(r["nngb"].sum()) / n_s * p.n / (t_bin + per_target * p.n))
    value = statistics.mean(rates)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"{args.config} (BASELINE.json configs, DESIGN.md §3)",
                                            "n_particles": p.n, "cells": f"{p.nc}^3",
                                            "sample_targets_per_step": n_s},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": f"oracle_celllist on {n_s} random targets of {p.name} per step; rate "
                                       f"extrapolated to a full pass (binning {t_bin:.2f} s once + per-target cost)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import paper_1804_06231_b200 as pv
    import synth
    from paper_1804_06231_b200 import slabs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pv.load()

    t_gen = time.perf_counter()
    p = synth.make(args.config)                         # every rank: the same seeded set
    nlev = args.levels or (3 if args.config == "c4" else 1)
    levels = pv.level_grids(p.xyzh[:, 3], p.nc, max_levels=nlev) if nlev > 1 else None
    if world == 1:
        part = slabs.Slab.single(p)
    else:
        balance = args.balance if args.balance >= 0 else int(args.config == "c4")
        bounds = slabs.balanced_bounds(slabs.plane_costs(p.xyzh, p.nc, p.box), world) if balance else None
        part = slabs.Slab.from_set(p, rank, world, bounds)
        del p
    t_gen = time.perf_counter() - t_gen
    runner = slabs.SlabRunner(part, dist=dist, levels=levels, engine=args.engine)
    runner.upload()
    stream = torch.cuda.current_stream()

    # one counted pass (outside the timed region): interactions, candidates per kind
    st = pv.Stats()
    runner.step(stats=st)
    runner.check()
    counts = st.read()
    nngb_sum = int(runner.out.nngb[:runner.n_own].sum(dtype=torch.int64).item())
    cand_sum, hit_sum = sum(counts["cand"]), sum(counts["hits"])
    assert hit_sum == nngb_sum, (hit_sum, nngb_sum)
    if dist:
        t = torch.tensor([nngb_sum, cand_sum, counts["band"]] + counts["cand"] + counts["hits"], dtype=torch.int64,
                         device="cuda")
        dist.all_reduce(t)
        tot_inter, tot_cand, tot_band = int(t[0]), int(t[1]), int(t[2])
        tot_kind = ([int(v) for v in t[3:7]], [int(v) for v in t[7:11]])
    else:
        tot_inter, tot_cand, tot_band = nngb_sum, cand_sum, counts["band"]
        tot_kind = (counts["cand"], counts["hits"])

    for _ in range(args.warmup):
        runner.step()
    torch.cuda.synchronize()

    nst = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(nst)]
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(nst):
            runner.step(events=ev[k])
        t1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    ms_total = t0.elapsed_time(t1)
    stage = {"exchange": [], "build": [], "sort": [], "density": []}
    for k in range(nst):
        e = ev[k]
        stage["exchange"].append(e[0].elapsed_time(e[1]))
        stage["build"].append(e[1].elapsed_time(e[2]))
        stage["sort"].append(e[2].elapsed_time(e[3]))
        stage["density"].append(e[3].elapsed_time(e[4]))
    ms_step = ms_total / nst
    if dist:
        t = torch.tensor([ms_step, statistics.mean(stage["density"])], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step_max, dens_max = float(t[0]), float(t[1])
    else:
        ms_step_max, dens_max = ms_step, statistics.mean(stage["density"])
    value = tot_inter / (ms_step_max * 1e-3)

    # e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        # a serving loop: H2D of step k+1 and D2H of step k-1 overlap step k; the pipeline's fill
        # (first H2D) and drain (last D2H) stay inside the timed region, amortised over >= 10 steps
        e2e_steps = max(10, nst)
        e2e_ms, h2d, d2h = runner.e2e_time(steps=e2e_steps, warmup=1)
        if dist:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t[0])
        e2e = {"value": tot_inter / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": e2e_steps,
               "pipelined": "3 streams, double-buffered inputs/outputs; fill and drain inside the timed region"}

    dens_ms_local = statistics.mean(stage["density"])
    flops = FLOP_CAND * cand_sum + FLOP_HIT * hit_sum          # this rank's density launch
    achieved = flops / (dens_ms_local * 1e-3) / 1e12
    prof = _profile_ncu(args.config) if args.engine == "gather" else None
    roof = {"bound": "alu", "kernel": "k_density_v5 (sph_density_all incl. its tile list and transpose)"
            if args.engine == "gather" else "k_density_pair_sym colour phases (sph_density_all_sym)",
            "achieved": achieved, "peak": FP32_PEAK_TFLOPS,
            "unit": "TFLOP/s", "frac": achieved / FP32_PEAK_TFLOPS,
            "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (= ncu ffma peak_sustained x 2 x "
                           "f_SM; DESIGN.md §6); MEASURED_PEAKS.json has no FP32 figure",
            "useful_flops": "8 per pseudo-Verlet candidate + 48 per in-range interaction (SURVEY §8(d))",
            "traffic": prof["dram_bytes"] if prof else None,
            "flops_per_launch": flops, "launch_ms": dens_ms_local}
    if prof:       # the measured forms, from the committed ncu capture of the same kernel and config
        roof.update({"measured_frac": prof["measured_frac"], "measured_tflops": prof["fp32_tflops_measured"],
                     "hbm_frac": prof["hbm_frac_of_measured_6548"], "hbm_gbs": prof["hbm_gbs"],
                     "warp_efficiency": prof["warp_efficiency"], "fma_pipe_active_pct": prof["fma_pipe_active_pct"],
                     "issue_active_pct": prof["issue_active_pct"],
                     "measured_source": "profiles/r2/ncu_fp32.json (ncu, one launch of %s at %s: F = 2 ffma + fadd + "
                                        "fmul + 4 ffma2 + 2 fadd2 + 2 fmul2 over ncu's ffma peak)" %
                                        (prof["kernel"], args.config)})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(part.pset, args.cpu_seconds)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": nst,
                "warmup": args.warmup, "ms_per_step": ms_step_max, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"{args.config} (BASELINE.json configs, DESIGN.md §3)",
                           "n_particles": part.n_global, "cells": f"{part.nc}^3",
                           "parallelism": f"x-slab{world}" if world > 1 else "single",
                           "slab_planes": [part.x_lo, part.x_hi] if world > 1 else None,
                           "level_grids": [lv[0] for lv in runner.levels],
                           "l2": "inputs (>= 4 GB at c5) larger than L2; no flush",
                           "step": ("ghost exchange + build_sort_cells (fused; stage 'build' includes the small "
                                    "cells' lists, 'sort' the larger cells' tiers) + " if len(runner.levels) == 1 else
                                    "ghost exchange + build_cells + sort_cells + ") +
                                   ("density_all" if args.engine == "gather" else "density_all_sym (colour phases)")},
                "interactions_per_step": tot_inter, "candidates_per_step": tot_cand,
                "hit_fraction": tot_inter / max(1, tot_cand),
                "per_orientation": {k: {"candidates": tot_kind[0][n], "interactions": tot_kind[1][n],
                                        "hit_fraction": tot_kind[1][n] / max(1, tot_kind[0][n])}
                                    for n, k in enumerate(("self", "face", "edge", "corner"))},
                "band_pairs": tot_band,
                "evaluations_per_s": tot_cand / (ms_step_max * 1e-3),              # SV §8(d)
                "particles_per_s": part.n_global / (ms_step_max * 1e-3),
                "stage_ms": {k: statistics.mean(v) for k, v in stage.items()},
                "stage_ms_stats": {k: {"median": statistics.median(v), "min": min(v), "max": max(v)}
                                   for k, v in stage.items()},
                "density_ms_max_over_ranks": dens_max,
                "gpu_launches": runner.launches_per_step * nst,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
                "gen_seconds": t_gen}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reuse(args):
    """The list-reuse time loop on one GPU: K timed steps of drift + density
    with the rebuilds (gather positions, build, sort) they trigger, inside the timed region."""
    import numpy as np
    import torch
    import paper_1804_06231_b200 as pv
    import synth
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    pv.load()
    p = synth.make(args.config)
    cl = p.box / p.nc
    skin = args.skin_frac * cl
    loop = pv.ReuseLoop(p.nc, p.n, skin, box=p.box)
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    loop.start(x, v)
    dt = 0.999 * skin / args.rebuild_every / max(loop.vmax, 1e-30)
    dt = min(dt, 0.999 * (skin - loop.step_bound(0.0)) / args.rebuild_every / max(loop.vmax, 1e-30))
    st = pv.Stats()
    loop.step(dt, stats=st)                             # counted step (outside the timed region)
    loop.check()
    counts = st.read()
    for _ in range(args.warmup):
        loop.step(dt)
    torch.cuda.synchronize()
    r0 = loop.rebuilds
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        torch.cuda.synchronize()
        e0.record(s)
        for k in range(args.steps):
            loop.step(dt, events=dev[k])
        e1.record(s)
        torch.cuda.synchronize()
    loop.check()
    ms = e0.elapsed_time(e1) / args.steps
    dens_ms = sum(a.elapsed_time(b) for a, b in dev) / args.steps
    inter = int(sum(counts["hits"]))
    nreb = loop.rebuilds - r0
    from paper_1804_06231_b200 import slabs
    # per step: k_drift + the density pass; per rebuild: k_gather_positions + build + sort
    launches = args.steps * (1 + slabs.DENSITY_LAUNCHES) + nreb * (1 + slabs.BUILD_LAUNCHES + slabs.SORT_LAUNCHES)
    flops = FLOP_CAND * int(sum(counts["cand"])) + FLOP_HIT * inter
    achieved = flops / (dens_ms * 1e-3) / 1e12
    roof = {"bound": "alu", "kernel": "k_density_v5 (sph_density_all incl. its tile list and transpose)",
            "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP32_PEAK_TFLOPS,
            "useful_flops": "8 per pseudo-Verlet candidate + 48 per in-range interaction (SURVEY §8(d)); windows "
                            "widened by 2 max_dx(cj) under reuse", "traffic": None, "launch_ms": dens_ms}
    line = {"metric": METRIC, "value": inter / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "mode": "reuse",
            "config": {"workload": f"{args.config} (BASELINE.json configs, DESIGN.md §3)", "n_particles": p.n,
                       "cells": f"{p.nc}^3", "parallelism": "single", "skin_over_cl": args.skin_frac,
                       "dt": dt, "step": "sph_drift + sph_density_all; rebuild (sph_gather_positions + "
                                         "sph_build_cells + sph_sort_cells) when the skin would be exceeded",
                       "l2": "inputs larger than L2; no flush"},
            "rebuilds_in_timed_steps": nreb, "interactions_per_step": inter,
            "candidates_per_step": int(sum(counts["cand"])),
            "stage_ms": {"density": dens_ms, "drift_and_rebuilds": ms - dens_ms},
            "gpu_launches": launches, "roofline": roof, "cpu_baseline": None, "e2e": None, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.reuse:
        run_reuse(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
