#!/usr/bin/env python
"""test27cells on the GPU: the paper's benchmark of
one 216-particle cell and its 26 equally populated neighbours, batched.

A periodic nc^3 grid in which every cell holds exactly 216 uniform random particles
(synth.test27cells_set: h = 1.2348 x the mean spacing, so gamma h = 0.376 C_l) makes every
cell the centre of one instance.  The cell-pair kernel of the C ABI (`sph_density_pair`,
one CTA per ordered pair, one-sided gather) runs over all pairs of one orientation class
(faces, edges, corners) of all cells, the self kernel over all cells; each is timed with
CUDA events (median of --reps after --warmup).  The whole-pass engine (`sph_density_all`)
runs on the same set for comparison.

Reported per orientation (the paper's Table 3 layout): GPU time per SYMMETRIC cell pair
(= two one-sided gathers, the work of the paper's pair function: both cells updated; and
the symmetric kernel `sph_density_pair_sym`, one evaluation per distance),
in-range interactions and pseudo-Verlet candidates per pair, interactions/s; and the
weighted total of one instance, 8 corner + 12 edge + 6 face pairs.  The paper's
single-core AVX times are printed as context only (other hardware; Table 3).  The
raw-interaction test of Table 2 (one particle with 2560 others, full masks, no
neighbour search) is `sph_calibrate` mode 2 (include/sph_calib.h): the same M4 interaction
with FFMA2 on every (i, j), no distance test; its rate gives the time of one particle's 2560
interactions on the whole GPU and the fraction of that rate the full pipeline reaches.

usage: python bench_test27cells.py [--nc 24] [--reps 5] [--warmup 3]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_AVX_MS = {"corner": 0.00070, "edge": 0.0035, "face": 0.034, "total": 0.25}   # Table 3 (COSMA-5, AVX)
CLASSES = {"face": 1, "edge": 2, "corner": 3}                                       # nonzero offset components
KIND_INDEX = {"self": 0, "face": 1, "edge": 2, "corner": 3}                         # sph_stats index


def pairs_of(nc: int, nonzero: int, torch):
    """(ci, cj) int32 pairs for every cell ci and every offset with `nonzero` nonzero
    components (periodic neighbours, x-major cell ids)."""
    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)
            if (a != 0) + (b != 0) + (c != 0) == nonzero]
    cell = torch.arange(nc ** 3, dtype=torch.int64)
    ix, iy, iz = cell // (nc * nc), (cell // nc) % nc, cell % nc
    out = []
    for a, b, c in offs:
        cj = (((ix + a) % nc) * nc + (iy + b) % nc) * nc + (iz + c) % nc
        out.append(torch.stack([cell, cj], dim=1))
    return torch.cat(out).to(torch.int32).contiguous(), len(offs)


def half_pairs_of(nc: int, nonzero: int, torch):
    """(ci, cj) for every cell and the lexicographically positive offsets of one class: each
    unordered neighbour pair once (the symmetric kernel's input)."""
    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)
            if (a != 0) + (b != 0) + (c != 0) == nonzero and (a, b, c) > (0, 0, 0)]
    cell = torch.arange(nc ** 3, dtype=torch.int64)
    ix, iy, iz = cell // (nc * nc), (cell // nc) % nc, cell % nc
    out = [torch.stack([cell, (((ix + a) % nc) * nc + (iy + b) % nc) * nc + (iz + c) % nc], dim=1) for a, b, c in offs]
    return torch.cat(out).to(torch.int32).contiguous()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nc", type=int, default=24)
    ap.add_argument("--per-cell", type=int, default=216)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import torch
    import paper_1804_06231_b200 as pv
    import synth
    pv.load()
    p = synth.test27cells_set(seed=27, nc=args.nc, per_cell=args.per_cell)
    ncell = args.nc ** 3
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    dp = pv.DensityPass(p.nc, p.n)
    pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws)
    pv.sph_sort_cells(dp.grid, dp.cells, dp.ws)
    dp.check()
    acc = pv.Out.alloc(p.n, zero=True)
    cells_all = torch.arange(ncell, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    res = {}
    # self cells
    st = pv.Stats()
    pv.sph_density_self(dp.grid, dp.cells, cells_all, acc, dp.ws, stats=st)
    torch.cuda.synchronize()
    cnt = st.read()
    ms = timed(lambda: pv.sph_density_self(dp.grid, dp.cells, cells_all, acc, dp.ws))
    res["self"] = {"ms_all_cells": ms, "us_per_cell": 1e3 * ms / ncell,
                   "interactions_per_cell": cnt["hits"][0] / ncell, "candidates_per_cell": cnt["cand"][0] / ncell,
                   "interactions_per_s": cnt["hits"][0] / (ms * 1e-3)}
    for name, nz in CLASSES.items():
        pr, k = pairs_of(args.nc, nz, torch)
        pr = pr.cuda()
        st = pv.Stats()
        pv.sph_density_pair(dp.grid, dp.cells, pr, acc, dp.ws, stats=st)
        torch.cuda.synchronize()
        cnt = st.read()
        ki = KIND_INDEX[name]
        ms = timed(lambda: pv.sph_density_pair(dp.grid, dp.cells, pr, acc, dp.ws))
        nsym = ncell * k / 2                              # symmetric pairs = one-sided pairs / 2
        # the symmetric kernel: each unordered pair once, both cells updated
        hp = half_pairs_of(args.nc, nz, torch).cuda()
        st2 = pv.Stats()
        pv.sph_density_pair_sym(dp.grid, dp.cells, hp, acc, dp.ws, stats=st2)
        torch.cuda.synchronize()
        cnt2 = st2.read()
        ms_sym = timed(lambda: pv.sph_density_pair_sym(dp.grid, dp.cells, hp, acc, dp.ws))
        res[name] = {"one_sided_pairs": int(pr.shape[0]), "ms_all_pairs": ms,
                     "sym_kernel_us_per_symmetric_pair": 1e3 * ms_sym / hp.shape[0],
                     "sym_kernel_candidates_per_pair": cnt2["cand"][ki] / hp.shape[0],
                     "sym_kernel_interactions_per_pair": cnt2["hits"][ki] / hp.shape[0],
                     "us_per_symmetric_pair": 1e3 * ms / nsym,
                     "interactions_per_symmetric_pair": cnt["hits"][ki] / nsym,
                     "candidates_per_symmetric_pair": cnt["cand"][ki] / nsym,
                     "interactions_per_s": cnt["hits"][ki] / (ms * 1e-3),
                     "paper_avx_us_per_pair": 1e3 * PAPER_AVX_MS[name]}
    total_us = 8 * res["corner"]["us_per_symmetric_pair"] + 12 * res["edge"]["us_per_symmetric_pair"] + \
        6 * res["face"]["us_per_symmetric_pair"]
    total_sym_us = 8 * res["corner"]["sym_kernel_us_per_symmetric_pair"] + \
        12 * res["edge"]["sym_kernel_us_per_symmetric_pair"] + 6 * res["face"]["sym_kernel_us_per_symmetric_pair"]
    # the whole-pass engine on the same set: self + 26 one-sided gathers of every cell
    out = pv.Out.alloc(p.n)
    ms_all = timed(lambda: pv.sph_density_all(dp.grid, dp.cells, out, dp.ws))
    inter_all = sum(res[k]["interactions_per_cell"] if k == "self" else 0 for k in res) * ncell
    inter_all += sum(res[k]["interactions_per_symmetric_pair"] * ncell * {"face": 3, "edge": 6, "corner": 4}[k]
                     for k in ("face", "edge", "corner"))
    # Table 2 analogue: full-mask interactions (sph_calibrate mode 3: the production packed body
    # interact2 of density_v5.cuh, 256 per thread per iteration; mode 2 = the scalar reference body)
    import ctypes
    from paper_1804_06231_b200 import _lib
    L = _lib.load()
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, threads, iters = sm * 8, 256, 40
    buf = torch.zeros(1, device="cuda")
    call = lambda: L.sph_calibrate(3, blocks, threads, iters, ctypes.c_void_p(buf.data_ptr()),   # noqa: E731
                                   ctypes.c_void_p(s.cuda_stream))
    ms_raw = timed(call)
    raw_rate = 256 * iters * blocks * threads / (ms_raw * 1e-3)
    call2 = lambda: L.sph_calibrate(2, blocks, threads, iters, ctypes.c_void_p(buf.data_ptr()),   # noqa: E731
                                    ctypes.c_void_p(s.cuda_stream))
    raw_rate_scalar = 256 * iters * blocks * threads / (timed(call2) * 1e-3)
    line = {"benchmark": "test27cells (batched, P:195)", "n_particles": p.n, "cells": ncell,
            "per_cell": args.per_cell, "gamma_h_over_cl": float(synth.GAMMA * p.xyzh[0, 3] * args.nc),
            "dtype": "f32", "data": "synthetic", "reps": args.reps, "warmup": args.warmup,
            "orientations": res,
            "weighted_total_us_per_instance": total_us,
            "weighted_total_us_per_instance_sym_kernel": total_sym_us,
            "weighted_total_definition": "8 corner + 12 edge + 6 face symmetric pairs (P:250)",
            "paper_avx_weighted_total_us": 1e3 * PAPER_AVX_MS["total"],
            "density_all_ms": ms_all, "density_all_us_per_cell": 1e3 * ms_all / ncell,
            "density_all_interactions_per_s": inter_all / (ms_all * 1e-3),
            "raw_fullmask_interactions_per_s": raw_rate,
            "raw_fullmask_body": "interact2 (density_v5.cuh, FFMA2 pairs: the production body)",
            "raw_fullmask_interactions_per_s_scalar_body": raw_rate_scalar,
            "raw_us_per_2560_interactions": 2560 / raw_rate * 1e6,
            "paper_avx_raw_ms_per_2560": 0.0084,
            "pipeline_fraction_of_raw": inter_all / (ms_all * 1e-3) / raw_rate}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
