#!/usr/bin/env python
"""List reuse across steps ("max_dx"), measured.

One configuration (default c5), two ways of computing the density of K successive drifted
states x_k = x_0 + k v dt:
  * full: every step re-bins and re-sorts (sph_build_cells + sph_sort_cells + sph_density_all
    on a grid without skin);
  * reuse: cells and lists built once on a grid with skin s, then every step is
    sph_drift + sph_density_all with each neighbour cell's window widened by 2 max_dx(c)
    (its particles' largest displacement since the build, R17).
dt is chosen so that the K drifts stay inside the skin (K |v|max dt <= s).  Both are timed
with CUDA events over the K steps (after warm-up on separate buffers); the line reports the
ms per step of each, the candidate increase caused by the wider windows, and the largest
relative difference of rho between the two (the same states up to the fp32 wrap of positions
that left the box, summed in different orders).

usage: python bench_reuse.py [--config c5] [--steps 5] [--skin-frac 0.01]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--skin-frac", type=float, default=0.01, help="skin / C_l")
    args = ap.parse_args()

    import numpy as np
    import torch
    import paper_1804_06231_b200 as pv
    import synth
    pv.load()
    p = synth.make(args.config)
    cl = 1.0 / p.nc
    skin = args.skin_frac * cl
    K = args.steps
    vmax = float(np.sqrt((p.vm[:, :3].astype(np.float64) ** 2).sum(1)).max())
    dt = 0.99 * skin / (K * vmax)
    x0, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    s = torch.cuda.current_stream()

    def ev():
        return torch.cuda.Event(enable_timing=True)

    # ---- full: re-bin and re-sort every step (positions drifted on the host side of the API,
    # wrapped into [0, 1) as the re-binning requires) -----------------------------------------
    full = pv.DensityPass(p.nc, p.n)
    xu = x0.clone()
    xs = [x0.clone()]
    for k in range(K):                                   # x_{k+1} = x_k + v dt (as sph_drift rounds it)
        xu[:, :3] = xu[:, :3] + (v[:, :3] * dt)
        xn = xu.clone()
        w = torch.remainder(xu[:, :3], 1.0)
        xn[:, :3] = torch.where(w >= 1.0, torch.zeros_like(w), w)   # -tiny mod 1 rounds to 1.0
        xs.append(xn)
    full.run(xs[1], v)                                   # warm-up
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record(s)
    for k in range(1, K + 1):
        full.run(xs[k], v)
    e1.record(s)
    torch.cuda.synchronize()
    ms_full = e0.elapsed_time(e1) / K
    rho_full = full.out.rho.clone()                      # state K
    st_full = pv.Stats()
    full.run(xs[K], v, stats=st_full)                    # state K again, counted
    torch.cuda.synchronize()
    full.check()

    # ---- reuse: build once with skin, then drift + density ------------------------------------
    re = pv.DensityPass(p.nc, p.n, skin=skin)
    pv.sph_build_cells(re.grid, x0, v, re.cells, re.ws)
    pv.sph_sort_cells(re.grid, re.cells, re.ws)
    pv.sph_density_all(re.grid, re.cells, re.out, re.ws)  # warm-up on state 0
    torch.cuda.synchronize()
    md = torch.zeros(1, dtype=torch.float32, device="cuda")
    e0, e1 = ev(), ev()
    e0.record(s)
    for k in range(1, K + 1):
        pv.sph_drift(re.grid, re.cells, dt, md)
        pv.sph_density_all(re.grid, re.cells, re.out, re.ws)
    e1.record(s)
    torch.cuda.synchronize()
    re.check()
    ms_reuse = e0.elapsed_time(e1) / K
    st_re = pv.Stats()
    pv.sph_density_all(re.grid, re.cells, pv.Out.alloc(p.n), re.ws, stats=st_re)   # state K again, counted
    torch.cuda.synchronize()
    cf, cr = st_full.read(), st_re.read()
    drift_bound = K * float(md.item())
    rel = float(((re.out.rho - rho_full).abs() / rho_full).max())
    line = {"benchmark": "pseudo-Verlet list reuse (P:102 max_dx)", "config": args.config, "n_particles": p.n,
            "steps": K, "skin_over_cl": args.skin_frac, "dt": dt, "displacement_bound": drift_bound,
            "ms_per_step_full": ms_full, "ms_per_step_reuse": ms_reuse, "speedup": ms_full / ms_reuse,
            "candidates_full": int(sum(cf["cand"])), "candidates_reuse": int(sum(cr["cand"])),
            "candidate_increase": sum(cr["cand"]) / max(1, sum(cf["cand"])) - 1.0,
            "interactions_full": int(sum(cf["hits"])), "interactions_reuse": int(sum(cr["hits"])),
            "rho_max_rel_diff_full_vs_reuse": rel, "dtype": "f32", "data": "synthetic"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
