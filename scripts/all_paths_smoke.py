"""One small invocation of every library path, each followed by the status check: build, sort
(every tier incl. the radix tiers), the gather pass (v5 tiles + the dense engine), the level
passes, the symmetric whole pass and the reuse loop.  (compute-sanitizer is not available on
the GPU pool; the library's own status word and bounds checks are what this exercises.)
usage (GPU): python scripts/all_paths_smoke.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1804_06231_b200 as pv  # noqa: E402
import synth  # noqa: E402

pv.load()
p = synth.make("c1")
x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
dp = pv.DensityPass(p.nc, p.n)
dp.run(x, v)
dp.check()
pv.sph_density_all_sym(dp.grid, dp.cells, dp.out, dp.ws)
dp.check()
# one dense cell (radix sort tiers, k_stable_radix, k_density_dense with its z-sorted self sweep)
rng = np.random.default_rng(3)
occ, nc, Cl, nbg = 3000, 4, 0.25, 300
xyzh = np.zeros((nbg + occ, 4), np.float32)
xyzh[:nbg, :3] = rng.integers(0, 2 ** 24, size=(nbg, 3)) / 2 ** 24
xyzh[nbg:, :3] = np.floor((1 + rng.random((occ, 3))) * Cl * 2 ** 24) / 2 ** 24
xyzh[:, 3] = (0.2 * Cl / synth.GAMMA) * (1 - 0.5 * rng.random(nbg + occ))
vm = np.zeros_like(xyzh)
vm[:, :3] = rng.standard_normal((nbg + occ, 3))
vm[:, 3] = 1.0 / (nbg + occ)
dq = pv.DensityPass(nc, xyzh.shape[0])
dq.run(torch.from_numpy(xyzh).cuda(), torch.from_numpy(vm).cuda())
dq.check()
# level passes on a small clustered set
hx = p.xyzh.copy()
hx[:, 3] *= np.where(np.arange(p.n) % 3 == 0, 0.3, 1.0).astype(np.float32)
lv = pv.level_grids(hx[:, 3], p.nc)
lp = pv.LevelPasses(lv, p.n)
lp.run(torch.from_numpy(hx).cuda(), v)
lp.check()
# reuse loop: a few drifted steps with a rebuild
loop = pv.ReuseLoop(p.nc, p.n, 0.01 * p.box / p.nc, box=p.box)
loop.start(x.clone(), v)
dt = 0.3 * (0.01 * p.box / p.nc) / max(loop.vmax, 1e-30)
for _ in range(5):
    loop.step(dt)
loop.check()
torch.cuda.synchronize()
print("all paths ok")
