"""Per-phase warp-cycle breakdown of k_density_v4 (round 1): builds
exp/so_phase.so (-DPVSPH_PHASE_TIMING) if it is missing or stale, then runs the v4 engine on one
config: `PVSPH_ENGINE=v4 python scripts/phase_timing.py c5` on a GPU (profiling helper, not
product code)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_1804_06231_b200 import _lib
from _variant import build_variant
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
L = _lib.load(build_variant("so_phase.so", ["PVSPH_PHASE_TIMING"]))
import paper_1804_06231_b200 as pv
import synth
p = synth.make(cfg)
x = torch.from_numpy(p.xyzh).cuda(); v = torch.from_numpy(p.vm).cuda()
dp = pv.DensityPass(p.nc, p.n)
pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws); pv.sph_sort_cells(dp.grid, dp.cells, dp.ws)
buf = (ctypes.c_ulonglong * 12)()
pv.sph_density_all(dp.grid, dp.cells, dp.out, dp.ws); torch.cuda.synchronize()
L.sph_debug_phase_cycles(buf, 1)
pv.sph_density_all(dp.grid, dp.cells, dp.out, dp.ws); torch.cuda.synchronize()
L.sph_debug_phase_cycles(buf, 1)
names = ["stage", "search", "sweep", "drain", "final drain", "barrier(top)", "  P/V copy", "  list copy",
         "  table scan", "  tab->seg sizes", "  seg scan"]
tot = sum(buf[k] for k in range(6))
for k in range(11):
    print(f"{names[k]:14s} {buf[k]:>16d} warp-cycles  {100.0 * buf[k] / tot:5.1f} %")
