"""Lane efficiency of k_density_v5's sweeps and drains (DESIGN.md §6.1 round 2): builds
exp/so_v5stats.so (-DV5_STATS: per-warp counters in the kernel) if missing or stale, runs one
density pass per config and prints, per particle, the issued sweep lane-slots against the
window candidates and the drain lane-slots against the popped hits.
usage (GPU): python scripts/v5_lane_stats.py c3 [c5 ...]  (profiling helper, not product code)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _variant import build_variant  # noqa: E402
from paper_1804_06231_b200 import _lib  # noqa: E402

L = _lib.load(build_variant("so_v5stats.so", ["V5_STATS"]))
import paper_1804_06231_b200 as pv  # noqa: E402
import synth  # noqa: E402

for cfg in sys.argv[1:] or ["c3"]:
    p = synth.make(cfg)
    buf = (ctypes.c_ulonglong * 16)()
    L.sph_debug_v5(buf)
    b0 = list(buf)
    pv.density(p.xyzh, p.vm, p.nc, stats=False)
    L.sph_debug_v5(buf)
    b = [x - y for x, y in zip(buf, b0)]
    n = p.n
    print(f"{cfg}: sweep lane-slots {b[12] / n:.1f}, window candidates {b[13] / n:.1f} "
          f"(efficiency {b[13] / max(1, b[12]):.3f}); drain lane-slots/2 {b[10] / n:.1f}, popped {b[11] / n:.1f} "
          f"(efficiency {b[11] / max(1, b[10]):.3f}); left for the final drain {b[15] / n:.2f}; warps {b[9]}")
