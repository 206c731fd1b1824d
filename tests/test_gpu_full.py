"""Full-size parity at BASELINE.json's configurations, in the launch configuration bench.py
times (slabs.SlabRunner on one GPU: build_cells -> sort_cells -> density_all per level grid,
levels as bench.py picks them), checked against the fp64 cell-list oracle on the samples
SURVEY.md §8(c) names: c3 every particle; c5 and c4 2^20 random particles plus every particle
of the 16 slab-boundary planes (first and last plane of each slab at 2/4/8 GPUs, equal and
cost-balanced cuts), plus whole-set invariants."""
import numpy as np
import pytest

import oracle
import synth
from tests._compare import compare

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def pv():
    import paper_1804_06231_b200 as pv
    pv.load()
    return pv


def _run_bench_path(pv, p, cfg):
    """Exactly bench.py's N=1 step: SlabRunner over the single slab, level grids as bench.py
    chooses them (3 for the clustered c4, else 1)."""
    from paper_1804_06231_b200 import slabs
    nlev = 3 if cfg == "c4" else 1
    levels = pv.level_grids(p.xyzh[:, 3], p.nc, max_levels=nlev) if nlev > 1 else None
    runner = slabs.SlabRunner(slabs.Slab.single(p), levels=levels)
    runner.upload()
    st = pv.Stats()
    runner.step(stats=st)
    runner.check()
    out = runner.out.to_numpy()
    del runner
    torch.cuda.empty_cache()
    return out, st.read(), levels


def _boundary_planes(p):
    """Cell x-planes that are the first or last plane of some slab at 2, 4 or 8 GPUs, for
    equal cuts and for the cost-balanced cuts bench.py uses on c4."""
    from paper_1804_06231_b200 import slabs
    planes = set()
    costs = None
    for w in (2, 4, 8):
        cuts = [slabs.slab_bounds(p.nc, w, r) for r in range(w)]
        if costs is None:
            costs = slabs.plane_costs(p.xyzh, p.nc, p.box)
        cuts += slabs.balanced_bounds(costs, w)
        for lo, hi in cuts:
            planes.update((lo % p.nc, (hi - 1) % p.nc))
    return sorted(planes)


def _sample(p, k, seed):
    rng = np.random.default_rng(seed)
    idx = rng.choice(p.n, k, replace=False)
    pl = np.clip(np.floor(p.xyzh[:, 0].astype(np.float64) * p.nc), 0, p.nc - 1).astype(np.int64)
    planes = _boundary_planes(p)
    b = np.nonzero(np.isin(pl, planes))[0]
    return np.unique(np.concatenate([idx, b])), len(planes), b.size


def test_c3_full_size_every_particle(pv):
    """c3 (2,097,152 particles, 47^3 cells): every particle against the cell-list oracle."""
    p = synth.make("c3")
    got, st, _ = _run_bench_path(pv, p, "c3")
    rep = compare(got, oracle.celllist(p.xyzh, p.vm, p.nc), None, "c3 full")
    assert rep["checked"] == p.n
    assert sum(st["hits"]) == int(got["nngb"].astype(np.int64).sum())


def test_c5_full_size_sampled(pv):
    """c5 (134,217,728 particles, 184^3 cells): 2^20 random + every particle of the 16
    slab-boundary planes (~11.6 M)."""
    p = synth.make("c5")
    got, st, _ = _run_bench_path(pv, p, "c5")
    idx, nplanes, nb = _sample(p, 1 << 20, 55)
    assert nplanes >= 16 and nb > 10_000_000
    rep = compare(got, oracle.celllist(p.xyzh, p.vm, p.nc, targets=idx), idx, "c5 2^20 + 16 planes")
    assert rep["checked"] >= nb
    # whole-set invariants: every particle written once, counters consistent
    assert np.all(np.isfinite(got["rho"])) and np.all(got["rho"] > 0)
    assert sum(st["hits"]) == int(got["nngb"].astype(np.int64).sum())
    assert 45.0 < got["nngb"].mean() < 55.0                     # ~48 neighbours (BASELINE configs)


def test_c4_clustered_three_levels_sampled(pv):
    """c4 (16,777,216 particles, 60 % in 512 Plummer spheres, 83^3 cells) through the
    three level grids bench.py runs: 2^20 random particles, every particle of the slab-boundary
    planes (equal and balanced cuts), and the densest cells' particles."""
    p = synth.make("c4")
    got, st, levels = _run_bench_path(pv, p, "c4")
    assert levels is not None and len(levels) == 3
    idx, _, nb = _sample(p, 1 << 20, 44)
    cell, order, start = oracle.bin_cells(p.xyzh, p.nc)
    occ = np.diff(start)
    dense = np.argsort(occ)[-3:]
    extra = np.concatenate([order[start[c]:start[c + 1]] for c in dense])
    idx = np.unique(np.concatenate([idx, extra]))
    rep = compare(got, oracle.celllist(p.xyzh, p.vm, p.nc, targets=idx), idx, "c4 3 levels")
    assert rep["checked"] >= nb
    assert np.all(np.isfinite(got["rho"])) and np.all(got["rho"] > 0)
    assert sum(st["hits"]) == int(got["nngb"].astype(np.int64).sum())
