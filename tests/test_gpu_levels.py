"""Level passes for clustered data: several uniform cell grids, each home
to the particles whose support fits its cells, every grid binning all particles as
neighbour sources.  Parity with the fp64 oracle on clustered sets, the home split of a
single pass, and agreement with the single-grid engine."""
import numpy as np
import pytest

import oracle
import synth
from tests._compare import compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pv():
    import paper_1804_06231_b200 as pv
    pv.load()
    return pv


@pytest.fixture(scope="module")
def clustered():
    # a small c4-like set: 60 % in 16 Plummer spheres, 40 % background; nc from the
    # background density as in reading B22 (13 cells for 65,536 particles)
    from synth import gen
    return gen.clustered_set("cl64k", seed=7, n=65536, nc=13, n_spheres=16)


def test_level_grids_partition(pv, clustered):
    lv = pv.level_grids(clustered.xyzh[:, 3], clustered.nc, max_levels=3)
    assert [nc for nc, _, _ in lv] == [13, 26, 52]
    h = clustered.xyzh[:, 3]
    home = np.zeros(h.size, np.int64)
    for nc, lo, hi in lv:
        sel = (h > lo) & (h <= hi)
        home += sel
        assert np.all(synth.GAMMA * h[sel].astype(np.float64) <= 1.0 / nc)
    assert np.all(home == 1)                     # every particle home on exactly one level


def test_levels_vs_oracle(pv, clustered):
    p = clustered
    lv = pv.level_grids(p.xyzh[:, 3], p.nc, max_levels=3)
    got = pv.density_levels(p.xyzh, p.vm, lv, stats=True)
    ref = oracle.celllist(p.xyzh, p.vm, p.nc)
    compare(got, ref, None, "levels cl64k")
    assert sum(got["stats"]["hits"]) == int(got["nngb"].astype(np.int64).sum())


def test_levels_match_single_grid(pv, clustered):
    """Same neighbour sets as the single-grid engine (exact counts); values within fp32
    summation-order differences."""
    p = clustered
    one = pv.density(p.xyzh, p.vm, p.nc)
    lv = pv.density_levels(p.xyzh, p.vm, pv.level_grids(p.xyzh[:, 3], p.nc, max_levels=3))
    assert np.array_equal(one["nngb"], lv["nngb"])
    assert np.max(np.abs(one["rho"] / lv["rho"] - 1)) < 1e-5


def test_home_split_leaves_others_untouched(pv, clustered):
    """One pass with a home range writes exactly its home particles' outputs."""
    p = clustered
    lv = pv.level_grids(p.xyzh[:, 3], p.nc, max_levels=3)
    nc, lo, hi = lv[1]
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    dp = pv.DensityPass(nc, p.n, h_home=(lo, hi))
    dp.out.rho.fill_(-7.0)
    dp.out.nngb.fill_(-7)
    dp.run(x, v)
    dp.check()
    got = dp.out.to_numpy()
    h = p.xyzh[:, 3]
    home = (h > lo) & (h <= hi)
    assert np.all(got["rho"][~home] == -7.0) and np.all(got["nngb"][~home] == -7)
    idx = np.nonzero(home)[0]
    ref = oracle.celllist(p.xyzh, p.vm, p.nc, targets=idx)
    compare(got, ref, idx, "home split")


def test_large_h_neighbour_only_accepted(pv, clustered):
    """On a fine grid, particles whose support exceeds the cell are neighbour-only: the build
    accepts them (no SPH_EH_RANGE) when they are outside the home range, rejects them when
    all particles are home."""
    p = clustered
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    lv = pv.level_grids(p.xyzh[:, 3], p.nc, max_levels=3)
    nc, lo, hi = lv[-1]
    dp = pv.DensityPass(nc, p.n, h_home=(lo, hi))
    dp.run(x, v)
    dp.check()                                   # fine: big-h particles are not home here
    dp2 = pv.DensityPass(nc, p.n)
    pv.sph_build_cells(dp2.grid, x, v, dp2.cells, dp2.ws)
    assert pv.sph_status(dp2.ws) == 2            # SPH_EH_RANGE without a home range
