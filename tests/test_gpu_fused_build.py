"""sph_build_sort_cells (ABI v7) against sph_build_cells + sph_sort_cells: every output of the
two paths bitwise equal -- cell starts, the SoA arrays, perm, slot_cell, cell_nhome, cell_hmax
and the 13 sorted lists of every cell -- on uniform sets (nearly every cell on the fused
small tier), a clustered set (every sort tier), a slab grid with ghost planes and empty input.
The oracle parity of the lists and of the density (tests/test_gpu_parity.py) runs through both
paths: DensityPass.run uses the fused call, the build/sort tests the separate ones."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pv():
    import paper_1804_06231_b200 as pv
    assert torch.cuda.is_available()
    pv.load()
    return pv


def _state(dp, n):
    c = dp.cells
    return dict(start=c.cell_start.cpu().numpy(), xyzh=c.xyzh[:n].cpu().numpy(), vm=c.vm[:n].cpu().numpy(),
                perm=c.perm[:n].cpu().numpy(), slot_cell=c.slot_cell[:n].cpu().numpy(),
                nhome=c.cell_nhome.cpu().numpy(), hmax=c.cell_hmax.cpu().numpy(),
                order=c.order[:, :n].cpu().numpy())


def _both(pv, xyzh, vm, nc, n_own=None, n_ghost=0, **grid):
    x, v = torch.from_numpy(xyzh).cuda(), torch.from_numpy(vm).cuda()
    n = xyzh.shape[0]
    n_own = n if n_own is None else n_own
    out = []
    for fused in (False, True):
        dp = pv.DensityPass(nc, n_own, capacity=max(n, 1), **grid)
        dp.cells.order.fill_(-1)
        if fused:
            pv.sph_build_sort_cells(dp.grid, x, v, dp.cells, dp.ws, n_own=n_own, n_ghost=n_ghost)
        else:
            pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws, n_own=n_own, n_ghost=n_ghost)
            pv.sph_sort_cells(dp.grid, dp.cells, dp.ws)
        dp.check()
        out.append(_state(dp, dp.cells.n))
    return out


def _assert_equal(a, b):
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_fused_equals_separate_uniform(pv, cfg):
    p = synth.make(cfg)
    _assert_equal(*_both(pv, p.xyzh, p.vm, p.nc))


def test_fused_equals_separate_every_tier(pv):
    """Cells of 0 .. ~5000 particles: the fused small tier (<= 32) beside k_sort_mid,
    k_sort_warp256 and the radix tiers, which the fused call leaves to sph_sort_cells."""
    rng = np.random.default_rng(7)
    nc = 6
    pts = [rng.random((3000, 3))]                                  # background, ~14 per cell
    for occ, c in ((40, (1, 1, 1)), (200, (2, 3, 4)), (700, (4, 4, 0)), (5000, (5, 0, 2))):
        pts.append((np.array(c) + rng.random((occ, 3))) / nc)
    pos = np.floor(np.concatenate(pts) * 2 ** 24) / 2 ** 24
    n = pos.shape[0]
    xyzh = np.zeros((n, 4), np.float32)
    xyzh[:, :3] = pos
    xyzh[:, 3] = 0.4 / nc / synth.GAMMA
    vm = np.zeros_like(xyzh)
    vm[:, :3] = rng.normal(size=(n, 3))
    vm[:, 3] = 1.0 / n
    perm = rng.permutation(n)
    _assert_equal(*_both(pv, xyzh[perm].copy(), vm[perm].copy(), nc))


def test_fused_equals_separate_slab_with_ghosts(pv):
    p = synth.make("c1")
    nc = p.nc
    ix = np.clip(np.floor(p.xyzh[:, 0].astype(np.float64) * nc).astype(int), 0, nc - 1)
    own = (ix >= 1) & (ix < 3)
    ghost = (ix == 0) | (ix == 3)
    xyzh = np.concatenate([p.xyzh[own], p.xyzh[ghost]])
    vm = np.concatenate([p.vm[own], p.vm[ghost]])
    _assert_equal(*_both(pv, xyzh, vm, nc, n_own=int(own.sum()), n_ghost=int(ghost.sum()), x_lo=1, x_hi=3,
                         ghost_x=1))


def test_fused_zero_particles(pv):
    z = np.zeros((0, 4), np.float32)
    a, b = _both(pv, z, z, 4)
    _assert_equal(a, b)
