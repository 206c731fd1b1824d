"""List reuse across steps ("max_dx"): cells and
sorted lists built once, positions drifted by sph_drift, density with windows widened by
4 skin -- exact against the fp64 oracle on the drifted positions."""
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


def _drifted(xyzh, vm, dt):
    """x + v dt with the kernel's two fp32 roundings (v dt, then the sum)."""
    x = xyzh.copy()
    dt32 = np.float32(dt)
    for a in range(3):
        x[:, a] = (xyzh[:, a] + (vm[:, a] * dt32).astype(np.float32)).astype(np.float32)
    return x


@pytest.mark.parametrize("frac", [0.5, 0.95])
def test_drift_then_density_vs_oracle(pv, frac):
    p = synth.tiny_random_set(seed=11, n=12000, nc=8, h_frac=0.8)     # gamma h <= 0.8 C_l
    cl = 1.0 / p.nc
    skin = 0.08 * cl                                                   # gamma h + 2 skin <= 0.96 C_l
    vnorm = np.sqrt((p.vm[:, :3].astype(np.float64) ** 2).sum(1)).max()
    dt = frac * skin / vnorm
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    dp = pv.DensityPass(p.nc, p.n, skin=skin)
    pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws)
    pv.sph_sort_cells(dp.grid, dp.cells, dp.ws)
    md = torch.zeros(1, dtype=torch.float32, device="cuda")
    pv.sph_drift(dp.grid, dp.cells, dt, md)
    pv.sph_density_all(dp.grid, dp.cells, dp.out, dp.ws)
    dp.check()
    got = dp.out.to_numpy()
    xd = _drifted(p.xyzh, p.vm, dt)
    assert (xd[:, :3] < 0).any() or (xd[:, :3] >= 1).any()           # some particles left the box
    compare(got, oracle.bruteforce(xd, p.vm), None, f"reuse frac={frac}")
    step = (p.vm[:, :3] * np.float32(dt)).astype(np.float32).astype(np.float64)   # the fp32 increments
    disp = np.sqrt((step ** 2).sum(1)).max()
    assert abs(float(md.item()) - disp) <= 1e-6 * disp


def test_two_drifts_accumulate(pv):
    """Two drifts within one skin (the displacement adds up) still give exact results."""
    p = synth.tiny_random_set(seed=12, n=8000, nc=6, h_frac=0.8)
    skin = 0.08 / p.nc
    dt = 0.45 * skin / np.sqrt((p.vm[:, :3].astype(np.float64) ** 2).sum(1)).max()
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    dp = pv.DensityPass(p.nc, p.n, skin=skin)
    pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws)
    pv.sph_sort_cells(dp.grid, dp.cells, dp.ws)
    pv.sph_drift(dp.grid, dp.cells, dt)
    pv.sph_drift(dp.grid, dp.cells, dt)
    pv.sph_density_all(dp.grid, dp.cells, dp.out, dp.ws)
    dp.check()
    xd = _drifted(_drifted(p.xyzh, p.vm, dt), p.vm, dt)
    compare(dp.out.to_numpy(), oracle.bruteforce(xd, p.vm), None, "two drifts")


def test_build_rejects_support_plus_skin_above_cell(pv):
    """gamma h + 2 skin > C_l for a home particle -> SPH_EH_RANGE (the 27 cells would no
    longer hold every neighbour after a drift)."""
    p = synth.tiny_random_set(seed=13, n=2000, nc=6, h_frac=0.95)
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    dp = pv.DensityPass(p.nc, p.n, skin=0.05 / p.nc)
    pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws)
    assert pv.sph_status(dp.ws) == 2
