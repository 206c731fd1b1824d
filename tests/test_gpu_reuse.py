"""List reuse across steps ("max_dx"): cells and
sorted lists built once, positions drifted by sph_drift (per-cell max_dx accumulated), density
with windows widened by 2 max_dx of each neighbour cell -- exact against the fp64 oracle on the
drifted positions; and the ReuseLoop that rebuilds when the skin would be exceeded."""
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
    inc = (xd[:, :3].astype(np.float64) - p.xyzh[:, :3].astype(np.float64))     # the stored increments
    disp = np.sqrt((inc ** 2).sum(1)).max()
    assert disp <= float(md.item()) <= disp * (1 + 1e-5)


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


def _wrap(x):
    """sph_gather_positions' rule: x < 0 -> x + 1, x >= 1 -> x - 1, a result of 1 -> 0 (fp32)."""
    y = x.copy()
    for a in range(3):
        c = y[:, a]
        c = np.where(c < 0, (c + np.float32(1.0)).astype(np.float32), c)
        c = np.where(c >= 1, (c - np.float32(1.0)).astype(np.float32), c)
        c = np.where(c >= 1, np.float32(0.0), c)
        y[:, a] = c.astype(np.float32)
    return y


def test_cell_dx_is_per_cell_max_displacement(pv):
    """cell_dx (the paper's max_dx) equals, per cell, the largest accumulated displacement of its
    particles (host replay of the fp32 drifts), and bounds |x - x_build|."""
    p = synth.tiny_random_set(seed=14, n=6000, nc=6, h_frac=0.8)
    skin = 0.08 / p.nc
    v64 = p.vm[:, :3].astype(np.float64)
    dt = 0.3 * skin / np.sqrt((v64 ** 2).sum(1)).max()
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    dp = pv.DensityPass(p.nc, p.n, skin=skin)
    pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws)
    pv.sph_sort_cells(dp.grid, dp.cells, dp.ws)
    x0 = p.xyzh.copy()
    x1 = _drifted(x0, p.vm, dt)
    x2 = _drifted(x1, p.vm, dt)
    for _ in range(2):
        pv.sph_drift(dp.grid, dp.cells, dt)
    torch.cuda.synchronize()
    acc = np.zeros(p.n)
    for a, b in ((x0, x1), (x1, x2)):
        acc += np.sqrt(((b[:, :3].astype(np.float64) - a[:, :3].astype(np.float64)) ** 2).sum(1))
    cell, order, start = oracle.bin_cells(p.xyzh, p.nc)
    exp = np.zeros(p.nc ** 3)
    np.maximum.at(exp, cell, acc)
    got = dp.cells.cell_dx.cpu().numpy().astype(np.float64)
    assert np.all(got >= exp) and np.all(got <= exp * (1 + 1e-5) + 1e-12)
    true = np.sqrt(((x2[:, :3].astype(np.float64) - x0[:, :3].astype(np.float64)) ** 2).sum(1))
    assert np.all(true <= acc * (1 + 1e-6))


def test_per_cell_windows_are_tighter_than_skin(pv, monkeypatch):
    """With per-cell max_dx the windows grow by 2 max_dx(cj) <= 2 skin instead of the 4 skin the
    other engines use: fewer candidates, the same neighbours (values within tolerance)."""
    p = synth.tiny_random_set(seed=15, n=12000, nc=8, h_frac=0.8)
    skin = 0.08 / p.nc
    dt = 0.25 * skin / np.sqrt((p.vm[:, :3].astype(np.float64) ** 2).sum(1)).max()
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    dp = pv.DensityPass(p.nc, p.n, skin=skin)
    pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws)
    pv.sph_sort_cells(dp.grid, dp.cells, dp.ws)
    pv.sph_drift(dp.grid, dp.cells, dt)
    st = pv.Stats()
    pv.sph_density_all(dp.grid, dp.cells, dp.out, dp.ws, stats=st)
    dp.check()
    got = dp.out.to_numpy()
    xd = _drifted(p.xyzh, p.vm, dt)
    ref = oracle.bruteforce(xd, p.vm)
    compare(got, ref, None, "per-cell max_dx")
    c_cell = sum(st.read()["cand"])
    nd = pv.DensityPass(p.nc, p.n)                      # exact windows on the drifted state itself
    xw = torch.from_numpy(_wrap(xd)).cuda()
    st0 = pv.Stats()
    nd.run(xw, v, stats=st0)
    c_exact = sum(st0.read()["cand"])
    monkeypatch.setenv("PVSPH_ENGINE", "v4")            # the round-1 engine: every window + 4 skin
    st4 = pv.Stats()
    pv.sph_density_all(dp.grid, dp.cells, pv.Out.alloc(p.n), dp.ws, stats=st4)
    monkeypatch.delenv("PVSPH_ENGINE")
    c_skin = sum(st4.read()["cand"])
    assert c_exact <= c_cell < c_skin
    assert sum(st.read()["hits"]) == sum(st4.read()["hits"])


def test_reuse_loop_rebuilds_and_stays_exact(pv):
    """ReuseLoop over 12 steps with a skin of ~4 steps: it rebuilds (gather + wrap + build + sort)
    before the skin could be exceeded; the final state's density equals the fp64 oracle on the
    host replay of the same fp32 drifts and wraps."""
    p = synth.tiny_random_set(seed=16, n=10000, nc=7, h_frac=0.8)
    skin = 0.08 / p.nc
    vmax = np.sqrt((p.vm[:, :3].astype(np.float64) ** 2).sum(1)).max()
    dt = 0.24 * skin / vmax
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    loop = pv.ReuseLoop(p.nc, p.n, skin)
    loop.start(x, v)
    xh = p.xyzh.copy()
    K = 12
    for k in range(K):
        before = loop.rebuilds
        loop.step(dt)
        if loop.rebuilds > before:                      # host replay: the wrap happens at rebuilds
            xh = _wrap(xh)
        xh = _drifted(xh, p.vm, dt)
    loop.check()
    assert loop.rebuilds >= 2 and all(b > 0 for b in loop.rebuild_steps)
    compare(loop.dp.out.to_numpy(), oracle.bruteforce(xh, p.vm), None, "reuse loop")
    gx = torch.empty((p.n, 4), dtype=torch.float32, device="cuda")
    pv.sph_gather_positions(loop.dp.grid, loop.dp.cells, gx, p.n)
    assert np.array_equal(gx.cpu().numpy(), _wrap(xh))


@pytest.mark.parametrize("world", [2, 3])
def test_slab_reuse_with_migration_bitwise_equal_single(pv, world):
    """List reuse on x-slabs (fake ranks, device copies): every rank drifts its owned particles
    and ghost copies; at each rebuild particles that crossed a slab face migrate, the owned set is
    re-merged in global-id order and the ghosts re-exchanged.  Outputs after 12 steps (>= 2
    rebuilds, with migrations) are bitwise those of the single-GPU ReuseLoop, and match the
    fp64 oracle on the host replay."""
    from paper_1804_06231_b200 import slabs
    p = synth.tiny_random_set(seed=21, n=30000, nc=9, h_frac=0.8)
    skin = 0.08 / p.nc
    vmax = float(np.sqrt((p.vm[:, :3].astype(np.float64) ** 2).sum(1)).max())
    dt = 0.24 * skin / vmax
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    one = pv.ReuseLoop(p.nc, p.n, skin)
    one.start(x, v)
    ranks = [slabs.SlabReuse(slabs.Slab.from_set(p, r, world), skin, one.vmax) for r in range(world)]
    tr = slabs.ReuseTransport(ranks)
    tr.start()
    xh = p.xyzh.copy()
    moved = 0
    for k in range(12):
        before = one.rebuilds
        one.step(dt)
        n_before = [rr.n_own for rr in ranks]
        tr.step(dt)
        moved += sum(abs(a - rr.n_own) for a, rr in zip(n_before, ranks))
        if one.rebuilds > before:
            xh = _wrap(xh)
        xh = _drifted(xh, p.vm, dt)
    for rr in ranks:
        rr.check()
    assert one.rebuilds >= 2 and all(rr.rebuilds == one.rebuilds for rr in ranks)
    assert moved > 0                                      # particles did change slabs
    assert sum(rr.n_own for rr in ranks) == p.n
    got = tr.gather(p.n)
    ref1 = one.dp.out.to_numpy()
    for key in ref1:
        assert np.array_equal(got[key], ref1[key]), key
    compare(got, oracle.bruteforce(xh, p.vm), None, f"slab reuse p={world}")


def test_max_speed(pv):
    """sph_max_speed == max of the fp64 norms of the fp32 velocities (the reuse loop's speed
    bound), 0 for no particles."""
    rng = np.random.default_rng(3)
    vm = rng.standard_normal((100003, 4)).astype(np.float32)
    ref = float(np.max(np.sqrt((vm[:, :3].astype(np.float64) ** 2).sum(1))))
    got = pv.sph_max_speed(torch.from_numpy(vm).cuda())
    assert abs(got - ref) <= 1e-15 * ref
    assert pv.sph_max_speed(torch.from_numpy(vm).cuda(), 0) == 0.0
