"""x-slab decomposition on one GPU (fake ranks: the exchange done with device copies):
outputs bitwise identical to the single-GPU pass for p = 2, 3, 4."""
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


@pytest.mark.parametrize("cfg,world", [("c1", 2), ("c2", 2), ("c2", 3), ("c2", 4), ("c3", 2), ("c3", 4)])
def test_fake_ranks_bitwise_equal_single(pv, cfg, world):
    from paper_1804_06231_b200.slabs import FakeRanks
    p = synth.make(cfg)
    single = pv.density(p.xyzh, p.vm, p.nc)
    fr = FakeRanks(p, world)
    fr.step()
    got = fr.gather()
    for f in single:
        assert np.array_equal(single[f], got[f]), (cfg, world, f)
    if cfg == "c1":
        compare(got, oracle.bruteforce(p.xyzh, p.vm), None, f"{cfg} p={world}")


def test_slab_boundary_particles_vs_oracle(pv):
    """Particles within one cell of a slab boundary (p = 4, c3) against the oracle."""
    from paper_1804_06231_b200.slabs import FakeRanks, planes_of, slab_bounds
    p = synth.make("c3")
    fr = FakeRanks(p, 4)
    fr.step()
    got = fr.gather()
    pl = planes_of(p.xyzh, p.nc)
    edges = set()
    for r in range(4):
        lo, hi = slab_bounds(p.nc, 4, r)
        edges |= {lo, hi - 1}
    idx = np.nonzero(np.isin(pl, sorted(edges)))[0]
    idx = idx[:: max(1, idx.size // 50000)]
    compare(got, oracle.celllist(p.xyzh, p.vm, p.nc, targets=idx), idx, "slab boundaries")


def test_e2e_pipeline_results(pv):
    """The pipelined host-buffer path (bench.py's e2e leg: double-buffered inputs/outputs,
    copies on their own streams) returns exactly the device pass's results."""
    from paper_1804_06231_b200.slabs import Slab, SlabRunner
    p = synth.make("c2")
    single = pv.density(p.xyzh, p.vm, p.nc)
    r = SlabRunner(Slab.from_set(p, 0, 1))
    r.upload()
    ms, h2d, d2h = r.e2e_time(steps=3, warmup=1)
    assert ms > 0 and h2d == 32 * p.n and d2h == 36 * p.n
    got = {k: v.numpy() for k, v in r.e2e_host.items()}
    for f in ("rho", "rho_dh", "wcount", "wcount_dh", "div_v", "nngb"):
        assert np.array_equal(single[f], got[f]), f
    for k, ax in enumerate("xyz"):
        assert np.array_equal(single["curl_" + ax], got["curl_v"][k]), ax


def test_symmetric_pairs_on_slabs(pv):
    """sph_density_pair_sym on x-slabs: j in a ghost cell is never updated.  Each rank lists,
    for every owned cell, the 13 positive offsets (an owned or ghost neighbour) plus the
    negative offsets that land in a ghost plane; + self over owned cells + finalize, gathered
    over ranks == the oracle."""
    import torch
    from paper_1804_06231_b200.slabs import FakeRanks
    p = synth.make("c2")
    fr = FakeRanks(p, 2)
    fr.step()                                    # builds cells with ghosts on every rank
    res = {}
    for r in fr.runners:
        ny = nz = p.nc
        nxl = r.nxl
        cells = np.arange(nxl * ny * nz)
        jx, iy, iz = cells // (ny * nz), (cells // nz) % ny, cells % nz
        own = (jx >= 1) & (jx < nxl - 1)
        pairs = []
        for a in (-1, 0, 1):
            for b in (-1, 0, 1):
                for c in (-1, 0, 1):
                    if (a, b, c) == (0, 0, 0):
                        continue
                    kx = jx + a
                    cj = (kx * ny + (iy + b) % ny) * nz + (iz + c) % nz
                    ghost_j = (kx == 0) | (kx == nxl - 1)
                    sel = own & (kx >= 0) & (kx < nxl) & (((a, b, c) > (0, 0, 0)) | ghost_j)
                    pairs.append(np.stack([cells[sel], cj[sel]], 1))
        pr = torch.from_numpy(np.concatenate(pairs).astype(np.int32)).cuda().contiguous()
        acc = pv.Out.alloc(r.n_own, zero=True)
        owned = torch.from_numpy(cells[own].astype(np.int32)).cuda()
        pv.sph_density_self(r.grid, r.cells, owned, acc, r.ws)
        pv.sph_density_pair_sym(r.grid, r.cells, pr, acc, r.ws)
        pv.sph_density_finalize(acc)
        r.check()
        for k, v in acc.to_numpy().items():
            res.setdefault(k, np.zeros(p.n, v.dtype))[r.slab.gid] = v
    compare(res, oracle.celllist(p.xyzh, p.vm, p.nc), None, "symmetric pairs on slabs")


@pytest.mark.parametrize("world", [2, 3])
def test_balanced_slabs_bitwise_equal_single(pv, world):
    """Cost-balanced (uneven) x-slab cuts on clustered data: outputs bitwise identical to the
    single-GPU pass on the same grid (the tile cut and every particle's summation order do
    not depend on where the slabs are cut)."""
    from paper_1804_06231_b200.slabs import FakeRanks, slab_bounds
    p = synth.clustered_set("cl64k", seed=7, n=65536, nc=13, n_spheres=16)
    single = pv.density(p.xyzh, p.vm, p.nc)
    fr = FakeRanks(p, world, balance=True)
    assert fr.bounds != [slab_bounds(p.nc, world, r) for r in range(world)]   # really uneven
    fr.step()
    got = fr.gather()
    for f in single:
        assert np.array_equal(single[f], got[f]), (world, f)


@pytest.mark.parametrize("world,balance", [(2, False), (3, True)])
def test_levels_on_slabs_bitwise_equal_single(pv, world, balance):
    """Level passes on x-slabs: every level grid cut at the same x, its
    thinner ghost planes taken from the coarse ghosts -- outputs bitwise identical to the
    level passes on one GPU."""
    from paper_1804_06231_b200.slabs import FakeRanks
    p = synth.clustered_set("cl64k", seed=7, n=65536, nc=13, n_spheres=16)
    lv = pv.level_grids(p.xyzh[:, 3], p.nc, max_levels=3)
    assert len(lv) == 3
    single = pv.density_levels(p.xyzh, p.vm, lv)
    fr = FakeRanks(p, world, balance=balance, levels=lv)
    fr.step()
    got = fr.gather()
    for f in single:
        if f == "stats":
            continue
        assert np.array_equal(single[f], got[f]), (world, f)


def test_select_planes_vs_numpy(pv):
    """sph_select_planes: the owned particles of planes x_lo and x_hi-1, in input order, with
    exact counts (the binning rule of sph_build_cells)."""
    import torch
    from paper_1804_06231_b200.slabs import Slab, planes_of
    p = synth.make("c2")
    s = Slab.from_set(p, 1, 3)
    g = pv.make_grid(p.nc, 1.0, p.gamma, s.x_lo, s.x_hi, 1)
    x, v = torch.from_numpy(s.xyzh).cuda(), torch.from_numpy(s.vm).cuda()
    cap = s.n_own
    sx = torch.empty((2, cap, 4), dtype=torch.float32, device="cuda")
    sv = torch.empty_like(sx)
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    ws = pv.alloc_workspace(g, s.n_own)
    pv.sph_select_planes(g, x, v, s.n_own, sx, sv, cnt, ws)
    pv.check_status(ws)
    pl = planes_of(s.xyzh, p.nc)
    for k, plane in enumerate((s.x_lo, s.x_hi - 1)):
        idx = np.nonzero(pl == plane)[0]
        assert int(cnt[k]) == idx.size > 0
        assert np.array_equal(sx[k, :idx.size].cpu().numpy(), s.xyzh[idx])
        assert np.array_equal(sv[k, :idx.size].cpu().numpy(), s.vm[idx])


def test_select_planes_capacity(pv):
    """A boundary plane longer than the send buffer: SPH_ECAPACITY in the status word."""
    import torch
    from paper_1804_06231_b200.slabs import Slab
    p = synth.make("c2")
    s = Slab.from_set(p, 0, 2)
    g = pv.make_grid(p.nc, 1.0, p.gamma, s.x_lo, s.x_hi, 1)
    x, v = torch.from_numpy(s.xyzh).cuda(), torch.from_numpy(s.vm).cuda()
    sx = torch.empty((2, 8, 4), dtype=torch.float32, device="cuda")
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    ws = pv.alloc_workspace(g, s.n_own)
    pv.sph_select_planes(g, x, v, s.n_own, sx, torch.empty_like(sx), cnt, ws)
    assert pv.sph_status(ws) == 3
    assert int(cnt[0]) > 8                       # the true count is still reported


def test_mask_ghost_rows(pv):
    """sph_mask_ghost_rows: rows past each received count become the dead particle, the rest
    is untouched; counts read on the device (here 3 of 8 and 8 of 8, then 0 of 8)."""
    import torch
    cap = 8
    x = torch.rand((2, cap, 4), dtype=torch.float32, device="cuda")
    v = torch.rand((2, cap, 4), dtype=torch.float32, device="cuda")
    x0, v0 = x.clone(), v.clone()
    dx, dv = [0.5, 0.25, 0.125, 1e-6], [0.0, 0.0, 0.0, 1.0]
    for counts in ([3, 8], [0, 5]):
        x.copy_(x0)
        v.copy_(v0)
        n = torch.tensor(counts, dtype=torch.int64, device="cuda")
        pv.sph_mask_ghost_rows(x, v, n, dx, dv)
        torch.cuda.synchronize()
        for k in range(2):
            c = counts[k]
            assert torch.equal(x[k, :c], x0[k, :c]) and torch.equal(v[k, :c], v0[k, :c])
            assert torch.all(x[k, c:] == torch.tensor(dx, device="cuda"))
            assert torch.all(v[k, c:] == torch.tensor(dv, device="cuda"))


def test_partition_migrants_and_merge_by_id(pv):
    """sph_partition_migrants == the split rule (stable, input order kept) on random wrapped
    positions incl. the faces of the neighbour planes; sph_merge_by_id of the three lists (and
    of received migrants with fresh ids) == the argsort-by-id merge; counts exact."""
    import torch
    from paper_1804_06231_b200.slabs import split_migrants
    rng = np.random.default_rng(7)
    nc, x_lo, x_hi, n = 10, 3, 6, 20000
    x = np.zeros((n, 4), np.float32)
    x[:, :3] = rng.random((n, 3))
    x[:n // 10, 0] = (rng.integers(0, nc, n // 10) / nc).astype(np.float32)      # exactly on plane faces
    x[:, 3] = 0.01
    v = rng.standard_normal((n, 4)).astype(np.float32)
    gid = np.sort(rng.choice(10 * n, n, replace=False)).astype(np.int64)
    X, V, G = (torch.from_numpy(a).cuda() for a in (x, v, gid))
    g = pv.make_grid(nc, 1.0, 1.825742, x_lo, x_hi, 1)
    ws = pv.alloc_workspace(g, n)
    bufs = [[torch.zeros((n, 4), dtype=torch.float32, device="cuda"), torch.zeros((n, 4), dtype=torch.float32,
             device="cuda"), torch.zeros(n, dtype=torch.int64, device="cuda")] for _ in range(3)]
    cnt = torch.zeros(3, dtype=torch.int64, device="cuda")
    pv.sph_partition_migrants(g, n, X, V, G, bufs[0], bufs[1], bufs[2], cnt, ws)
    assert pv.sph_status(ws) == 0
    masks = split_migrants(X, nc, 1.0, x_lo, x_hi)
    c = cnt.tolist()
    for k, m in enumerate(masks):
        idx = torch.nonzero(m).squeeze(1)
        assert c[k] == idx.numel()
        assert torch.equal(bufs[k][0][:c[k]], X[idx]) and torch.equal(bufs[k][1][:c[k]], V[idx])
        assert torch.equal(bufs[k][2][:c[k]], G[idx])
    # merge: keep + lo + hi back == the original set in gid order
    ox, ov, og = torch.empty_like(X), torch.empty_like(V), torch.empty_like(G)
    pv.sph_merge_by_id([(bufs[2][0], bufs[2][1], bufs[2][2], c[2]), (bufs[0][0], bufs[0][1], bufs[0][2], c[0]),
                        (bufs[1][0], bufs[1][1], bufs[1][2], c[1])], ox, ov, og)
    torch.cuda.synchronize()
    assert torch.equal(og, G) and torch.equal(ox, X) and torch.equal(ov, V)
    # an empty list and a partial capacity overflow
    small = [[b[0][:5], b[1][:5], b[2][:5]] for b in bufs[:2]] + [bufs[2]]
    pv.sph_partition_migrants(g, n, X, V, G, small[0], small[1], small[2], cnt, ws)
    assert pv.sph_status(ws) == 3                  # SPH_ECAPACITY: a migrant list above 5
