"""The test27cells workload (bench_test27cells.py): 216 uniform random particles in
every cell of a periodic grid, h = 1.2348 x the mean spacing.  The batched cell-pair and
self kernels the benchmark times, and the whole-pass engine, against the fp64 oracle; the
per-orientation candidate counts against the oracle's Code 2 counts."""
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
def t27():
    return synth.test27cells_set(seed=27, nc=4)


def test_pairs_by_orientation_vs_oracle(pv, t27):
    """Self over all cells + the three orientation classes of bench_test27cells (each a
    separate sph_density_pair call, as timed) + finalize == the oracle; per-kind candidates
    and hits == Code 2 counts; sph_density_all agrees (nngb exact)."""
    import bench_test27cells as b27
    p = t27
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    dp = pv.DensityPass(p.nc, p.n)
    pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws)
    pv.sph_sort_cells(dp.grid, dp.cells, dp.ws)
    acc = pv.Out.alloc(p.n, zero=True)
    st = pv.Stats()
    pv.sph_density_self(dp.grid, dp.cells, torch.arange(p.nc ** 3, dtype=torch.int32, device="cuda"), acc, dp.ws,
                        stats=st)
    for nz in (1, 2, 3):
        pr, k = b27.pairs_of(p.nc, nz, torch)
        assert k == {1: 6, 2: 12, 3: 8}[nz] and pr.shape[0] == k * p.nc ** 3
        pv.sph_density_pair(dp.grid, dp.cells, pr.cuda(), acc, dp.ws, stats=st)
    pv.sph_density_finalize(acc)
    dp.check()
    got = acc.to_numpy()
    ref = oracle.celllist(p.xyzh, p.vm, p.nc)
    compare(got, ref, None, "test27cells self+pairs")
    cnt = st.read()
    c, unsafe = oracle.pv_counts(p.xyzh, p.nc)
    assert unsafe == 0
    tot = c.sum(axis=0)                                   # [kind][naive, pV candidates, hits]
    band = int(ref["band"].sum())                         # pairs within the 1e-6 h^2 band may go either way
    for k in range(4):
        assert abs(cnt["hits"][k] - tot[k, 2]) <= band, k
        assert abs(cnt["cand"][k] - tot[k, 1]) <= max(2, 1e-5 * tot[k, 1]), k
    out = pv.Out.alloc(p.n)
    pv.sph_density_all(dp.grid, dp.cells, out, dp.ws)
    dp.check()
    alln = out.to_numpy()
    assert np.array_equal(alln["nngb"], got["nngb"])
    compare(alln, ref, None, "test27cells density_all")


def _half_offsets_pairs(nc, nonzero=None):
    """(ci, cj) for every cell and one offset of each +-pair (13 per cell; or one class)."""
    cells = np.arange(nc ** 3, dtype=np.int64)
    ix, iy, iz = cells // (nc * nc), (cells // nc) % nc, cells % nc
    out = []
    for a in (-1, 0, 1):
        for b in (-1, 0, 1):
            for c in (-1, 0, 1):
                if (a, b, c) <= (0, 0, 0):                # lexicographically positive offsets only
                    continue
                if nonzero is not None and (a != 0) + (b != 0) + (c != 0) != nonzero:
                    continue
                cj = (((ix + a) % nc) * nc + (iy + b) % nc) * nc + (iz + c) % nc
                out.append(np.stack([cells, cj], 1))
    return torch.from_numpy(np.concatenate(out).astype(np.int32)).cuda().contiguous()


@pytest.mark.parametrize("case", ["c1", "test27cells"])
def test_symmetric_pairs_vs_oracle(pv, t27, case):
    """sph_density_pair_sym over the 13 positive offsets of every cell (each unordered pair once)
    + sph_density_self + finalize == the oracle (one distance evaluation, both sides);
    in-range pairs per kind == Code 2 hits (both sides counted)."""
    p = synth.make("c1") if case == "c1" else t27
    x, v = torch.from_numpy(p.xyzh).cuda(), torch.from_numpy(p.vm).cuda()
    dp = pv.DensityPass(p.nc, p.n)
    pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws)
    pv.sph_sort_cells(dp.grid, dp.cells, dp.ws)
    acc = pv.Out.alloc(p.n, zero=True)
    st = pv.Stats()
    pv.sph_density_self(dp.grid, dp.cells, torch.arange(p.nc ** 3, dtype=torch.int32, device="cuda"), acc, dp.ws,
                        stats=st)
    pv.sph_density_pair_sym(dp.grid, dp.cells, _half_offsets_pairs(p.nc), acc, dp.ws, stats=st)
    pv.sph_density_finalize(acc)
    dp.check()
    got = acc.to_numpy()
    ref = oracle.celllist(p.xyzh, p.vm, p.nc)
    compare(got, ref, None, f"{case} symmetric pairs")
    c, unsafe = oracle.pv_counts(p.xyzh, p.nc)
    tot = c.sum(axis=0)
    band = int(ref["band"].sum())
    cnt = st.read()
    for k in range(4):
        assert abs(cnt["hits"][k] - tot[k, 2]) <= band, k


def test_symmetric_pairs_dense_fallback(pv):
    """A cell above the symmetric kernel's staging capacity (SYM_MAXN = 512) takes the two
    one-sided global-memory sweeps; the result still equals the oracle."""
    from tests.test_gpu_parity import _dense_cell_set
    xyzh, vm, nc = _dense_cell_set(700)
    x, v = torch.from_numpy(xyzh).cuda(), torch.from_numpy(vm).cuda()
    dp = pv.DensityPass(nc, xyzh.shape[0])
    pv.sph_build_cells(dp.grid, x, v, dp.cells, dp.ws)
    pv.sph_sort_cells(dp.grid, dp.cells, dp.ws)
    acc = pv.Out.alloc(xyzh.shape[0], zero=True)
    pv.sph_density_self(dp.grid, dp.cells, torch.arange(nc ** 3, dtype=torch.int32, device="cuda"), acc, dp.ws)
    pv.sph_density_pair_sym(dp.grid, dp.cells, _half_offsets_pairs(nc), acc, dp.ws)
    pv.sph_density_finalize(acc)
    dp.check()
    compare(acc.to_numpy(), oracle.bruteforce(xyzh, vm), None, "symmetric dense fallback")
