"""Host-side x-slab logic on CPU: partition and the ghost exchange over gloo (world sizes 2-4)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def test_slab_partition_covers_every_particle_once():
    from paper_1804_06231_b200.slabs import Slab, planes_of, slab_bounds
    p = synth.make("c2")
    for world in (2, 3, 4, 6):
        seen = np.zeros(p.n, np.int64)
        for r in range(world):
            s = Slab.from_set(p, r, world)
            lo, hi = slab_bounds(p.nc, world, r)
            assert (s.x_lo, s.x_hi) == (lo, hi)
            pl = planes_of(s.xyzh, p.nc)
            assert np.all((pl >= lo) & (pl < hi))
            assert np.all(np.diff(s.gid) > 0)             # global order preserved
            seen[s.gid] += 1
        assert np.all(seen == 1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, sizes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1804_06231_b200.slabs import exchange_planes

    def plane(r, which):
        n = sizes[r][which]
        x = torch.zeros((n, 4), dtype=torch.float32)
        x[:, 0] = r
        x[:, 1] = which
        x[:, 2] = torch.arange(n, dtype=torch.float32)
        return x, x + 1000.0

    lo, hi = plane(rank, 0), plane(rank, 1)
    xb = torch.full((64, 4), -1.0)
    vb = torch.full((64, 4), -1.0)
    n_glo, n_ghi = exchange_planes(dist, rank, world, lo, hi, (xb, vb))
    left, right = (rank - 1) % world, (rank + 1) % world
    exp_lo, exp_hi = plane(left, 1), plane(right, 0)
    ok = (n_glo == exp_lo[0].shape[0] and n_ghi == exp_hi[0].shape[0] and
          torch.equal(xb[:n_glo], exp_lo[0]) and torch.equal(vb[:n_glo], exp_lo[1]) and
          torch.equal(xb[n_glo:n_glo + n_ghi], exp_hi[0]) and torch.equal(vb[n_glo:n_glo + n_ghi], exp_hi[1]) and
          bool((xb[n_glo + n_ghi:] == -1).all()))
    q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,sizes", [
    (2, [(3, 5), (4, 2)]),
    (2, [(0, 5), (4, 0)]),          # empty planes on both sides
    (3, [(1, 2), (3, 4), (5, 6)]),
    (4, [(2, 0), (0, 3), (7, 1), (1, 1)]),
])
def test_ghost_exchange_gloo(world, sizes):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sizes, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def test_balanced_bounds_cover_and_balance():
    """Cost-balanced x-slab cuts: contiguous cover of all planes, >= 2
    planes per slab, and on clustered data a smaller max/mean cost than equal cuts."""
    import numpy as np
    import synth
    from paper_1804_06231_b200.slabs import balanced_bounds, plane_costs, slab_bounds
    p = synth.clustered_set("cl64k", seed=7, n=65536, nc=13, n_spheres=16)
    costs = plane_costs(p.xyzh, p.nc)
    assert costs.shape == (13,) and np.all(costs >= 0)
    for world in (2, 3, 4, 6):
        b = balanced_bounds(costs, world)
        assert b[0][0] == 0 and b[-1][1] == 13 and all(b[k][1] == b[k + 1][0] for k in range(world - 1))
        assert all(hi - lo >= 2 for lo, hi in b)
        imb = max(costs[lo:hi].sum() for lo, hi in b) / (costs.sum() / world)
        eq = [slab_bounds(13, world, r) for r in range(world)]
        imb_eq = max(costs[lo:hi].sum() for lo, hi in eq) / (costs.sum() / world)
        assert imb <= imb_eq + 1e-9, (world, imb, imb_eq)


def test_plane_costs_uniform_lattice():
    """Closed form: one particle per cell of an nc^3 lattice -> every cell costs 1 x 27."""
    import numpy as np
    from paper_1804_06231_b200.slabs import plane_costs
    nc = 5
    g = (np.arange(nc) + 0.5) / nc
    x, y, z = np.meshgrid(g, g, g, indexing="ij")
    xyzh = np.zeros((nc ** 3, 4), np.float32)
    xyzh[:, 0], xyzh[:, 1], xyzh[:, 2] = x.ravel(), y.ravel(), z.ravel()
    assert np.array_equal(plane_costs(xyzh, nc), np.full(nc, 27.0 * nc * nc))


def test_slab_ghost_counts_exact():
    """A slab cut from the full set records how many particles its two ghost planes hold (the
    ghost buffer is sized from it: uneven, cost-balanced cuts can land on dense planes)."""
    import numpy as np
    import synth
    from paper_1804_06231_b200.slabs import Slab, balanced_bounds, plane_costs, planes_of
    p = synth.clustered_set("cl64k", seed=7, n=65536, nc=13, n_spheres=16)
    b = balanced_bounds(plane_costs(p.xyzh, p.nc), 3)
    pl = planes_of(p.xyzh, p.nc)
    for r in range(3):
        s = Slab.from_set(p, r, 3, b)
        lo, hi = b[r]
        assert s.ghost_n == int(((pl == (lo - 1) % 13) | (pl == hi % 13)).sum())
        assert s.n_own == int(((pl >= lo) & (pl < hi)).sum())


def _worker_fixed(rank, world, port, sizes, cap, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1804_06231_b200.slabs import exchange_fixed, mask_dead_ghosts

    def block(r, which):
        x = torch.full((cap, 4), -5.0)
        n = sizes[r][which]
        x[:n, 0] = r
        x[:n, 1] = which
        x[:n, 2] = torch.arange(n, dtype=torch.float32)
        return x

    send_x = torch.stack([block(rank, 0), block(rank, 1)])
    send_v = send_x + 1000.0
    send_n = torch.tensor(sizes[rank], dtype=torch.int64)
    recv_x = torch.zeros((2, cap, 4))
    recv_v = torch.zeros((2, cap, 4))
    recv_n = torch.zeros(2, dtype=torch.int64)
    for w in exchange_fixed(dist, rank, world, send_x, send_v, send_n, recv_x, recv_v, recv_n):
        w.wait()
    dead_x = torch.tensor([7.0, 8.0, 9.0, 0.5])
    dead_v = torch.tensor([0.0, 0.0, 0.0, 1.0])
    mask_dead_ghosts(recv_x, recv_v, recv_n, dead_x, dead_v, torch.arange(cap))
    left, right = (rank - 1) % world, (rank + 1) % world
    ok = recv_n.tolist() == [sizes[left][1], sizes[right][0]]
    for k, (src, which) in enumerate(((left, 1), (right, 0))):
        n = sizes[src][which]
        exp = block(src, which)
        ok = ok and torch.equal(recv_x[k, :n], exp[:n]) and torch.equal(recv_v[k, :n], exp[:n] + 1000.0)
        ok = ok and bool((recv_x[k, n:] == dead_x).all()) and bool((recv_v[k, n:] == dead_v).all())
    q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,sizes", [
    (2, [(3, 5), (4, 2)]),
    (2, [(0, 8), (8, 0)]),          # an empty and a full block
    (3, [(1, 2), (3, 4), (5, 6)]),
    (4, [(2, 0), (0, 3), (7, 1), (1, 1)]),
])
def test_fixed_capacity_exchange_gloo(world, sizes):
    """The runner's exchange (no host sync): whole fixed-capacity blocks and device-side counts
    over P2P, rows past each received count replaced by the dead row (dropped by the build)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_fixed, args=(r, world, port, sizes, 8, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def test_block_capacity_same_on_every_rank():
    """The ghost blocks' capacity comes from the largest boundary plane of ANY rank, so every rank
    sizes its P2P messages identically (equal and cost-balanced cuts)."""
    from paper_1804_06231_b200.slabs import Slab, balanced_bounds, plane_costs, planes_of
    p = synth.clustered_set("cl64k", seed=7, n=65536, nc=13, n_spheres=16)
    pl = planes_of(p.xyzh, p.nc)
    for bounds in (None, balanced_bounds(plane_costs(p.xyzh, p.nc), 3)):
        slabs = [Slab.from_set(p, r, 3, bounds) for r in range(3)]
        assert len({s.block_max for s in slabs}) == 1
        assert all(s.block_max >= max((pl == s.x_lo).sum(), (pl == s.x_hi - 1).sum()) for s in slabs)


def _worker_mig(rank, world, port, sizes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1804_06231_b200.slabs import exchange_arrays
    cap = 16

    def arrs(r, which):
        n = sizes[r][which]
        x = torch.zeros((cap, 4))
        x[:n, 0] = r
        x[:n, 1] = which
        x[:n, 2] = torch.arange(n, dtype=torch.float32)
        g = torch.zeros(cap, dtype=torch.int64)
        g[:n] = 1000 * r + 100 * which + torch.arange(n)
        return [x, x + 7.0, g]

    s_lo, s_hi = arrs(rank, 0), arrs(rank, 1)
    r_lo = [torch.zeros((cap, 4)), torch.zeros((cap, 4)), torch.zeros(cap, dtype=torch.int64)]
    r_hi = [torch.zeros((cap, 4)), torch.zeros((cap, 4)), torch.zeros(cap, dtype=torch.int64)]
    n_rlo, n_rhi = exchange_arrays(dist, rank, world, s_lo, s_hi, r_lo, r_hi, sizes[rank][0], sizes[rank][1],
                                   torch.device("cpu"))
    left, right = (rank - 1) % world, (rank + 1) % world
    ok = (n_rlo, n_rhi) == (sizes[left][1], sizes[right][0])
    for got, (src, which), n in ((r_lo, (left, 1), n_rlo), (r_hi, (right, 0), n_rhi)):
        exp = arrs(src, which)
        ok = ok and all(torch.equal(a[:n], b[:n]) for a, b in zip(got, exp))
    q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,sizes", [(2, [(3, 5), (4, 0)]), (3, [(1, 2), (0, 4), (5, 6)])])
def test_migration_exchange_gloo(world, sizes):
    """Migration at a reuse rebuild (slabs.SlabReuse): variable-size exchange of positions,
    (v, m) and global ids with both neighbours."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_mig, args=(r, world, port, sizes, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def test_split_migrants_rule():
    """A particle leaves its slab iff its x plane (the binning rule) is the neighbour's boundary
    plane; periodic wrap for the first and last slabs."""
    from paper_1804_06231_b200.slabs import split_migrants
    nc = 10
    x = torch.tensor([[0.05, 0, 0, 0], [0.15, 0, 0, 0], [0.35, 0, 0, 0], [0.45, 0, 0, 0], [0.95, 0, 0, 0]])
    lo, hi, keep = split_migrants(x, nc, 1.0, 2, 4)        # slab planes [2, 4)
    assert lo.tolist() == [False, True, False, False, False]
    assert hi.tolist() == [False, False, False, True, False]
    lo, hi, keep = split_migrants(x, nc, 1.0, 0, 4)        # first slab: the left neighbour owns plane 9
    assert lo.tolist() == [False, False, False, False, True] and hi.tolist()[3]


def test_sym_launch_count_matches_the_colour_phases():
    """slabs.sym_launches (the bench's gpu_launches for --engine sym) counts the kernels of one
    sph_density_all_sym call: 2 (self list + self kernel) + 3 per colour phase + 1 merge, with
    2 or 3 colours on each direction's first nonzero axis (13 directions: 1 along z, 3 along y,
    9 along x) -- the same rule as k_sym_phase_pairs / sym_dir_colours in density_pair.cuh."""
    from paper_1804_06231_b200 import slabs
    col = lambda n, per: 3 if per and n % 2 else 2      # noqa: E731
    for nx, ny, nz, per in [(47, 47, 47, True), (8, 8, 8, True), (7, 5, 6, True), (25, 184, 184, False)]:
        phases = col(nz, True) + 3 * col(ny, True) + 9 * col(nx, per)
        assert slabs.sym_launches(nx, ny, nz, per) == 3 + 3 * phases
    assert slabs.sym_launches(47, 47, 47, True) == 3 + 3 * 39
