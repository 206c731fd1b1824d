"""x-slab domain decomposition over GPUs with a one-cell ghost layer.

Rank r owns the cell planes [x_lo, x_hi) (equal or cost-balanced cuts) and
the particles inside them, in global input order.  Every step:

  1. sph_select_planes copies the owned particles of the boundary planes x_lo
     and x_hi-1, in input order (no binning pass);
  2. NCCL send/recv (torch.distributed P2P) of those planes to the left and
     right neighbours (periodic ring) -- counts first, then the particles --
     straight into the input buffer behind the owned particles;
  3. sph_build_cells over owned + ghost particles (ghost planes x_lo-1, x_hi),
     sph_sort_cells, sph_density_all.

The gather design needs no reverse exchange (ghosts are only j-sources).  With
stable in-cell order (home first, then input order) and ghosts received in the
sender's input order (= the global order), every particle sees the same
neighbours in the same order as on one GPU, so the outputs are bitwise
identical for any p (tests/test_gpu_slabs.py).

PyTorch is plumbing here: device buffers, the stream, and the process group.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import api as pv

BUILD_LAUNCHES = 8      # k_bin, 3 scan kernels, k_scatter_rec, k_stable_small/bitonic/big
SORT_LAUNCHES = 6       # k_sort_small, k_sort_mid, k_sort_warp256, k_sort_radix (medium, huge, giant)
SELECT_LAUNCHES = 5     # sph_select_planes: k_sel_count, 3 scan kernels, k_sel_write
DENSITY_LAUNCHES = 9    # k_row_home, k_v4_tiles (count), 3 scan kernels, k_v4_tiles (write), k_density_v5,
                        # k_density_dense, k_unpermute


def sym_launches(nxl: int, ny: int, nz: int, x_periodic: bool) -> int:
    """Kernels of one sph_density_all_sym call: the self-pass list and k_density_self, per
    colour phase the pair list, the warp-per-pair kernel and the CTA kernel of the deferred
    large pairs, and k_sym_merge.  Direction 0 is coloured along z, 1..3 along y, 4..12 along
    x (first nonzero component); an axis takes 3 colours when periodic and odd, else 2."""
    col = lambda n, per: 3 if per and n % 2 else 2   # noqa: E731
    phases = col(nz, True) + 3 * col(ny, True) + 9 * col(nxl, x_periodic)
    return 2 + 3 * phases + 1


def slab_bounds(nc: int, world: int, rank: int) -> tuple[int, int]:
    return rank * nc // world, (rank + 1) * nc // world


def plane_costs(xyzh: np.ndarray, nc: int, box: float = 1.0) -> np.ndarray:
    """Estimated density work per x-plane: sum over its cells of n_c x (particles in the 27
    cells around c), the naive candidate count of the cell (SURVEY.md §8(f) #2 "slab cuts by
    estimated work"; periodic neighbours)."""
    x = xyzh[:, :3].astype(np.float64) * nc / box
    ijk = np.clip(np.floor(x), 0, nc - 1).astype(np.int64)
    cnt = np.bincount((ijk[:, 0] * nc + ijk[:, 1]) * nc + ijk[:, 2], minlength=nc ** 3).reshape(nc, nc, nc)
    nb = np.zeros_like(cnt)
    for a in (-1, 0, 1):
        for b in (-1, 0, 1):
            for c in (-1, 0, 1):
                nb += np.roll(cnt, (a, b, c), axis=(0, 1, 2))
    return (cnt * nb).sum(axis=(1, 2)).astype(np.float64)


def balanced_bounds(costs: np.ndarray, world: int, min_planes: int = 2) -> list[tuple[int, int]]:
    """x-slab cuts minimising the largest per-rank estimated cost (contiguous partition of the
    planes, each slab >= `min_planes` planes: the ghost exchange needs two); dynamic programming
    over (rank, cut plane).  Equal cuts are one feasible partition, so the result is never worse."""
    nc = len(costs)
    if nc < world * min_planes:
        raise ValueError("each slab needs >= 2 cell planes")
    cum = np.concatenate([[0.0], np.cumsum(np.asarray(costs, np.float64))])
    inf = float("inf")
    best = np.full((world + 1, nc + 1), inf)       # best[r][i]: planes [0, i) on r ranks
    arg = np.zeros((world + 1, nc + 1), np.int64)
    best[0][0] = 0.0
    for r in range(1, world + 1):
        for i in range(r * min_planes, nc - (world - r) * min_planes + 1):
            for j in range((r - 1) * min_planes, i - min_planes + 1):
                v = max(best[r - 1][j], cum[i] - cum[j])
                if v < best[r][i]:
                    best[r][i], arg[r][i] = v, j
    bounds, i = [], nc
    for r in range(world, 0, -1):
        j = int(arg[r][i])
        bounds.append((j, i))
        i = j
    return bounds[::-1]


def planes_of(xyzh: np.ndarray, nc: int, box: float = 1.0) -> np.ndarray:
    """Cell x-plane of every particle: floor(x nc / box) in fp64, clamped (same rule as sph_build_cells)."""
    return np.clip(np.floor(xyzh[:, 0].astype(np.float64) * nc / box), 0, nc - 1).astype(np.int64)


@dataclass
class Slab:
    nc: int
    box: float
    gamma: float
    rank: int
    world: int
    x_lo: int
    x_hi: int
    xyzh: np.ndarray          # owned particles, global order
    vm: np.ndarray
    gid: np.ndarray           # their global indices
    n_global: int
    pset: object = None       # the full ParticleSet (single-GPU only)
    ghost_n: int = -1         # particles in the two ghost planes (known when cut from a full set)
    edge_n: int = -1          # particles in the larger of its own first and last planes
    block_max: int = -1       # the most particles of ANY rank's first or last plane (same on every rank)

    @staticmethod
    def single(p) -> "Slab":
        return Slab(p.nc, p.box, p.gamma, 0, 1, 0, p.nc, p.xyzh, p.vm, np.arange(p.n), p.n, p)

    @staticmethod
    def from_set(p, rank: int, world: int, bounds: list | None = None) -> "Slab":
        """bounds: [(x_lo, x_hi)] per rank (balanced_bounds), else equal plane counts."""
        if world == 1:
            return Slab.single(p)
        if bounds is None and p.nc // world < 2:
            raise ValueError("each slab needs >= 2 cell planes")
        lo, hi = bounds[rank] if bounds is not None else slab_bounds(p.nc, world, rank)
        pl = planes_of(p.xyzh, p.nc, p.box)
        gid = np.nonzero((pl >= lo) & (pl < hi))[0]
        per_plane = np.bincount(pl, minlength=p.nc)
        ghost_n = int(per_plane[(lo - 1) % p.nc] + per_plane[hi % p.nc])
        edge_n = int(max(per_plane[lo], per_plane[hi - 1]))
        all_b = bounds if bounds is not None else [slab_bounds(p.nc, world, r) for r in range(world)]
        block_max = int(max(max(per_plane[a], per_plane[b - 1]) for a, b in all_b))
        return Slab(p.nc, p.box, p.gamma, rank, world, lo, hi, np.ascontiguousarray(p.xyzh[gid]),
                    np.ascontiguousarray(p.vm[gid]), gid, p.n, ghost_n=ghost_n, edge_n=edge_n, block_max=block_max)

    @staticmethod
    def from_config(cfg: str, rank: int, world: int, balance: bool = False) -> "Slab":
        """balance: cut the slabs by estimated work (plane_costs) instead of equal planes."""
        import synth
        p = synth.make(cfg)
        bounds = balanced_bounds(plane_costs(p.xyzh, p.nc, p.box), world) if balance and world > 1 else None
        return Slab.from_set(p, rank, world, bounds)

    @property
    def n_own(self) -> int:
        return int(self.xyzh.shape[0])


def exchange_planes(dist, rank: int, world: int, send_lo, send_hi, recv) -> tuple[int, int]:
    """Periodic-ring ghost exchange of variable-size planes (counts first, then exact-size
    receives; the counts cross to the host).  Kept for the gloo tests and small tools; the
    runner uses exchange_fixed (no host synchronisation).

    send_lo = (xyzh, vm) of this rank's plane x_lo  -> goes to the left neighbour
    send_hi = (xyzh, vm) of this rank's plane x_hi-1 -> goes to the right neighbour
    recv    = (xyzh_buf, vm_buf): the left neighbour's plane x_hi-1 (our ghost plane
              x_lo-1) is written at [0, n_glo), the right neighbour's plane x_lo (our
              ghost plane x_hi) at [n_glo, n_glo + n_ghi).  Returns (n_glo, n_ghi).
    With p = 2 both neighbours are the same rank; NCCL matches same-peer messages in issue
    order, so every rank issues sends [to right, to left] and receives [from left, from right]."""
    left, right = (rank - 1) % world, (rank + 1) % world
    dev = send_lo[0].device
    cnt_send = torch.tensor([send_hi[0].shape[0], send_lo[0].shape[0]], dtype=torch.int64, device=dev)
    cnt_recv = torch.zeros(2, dtype=torch.int64, device=dev)
    ops = [dist.P2POp(dist.isend, cnt_send[0:1], right), dist.P2POp(dist.isend, cnt_send[1:2], left),
           dist.P2POp(dist.irecv, cnt_recv[0:1], left), dist.P2POp(dist.irecv, cnt_recv[1:2], right)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    n_glo, n_ghi = (int(v) for v in cnt_recv.tolist())
    xb, vb = recv
    if n_glo + n_ghi > xb.shape[0]:
        raise RuntimeError(f"ghost capacity {xb.shape[0]} < {n_glo + n_ghi}")
    ops = []
    if send_hi[0].shape[0]:
        ops += [dist.P2POp(dist.isend, send_hi[0], right), dist.P2POp(dist.isend, send_hi[1], right)]
    if send_lo[0].shape[0]:
        ops += [dist.P2POp(dist.isend, send_lo[0], left), dist.P2POp(dist.isend, send_lo[1], left)]
    if n_glo:
        ops += [dist.P2POp(dist.irecv, xb[0:n_glo], left), dist.P2POp(dist.irecv, vb[0:n_glo], left)]
    if n_ghi:
        ops += [dist.P2POp(dist.irecv, xb[n_glo:n_glo + n_ghi], right),
                dist.P2POp(dist.irecv, vb[n_glo:n_glo + n_ghi], right)]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return n_glo, n_ghi


def exchange_fixed(dist, rank: int, world: int, send_x, send_v, send_n, recv_x, recv_v, recv_n):
    """Fixed-capacity periodic-ring ghost exchange (no host synchronisation): every rank sends
    its two whole send buffers and their device-side counts, and receives its two ghost blocks.

    send_x, send_v: [2, cap, 4] -- block 0 = plane x_lo (to the left neighbour), block 1 =
                    plane x_hi-1 (to the right neighbour); only the first send_n[k] rows are
                    particles.  send_n: int64[2] on the device.
    recv_x, recv_v: [2, cap, 4] -- block 0 from the left neighbour (our ghost plane x_lo-1),
                    block 1 from the right (ghost plane x_hi); recv_n: int64[2] their counts.
    cap must be the same on every rank (the message sizes must match).  Same-peer messages
    match in issue order (p = 2): sends [to right, to left], receives [from left, from right].
    Returns the torch.distributed work handles (wait() orders the current stream after them)."""
    left, right = (rank - 1) % world, (rank + 1) % world
    P = dist.P2POp
    ops = [P(dist.isend, send_n[1:2], right), P(dist.isend, send_x[1], right), P(dist.isend, send_v[1], right),
           P(dist.isend, send_n[0:1], left), P(dist.isend, send_x[0], left), P(dist.isend, send_v[0], left),
           P(dist.irecv, recv_n[0:1], left), P(dist.irecv, recv_x[0], left), P(dist.irecv, recv_v[0], left),
           P(dist.irecv, recv_n[1:2], right), P(dist.irecv, recv_x[1], right), P(dist.irecv, recv_v[1], right)]
    return dist.batch_isend_irecv(ops)


def mask_dead_ghosts(recv_x, recv_v, recv_n, dead_row_x, dead_row_v, ar, dead_host=None):
    """Rows beyond the received count of each ghost block become a 'dead' particle: inside the
    box but in an OWNED plane of this rank, so sph_build_cells drops it as a ghost outside the
    ghost planes (no slot, no error).  On the GPU: the library's sph_mask_ghost_rows (counts
    read on the device, no host synchronisation; dead_host = the dead rows' host values).  The
    torch.where form serves the CPU (gloo) tests of the exchange only."""
    if recv_x.is_cuda:
        dx, dv = dead_host if dead_host is not None else (dead_row_x.tolist(), dead_row_v.tolist())
        pv.sph_mask_ghost_rows(recv_x, recv_v, recv_n, dx, dv)
        return
    for k in range(2):
        keep = (ar < recv_n[k])[:, None]
        recv_x[k].copy_(torch.where(keep, recv_x[k], dead_row_x))
        recv_v[k].copy_(torch.where(keep, recv_v[k], dead_row_v))


class SlabRunner:
    """Device buffers and one density step of one rank."""

    def __init__(self, slab: Slab, dist=None, device="cuda", ghost_capacity: int | None = None, levels=None,
                 engine: str = "gather"):
        """levels: [(nc, h_min, h_max)] level passes; the first level's nc
        must be the slab's grid, the others multiples of it (on x-slabs each level owns the
        same x range)."""
        self.slab = slab
        self.engine = engine                     # "gather" (sph_density_all) or "sym" (sph_density_all_sym)
        if engine == "sym" and levels and len(levels) > 1:
            raise ValueError("the symmetric whole pass runs on a single grid (no level passes)")
        self.dist = dist
        self.world = slab.world
        self.rank = slab.rank
        self.n_own = slab.n_own
        self.nc = slab.nc
        self.n_global = slab.n_global
        self.pset = slab.pset
        ghost = self.world > 1
        self.levels = list(levels) if levels else [(slab.nc, 0.0, 0.0)]
        split = len(self.levels) > 1
        self.grid = pv.make_grid(slab.nc, slab.box, slab.gamma, slab.x_lo, slab.x_hi, int(ghost),
                                 self.levels[0][1:] if split else None)
        if ghost:
            # ghost blocks of a FIXED capacity, equal on every rank (the P2P message sizes must
            # match): the largest boundary plane of any rank + 5 % headroom for drift + 4096
            per_plane = self.n_own / max(1, slab.x_hi - slab.x_lo)
            if ghost_capacity is not None:
                self.bcap = int(ghost_capacity)
            elif slab.block_max >= 0:
                self.bcap = int(1.05 * slab.block_max) + 4096
            else:
                self.bcap = int(1.5 * per_plane) + 4096
        else:
            self.bcap = 0
        self.cap = self.n_own + 2 * self.bcap
        self.xin = torch.zeros((max(self.cap, 1), 4), dtype=torch.float32, device=device)
        self.vin = torch.zeros((max(self.cap, 1), 4), dtype=torch.float32, device=device)
        self.cells = pv.Cells.alloc(self.grid, self.cap, device)
        self.ws = pv.alloc_workspace(self.grid, self.cells.capacity, device)
        self.out = pv.Out.alloc(self.n_own, device)
        self.n_ghost = 2 * self.bcap             # both ghost blocks always (rows past a block's count are dead)
        self.plane = self.grid.nc[1] * self.grid.nc[2]   # cells per x plane
        self.nxl = (slab.x_hi - slab.x_lo) + (2 if ghost else 0)
        dens = DENSITY_LAUNCHES if engine != "sym" else \
            sym_launches(slab.x_hi - slab.x_lo + (2 if ghost else 0), slab.nc, slab.nc, not ghost)
        self.launches_per_step = (BUILD_LAUNCHES + SORT_LAUNCHES + dens) * len(self.levels) + \
            (SELECT_LAUNCHES if ghost else 0) + (len(self.levels) if split else 0)   # k_mark_needed per level
        if ghost:
            # send buffers of the boundary planes (sph_select_planes), the received counts, and
            # the 'dead' row for unused ghost slots: inside the box in this rank's middle owned
            # plane, which every level grid's build drops as a ghost outside its ghost planes
            b = self.bcap
            self.sel_x = torch.zeros((2, b, 4), dtype=torch.float32, device=device)
            self.sel_v = torch.zeros((2, b, 4), dtype=torch.float32, device=device)
            self.sel_n = torch.zeros(2, dtype=torch.int64, device=device)
            self.recv_n = torch.zeros(2, dtype=torch.int64, device=device)
            self.ar = torch.arange(b, dtype=torch.int64, device=device)
            cl = slab.box / slab.nc
            xm = ((slab.x_lo + slab.x_hi) // 2 + 0.5) * cl
            self.dead_host = ([xm, 0.5 * slab.box, 0.5 * slab.box, 1e-6 * cl], [0.0, 0.0, 0.0, 1.0])
            self.dead_x = torch.tensor(self.dead_host[0], dtype=torch.float32, device=device)
            self.dead_v = torch.tensor(self.dead_host[1], dtype=torch.float32, device=device)
            self.comm = torch.cuda.Stream(device=device) if str(device).startswith("cuda") else None
        self.device = device
        # finer level grids (one GPU): own cells and workspace each, same outputs
        self.extra = []
        for nc, lo, hi in self.levels[1:]:
            # level k on x-slabs: planes [x_lo f, x_hi f) of the f-times finer grid, its thinner
            # ghost planes taken from the coarse ghosts (the build drops the others)
            f = nc // slab.nc
            g = pv.make_grid(nc, slab.box, slab.gamma, slab.x_lo * f, slab.x_hi * f, int(ghost), h_home=(lo, hi))
            c = pv.Cells.alloc(g, self.cap, device)
            self.extra.append((g, c, pv.alloc_workspace(g, c.capacity, device)))

    # -- data ---------------------------------------------------------------
    def upload(self) -> None:
        if self.n_own:
            self.xin[:self.n_own].copy_(torch.from_numpy(self.slab.xyzh))
            self.vin[:self.n_own].copy_(torch.from_numpy(self.slab.vm))

    # -- ghost exchange -----------------------------------------------------
    def ghost_blocks(self):
        """Views of the two ghost blocks behind the owned particles: [2, bcap, 4]."""
        a, b = self.n_own, self.n_own + 2 * self.bcap
        return self.xin[a:b].view(2, self.bcap, 4), self.vin[a:b].view(2, self.bcap, 4)

    def select(self) -> None:
        """The owned particles of planes x_lo and x_hi-1 in input order into the send buffers
        (sph_select_planes: no binning pass); the counts stay on the device."""
        pv.sph_select_planes(self.grid, self.xin, self.vin, self.n_own, self.sel_x, self.sel_v, self.sel_n, self.ws)

    def boundary_planes(self):
        """The selected planes as ((xyzh, vm), (xyzh, vm)) views (host sync for the counts:
        tests and tools only; the step uses the fixed-capacity exchange)."""
        self.select()
        n_lo, n_hi = self.sel_n.tolist()
        return (self.sel_x[0, :n_lo], self.sel_v[0, :n_lo]), (self.sel_x[1, :n_hi], self.sel_v[1, :n_hi])

    def exchange(self) -> None:
        """Ghost exchange with no host synchronisation: select on the compute stream, the NCCL
        P2P transfer of the fixed-capacity blocks and counts on the comm stream, then the compute
        stream waits for it and marks the unused ghost rows dead."""
        self.select()
        rx, rv = self.ghost_blocks()
        cs = torch.cuda.current_stream()
        if self.comm is not None:
            self.comm.wait_stream(cs)
            with torch.cuda.stream(self.comm):
                for w in exchange_fixed(self.dist, self.rank, self.world, self.sel_x, self.sel_v, self.sel_n,
                                        rx, rv, self.recv_n):
                    w.wait()
            cs.wait_stream(self.comm)
        else:
            for w in exchange_fixed(self.dist, self.rank, self.world, self.sel_x, self.sel_v, self.sel_n,
                                    rx, rv, self.recv_n):
                w.wait()
        mask_dead_ghosts(rx, rv, self.recv_n, self.dead_x, self.dead_v, self.ar, self.dead_host)

    # -- one step -----------------------------------------------------------
    def step(self, stats=None, events=None) -> None:
        s = torch.cuda.current_stream()
        rec = (lambda k: events[k].record(s)) if events else (lambda k: None)
        rec(0)
        if self.world > 1:
            self.exchange()
        rec(1)
        self.compute(stats=stats, rec=rec)

    def compute(self, stats=None, rec=None) -> None:
        """Build, sort and density of every level grid on the current inputs (owned particles
        and the n_ghost ghosts behind them)."""
        rec = rec or (lambda k: None)
        if not self.extra:
            # one grid: build and sort in one call (the small cells' lists come out of the build's
            # placement pass); the "build" stage then holds both, "sort" only the larger cells' tiers
            pv.sph_build_sort_cells(self.grid, self.xin, self.vin, self.cells, self.ws, n_own=self.n_own,
                                    n_ghost=self.n_ghost)
            rec(2)
            rec(3)
            dens = pv.sph_density_all_sym if self.engine == "sym" else pv.sph_density_all
            dens(self.grid, self.cells, self.out, self.ws, stats=stats)
            rec(4)
            return
        pv.sph_build_cells(self.grid, self.xin, self.vin, self.cells, self.ws, n_own=self.n_own,
                           n_ghost=self.n_ghost)
        for g, c, ws in self.extra:
            pv.sph_build_cells(g, self.xin, self.vin, c, ws, n_own=self.n_own, n_ghost=self.n_ghost)
        rec(2)
        pv.sph_sort_cells(self.grid, self.cells, self.ws)
        for g, c, ws in self.extra:
            pv.sph_sort_cells(g, c, ws)
        rec(3)
        dens = pv.sph_density_all_sym if self.engine == "sym" else pv.sph_density_all
        dens(self.grid, self.cells, self.out, self.ws, stats=stats)
        for g, c, ws in self.extra:
            pv.sph_density_all(g, c, self.out, ws, stats=stats)
        rec(4)

    def check(self) -> None:
        """Raise on any error of the last step (one host sync): the workspaces' status words and
        a boundary plane larger than the fixed ghost block (sph_select_planes' overflow, whose
        status bit the next build would clear)."""
        if self.world > 1:
            n = self.sel_n.tolist()
            if max(n) > self.bcap:
                raise RuntimeError(f"boundary plane of {max(n)} particles exceeds the ghost block capacity {self.bcap}")
        pv.check_status(self.ws)
        for _, _, ws in self.extra:
            pv.check_status(ws)

    # -- end to end through host buffers -----------------------------------
    def e2e_time(self, steps: int = 3, warmup: int = 1):
        """ms per step through host buffers: every step copies its owned inputs from pinned
        host memory (H2D) and all its outputs back (D2H) inside the timed region.  Steps are
        pipelined over three streams with double-buffered device inputs and outputs: the H2D
        of step k+1 and the D2H of step k-1 run on the copy engines while step k computes,
        as a serving loop would.  Returns (ms, h2d_bytes, d2h_bytes)."""
        n = self.n_own
        hx = torch.from_numpy(self.slab.xyzh).pin_memory()
        hv = torch.from_numpy(self.slab.vm).pin_memory()
        names = ["rho", "rho_dh", "wcount", "wcount_dh", "div_v", "curl_v", "nngb"]
        bufs = [(self.xin, self.vin, self.out),
                (torch.zeros_like(self.xin), torch.zeros_like(self.vin), pv.Out.alloc(self.n_own, self.device))]
        host = [[torch.empty(getattr(o, k).shape, dtype=getattr(o, k).dtype, pin_memory=True) for k in names]
                for _, _, o in bufs]
        s_c = torch.cuda.current_stream()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()                      # noqa: E731
        in_ready, c_done, out_free = [ev(), ev()], [ev(), ev()], [ev(), ev()]
        for b in range(2):                                  # both buffer sets free at the start
            c_done[b].record(s_c)
            out_free[b].record(s_c)
        saved = (self.xin, self.vin, self.out)

        def one(k):
            b = k % 2
            xin, vin, out = bufs[b]
            with torch.cuda.stream(s_in):                   # inputs of step k (buffer free once step k-2 ran)
                s_in.wait_event(c_done[b])
                xin[:n].copy_(hx, non_blocking=True)
                vin[:n].copy_(hv, non_blocking=True)
                in_ready[b].record(s_in)
            s_c.wait_event(in_ready[b])
            s_c.wait_event(out_free[b])                     # outputs of step k-2 copied out
            self.xin, self.vin, self.out = xin, vin, out
            self.step()
            c_done[b].record(s_c)
            with torch.cuda.stream(s_out):                  # results of step k
                s_out.wait_event(c_done[b])
                for h, key in zip(host[b], names):
                    h.copy_(getattr(out, key), non_blocking=True)
                out_free[b].record(s_out)

        try:
            for k in range(warmup):
                one(k)
            torch.cuda.synchronize()
            if self.dist:
                self.dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s_c)
            for k in range(warmup, warmup + steps):
                one(k)
            s_c.wait_event(out_free[(warmup + steps - 1) % 2])   # the last results are on the host
            s_c.wait_event(out_free[(warmup + steps - 2) % 2])
            e1.record(s_c)
            torch.cuda.synchronize()
        finally:
            self.xin, self.vin, self.out = saved
        self.e2e_host = dict(zip(names, host[(warmup + steps - 1) % 2]))   # the last step's results
        h2d = 2 * n * 16
        d2h = sum(getattr(self.out, k).numel() * getattr(self.out, k).element_size() for k in names)
        return e0.elapsed_time(e1) / steps, h2d, d2h


class FakeRanks:
    """p slab ranks emulated in ONE process on one GPU, the ghost exchange done with
    device copies instead of NCCL (a test harness for the slab logic; nothing waits
    on another rank, every launch is ordered on one stream)."""

    def __init__(self, p, world: int, device="cuda", balance: bool = False, levels=None):
        self.world = world
        bounds = balanced_bounds(plane_costs(p.xyzh, p.nc, p.box), world) if balance else None
        self.bounds = bounds
        self.runners = [SlabRunner(Slab.from_set(p, r, world, bounds), dist=None, device=device, levels=levels)
                        for r in range(world)]
        for r in self.runners:
            r.upload()
        self.n_global = p.n

    def step(self) -> None:
        """The fixed-capacity exchange emulated with device copies: every runner's ghost block 0
        receives its left neighbour's block 1 (plane x_hi-1) and block 1 its right neighbour's
        block 0, counts included; then the same dead-row masking as the NCCL path."""
        for r in self.runners:
            r.select()
        W = self.world
        for k, r in enumerate(self.runners):
            rx, rv = r.ghost_blocks()
            left, right = self.runners[(k - 1) % W], self.runners[(k + 1) % W]
            assert left.bcap == r.bcap == right.bcap
            rx[0].copy_(left.sel_x[1])
            rv[0].copy_(left.sel_v[1])
            rx[1].copy_(right.sel_x[0])
            rv[1].copy_(right.sel_v[0])
            r.recv_n[0].copy_(left.sel_n[1])
            r.recv_n[1].copy_(right.sel_n[0])
            mask_dead_ghosts(rx, rv, r.recv_n, r.dead_x, r.dead_v, r.ar, r.dead_host)
        for r in self.runners:
            r.compute()
        for r in self.runners:
            r.check()

    def gather(self) -> dict:
        res = {}
        for r in self.runners:
            o = r.out.to_numpy()
            for k, v in o.items():
                if k not in res:
                    res[k] = np.zeros(self.n_global, v.dtype)
                res[k][r.slab.gid] = v
        return res


# ---------------------------------------------------------------------------
# list reuse on x-slabs: drift, stale cells, rebuild with migration
# ---------------------------------------------------------------------------
def exchange_arrays(dist, rank: int, world: int, send_lo: list, send_hi: list, recv_lo: list, recv_hi: list,
                    n_lo: int, n_hi: int, dev) -> tuple[int, int]:
    """Variable-size periodic-ring exchange of several arrays per direction (migration at a
    rebuild; host-synchronised counts).  send_lo goes to the left neighbour, send_hi to the
    right; recv_lo[k][:n] receives from the left, recv_hi from the right.  Same-peer issue
    order as exchange_planes.  Returns the received counts."""
    left, right = (rank - 1) % world, (rank + 1) % world
    cnt_send = torch.tensor([n_hi, n_lo], dtype=torch.int64, device=dev)
    cnt_recv = torch.zeros(2, dtype=torch.int64, device=dev)
    ops = [dist.P2POp(dist.isend, cnt_send[0:1], right), dist.P2POp(dist.isend, cnt_send[1:2], left),
           dist.P2POp(dist.irecv, cnt_recv[0:1], left), dist.P2POp(dist.irecv, cnt_recv[1:2], right)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    r_lo, r_hi = (int(v) for v in cnt_recv.tolist())
    if r_lo > recv_lo[0].shape[0] or r_hi > recv_hi[0].shape[0]:
        raise RuntimeError(f"migration capacity {recv_lo[0].shape[0]} < {max(r_lo, r_hi)}")
    ops = []
    if n_hi:
        ops += [dist.P2POp(dist.isend, a[:n_hi], right) for a in send_hi]
    if n_lo:
        ops += [dist.P2POp(dist.isend, a[:n_lo], left) for a in send_lo]
    if r_lo:
        ops += [dist.P2POp(dist.irecv, a[:r_lo], left) for a in recv_lo]
    if r_hi:
        ops += [dist.P2POp(dist.irecv, a[:r_hi], right) for a in recv_hi]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return r_lo, r_hi


def split_migrants(x: torch.Tensor, nc: int, box: float, x_lo: int, x_hi: int):
    """Masks of the owned particles (wrapped positions) whose x plane -- the binning rule of
    sph_build_cells -- is the left neighbour's last plane (x_lo - 1) or the right neighbour's
    first (x_hi), and of those that stay.  A particle moves at most one plane between rebuilds
    (displacement < skin < C_l / 2).  The rule as host logic (CPU tests, and the reference the
    GPU test holds sph_partition_migrants to); the product path calls the library."""
    pl = torch.clamp(torch.floor(x[:, 0].double() * nc / box), 0, nc - 1).long()
    lo = pl == (x_lo - 1) % nc
    hi = (pl == x_hi % nc) & ~lo
    return lo, hi, ~(lo | hi)


class SlabReuse(SlabRunner):
    """List reuse on x-slabs ("re-sort/re-bin (and migrate between slabs)
    only past a threshold").  Each rank drifts all its stored particles -- owned ones and
    the ghost copies, with identical fp32 increments -- and runs the density pass on the stale
    cells; before a drift could take a displacement past the skin every rank rebuilds at the same
    step (the bound uses the GLOBAL max |v|): positions gathered back to input order and wrapped
    (sph_gather_positions), particles that crossed a slab face migrate to the neighbour, the
    owned set is re-merged in global-id order (so in-cell orders, and the outputs, stay bitwise
    those of one GPU), the ghost planes are exchanged again and the cells rebuilt.

    transport: "dist" (torch.distributed P2P) or a FakeReuse coordinator (device copies)."""

    def __init__(self, slab: Slab, skin: float, vmax_global: float, dist=None, device="cuda", headroom=0.15):
        self.own_cap = int((1 + headroom) * slab.n_own) + 4096
        n0 = slab.n_own
        # SlabRunner sizes everything from n_own: build it for the headroom capacity, then shrink
        slab_cap = Slab(slab.nc, slab.box, slab.gamma, slab.rank, slab.world, slab.x_lo, slab.x_hi,
                        np.zeros((self.own_cap, 4), np.float32), np.zeros((self.own_cap, 4), np.float32),
                        np.zeros(self.own_cap, np.int64), slab.n_global, None, slab.ghost_n, slab.edge_n,
                        int(1.1 * slab.block_max) if slab.block_max >= 0 else -1)
        super().__init__(slab_cap, dist=dist, device=device)
        self.slab = slab
        self.n_own = n0
        self.skin = float(skin)
        self.grid = pv.make_grid(slab.nc, slab.box, slab.gamma, slab.x_lo, slab.x_hi, int(self.world > 1), skin=skin)
        self.vmax = float(vmax_global)
        self.gid = torch.zeros(self.own_cap, dtype=torch.int64, device=device)
        self.bound = 0.0
        self.rebuilds = 0
        mcap = int(0.1 * self.own_cap) + 4096
        self.mig = [[torch.zeros((mcap, 4), dtype=torch.float32, device=device),
                     torch.zeros((mcap, 4), dtype=torch.float32, device=device),
                     torch.zeros(mcap, dtype=torch.int64, device=device)] for _ in range(4)]   # send lo/hi, recv lo/hi
        self.keep = [torch.zeros((self.own_cap, 4), dtype=torch.float32, device=device),
                     torch.zeros((self.own_cap, 4), dtype=torch.float32, device=device),
                     torch.zeros(self.own_cap, dtype=torch.int64, device=device)]             # the staying particles
        self.mig_n = torch.zeros(3, dtype=torch.int64, device=device)
        self.out_view = None

    def upload(self) -> None:
        n = self.n_own
        self.xin[:n].copy_(torch.from_numpy(self.slab.xyzh))
        self.vin[:n].copy_(torch.from_numpy(self.slab.vm))
        self.gid[:n].copy_(torch.from_numpy(np.asarray(self.slab.gid, np.int64)))
        self.out = pv.Out.alloc(n, self.device)

    def outputs(self) -> "pv.Out":
        """The current owned particles' outputs (a view with n_out = n_own; curl rows keep the
        allocation stride, so the density call gets the full-size struct)."""
        return self.out

    def _build(self):
        pv.sph_build_cells(self.grid, self.xin, self.vin, self.cells, self.ws, n_own=self.n_own,
                           n_ghost=self.n_ghost)
        pv.sph_sort_cells(self.grid, self.cells, self.ws)
        self.bound = 0.0

    def step_bound(self, dt: float) -> float:
        return self.vmax * abs(dt) * (1.0 + 2.0 ** -20) + 3.0 ** 0.5 * 2.0 ** -24 * (self.slab.box + self.skin) * 1.01

    # -- rebuild pieces (the transport supplies the exchanges) --------------------------------
    def gather_owned(self) -> None:
        """Current positions of the owned particles back to their (input = gid) order, wrapped."""
        pv.sph_gather_positions(self.grid, self.cells, self.xin, self.n_own)

    def pack_migrants(self):
        """Split the owned set (sph_partition_migrants, stable): migrants to the left / right
        into the send buffers, the rest into `keep`; returns (n_lo, n_hi, n_keep) -- one host
        synchronisation per rebuild, for the message sizes."""
        pv.sph_partition_migrants(self.grid, self.n_own, self.xin, self.vin, self.gid, self.mig[0], self.mig[1],
                                  self.keep, self.mig_n, self.ws)
        n_lo, n_hi, n_keep = (int(c) for c in self.mig_n.tolist())
        if n_lo > self.mig[0][0].shape[0] or n_hi > self.mig[1][0].shape[0]:
            raise RuntimeError(f"migration buffer {self.mig[0][0].shape[0]} < {max(n_lo, n_hi)}")
        return n_lo, n_hi, n_keep

    def merge_owned(self, n_keep: int, r_lo: int, r_hi: int) -> None:
        """The kept particles plus the received migrants, in ascending global id
        (sph_merge_by_id: all three lists are ascending already)."""
        m = n_keep + r_lo + r_hi
        if m > self.own_cap:
            raise RuntimeError(f"owned capacity {self.own_cap} < {m}")
        pv.sph_merge_by_id([(self.keep[0], self.keep[1], self.keep[2], n_keep),
                            (self.mig[2][0], self.mig[2][1], self.mig[2][2], r_lo),
                            (self.mig[3][0], self.mig[3][1], self.mig[3][2], r_hi)],
                           self.xin, self.vin, self.gid)
        self.n_own = m
        self.out = pv.Out.alloc(m, self.device)      # outputs of the new owned set

    def rebuild_local(self):
        """After the (ghost) exchange: dead rows past the counts, then build and sort."""
        self._build()
        self.rebuilds += 1


class ReuseTransport:
    """Drives SlabReuse ranks through their exchanges: torch.distributed P2P for one rank per
    process (`dist`), or all ranks in one process with device copies (fake ranks, tests)."""

    def __init__(self, runners: list, dist=None):
        self.r = runners
        self.dist = dist

    def _ghosts(self):
        if self.dist is not None:
            for rr in self.r:
                rr.exchange()
            return
        W = len(self.r)
        for rr in self.r:
            rr.select()
        for k, rr in enumerate(self.r):
            rx, rv = rr.ghost_blocks()
            left, right = self.r[(k - 1) % W], self.r[(k + 1) % W]
            rx[0].copy_(left.sel_x[1])
            rv[0].copy_(left.sel_v[1])
            rx[1].copy_(right.sel_x[0])
            rv[1].copy_(right.sel_v[0])
            rr.recv_n[0].copy_(left.sel_n[1])
            rr.recv_n[1].copy_(right.sel_n[0])
            mask_dead_ghosts(rx, rv, rr.recv_n, rr.dead_x, rr.dead_v, rr.ar, rr.dead_host)

    def _migrate(self):
        packs = [rr.pack_migrants() for rr in self.r]
        if self.dist is not None:
            for rr, (n_lo, n_hi, keep) in zip(self.r, packs):
                r_lo, r_hi = exchange_arrays(self.dist, rr.rank, rr.world, rr.mig[0], rr.mig[1], rr.mig[2],
                                             rr.mig[3], n_lo, n_hi, rr.xin.device)
                rr.merge_owned(keep, r_lo, r_hi)
            return
        W = len(self.r)
        recv = []
        for k, rr in enumerate(self.r):
            left, right = self.r[(k - 1) % W], self.r[(k + 1) % W]
            r_lo = packs[(k - 1) % W][1]            # the left neighbour's particles moving right
            r_hi = packs[(k + 1) % W][0]            # the right neighbour's moving left
            for a in range(3):
                rr.mig[2][a][:r_lo].copy_(left.mig[1][a][:r_lo])
                rr.mig[3][a][:r_hi].copy_(right.mig[0][a][:r_hi])
            recv.append((r_lo, r_hi))
        for rr, (n_lo, n_hi, keep), (r_lo, r_hi) in zip(self.r, packs, recv):
            rr.merge_owned(keep, r_lo, r_hi)

    def start(self):
        for rr in self.r:
            rr.upload()
        self._ghosts()
        for rr in self.r:
            rr._build()

    def step(self, dt: float, stats=None):
        """One reuse step on every rank: rebuild (gather, migrate, ghosts, build, sort) first if
        the displacement bound would pass the skin, then drift + density."""
        rr0 = self.r[0]
        inc = rr0.step_bound(dt)
        if inc > rr0.skin:
            raise ValueError("one drift exceeds the skin")
        if rr0.bound + inc > rr0.skin:
            for rr in self.r:
                rr.gather_owned()
            self._migrate()
            self._ghosts()
            for rr in self.r:
                rr.rebuild_local()
        for rr in self.r:
            pv.sph_drift(rr.grid, rr.cells, dt)
            rr.bound += inc
            pv.sph_density_all(rr.grid, rr.cells, rr.out, rr.ws, stats=stats)

    def gather(self, n_global: int) -> dict:
        res = {}
        for rr in self.r:
            o = rr.out.to_numpy()
            g = rr.gid[:rr.n_own].cpu().numpy()
            for k, v in o.items():
                if k not in res:
                    res[k] = np.zeros(n_global, v.dtype)
                res[k][g] = v
        return res
