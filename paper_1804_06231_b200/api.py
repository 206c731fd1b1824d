"""Thin Python binding of libpvsph.so with the C ABI's names.

Argument marshalling only: torch supplies device memory and the stream;
every step of the density path runs in the library's CUDA kernels.  There
is no CPU fallback: without the built library or a GPU the calls raise.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import SphCells, SphGrid, SphOut, SphStats

GAMMA = 1.825742


class SphError(RuntimeError):
    def __init__(self, code: int, where: str):
        lib = _lib.load()
        msg = lib.sph_strerror(code).decode()
        super().__init__(f"{where}: {_lib.ERROR_NAMES.get(code, code)} ({msg})")
        self.code = code


def _check(code: int, where: str) -> None:
    if code != _lib.SPH_OK:
        raise SphError(code, where)


def _stream(stream=None) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def make_grid(nc, box=1.0, gamma=GAMMA, x_lo=0, x_hi=None, ghost_x=0, h_home=None, skin=0.0) -> SphGrid:
    """h_home = (h_min, h_max): level pass, only particles with h_min < h <= h_max are home.
    skin: list reuse, the largest displacement allowed between rebuilds (include/sph.h)."""
    if isinstance(nc, int):
        nc = (nc, nc, nc)
    if isinstance(box, (int, float)):
        box = (float(box),) * 3
    g = SphGrid()
    for k in range(3):
        g.nc[k] = int(nc[k])
        g.box[k] = float(box[k])
    g.x_lo = int(x_lo)
    g.x_hi = int(nc[0] if x_hi is None else x_hi)
    g.ghost_x = int(ghost_x)
    g.gamma = float(gamma)
    if h_home is not None:
        g.h_home_min, g.h_home_max = float(h_home[0]), float(h_home[1])
    g.skin = float(skin)
    return g


def ncell(grid: SphGrid) -> int:
    n = _lib.load().sph_ncell(ctypes.byref(grid))
    if n < 0:
        raise SphError(_lib.SPH_EINVAL, "sph_ncell")
    return int(n)


def workspace_bytes(grid: SphGrid, n_total: int) -> int:
    b = _lib.load().sph_workspace_bytes(ctypes.byref(grid), int(n_total))
    if b == 0:
        raise SphError(_lib.SPH_EINVAL, "sph_workspace_bytes")
    return int(b)


@dataclass
class Cells:
    """Device storage of sph_cells (owned by torch)."""
    capacity: int
    cell_start: torch.Tensor
    xyzh: torch.Tensor
    vm: torch.Tensor
    perm: torch.Tensor
    cell_hmax: torch.Tensor
    order: torch.Tensor         # (13, capacity) int16 storage of the uint16 sorted lists (include/sph.h)
    slot_cell: torch.Tensor     # (capacity,) int32
    cell_nhome: torch.Tensor    # (ncell,) int32: home particles per cell
    disp: torch.Tensor          # (capacity,) float32: displacement bound since the build (list reuse)
    cell_dx: torch.Tensor       # (ncell,) float32: per-cell max_dx
    n: int = 0

    @staticmethod
    def alloc(grid: SphGrid, capacity: int, device="cuda") -> "Cells":
        nce = ncell(grid)
        cap = max(int(capacity), 1)
        return Cells(cap, torch.empty(nce + 1, dtype=torch.int32, device=device),
                     torch.empty((cap, 4), dtype=torch.float32, device=device),
                     torch.empty((cap, 4), dtype=torch.float32, device=device),
                     torch.empty(cap, dtype=torch.int32, device=device),
                     torch.empty(nce, dtype=torch.float32, device=device),
                     torch.empty((_lib.SPH_NDIR, cap), dtype=torch.int16, device=device),
                     torch.empty(cap, dtype=torch.int32, device=device),
                     torch.empty(nce, dtype=torch.int32, device=device),
                     torch.zeros(cap, dtype=torch.float32, device=device),
                     torch.zeros(nce, dtype=torch.float32, device=device))

    def struct(self) -> SphCells:
        s = SphCells()
        s.capacity = self.capacity
        s.n = self.n
        s.cell_start, s.xyzh, s.vm = self.cell_start.data_ptr(), self.xyzh.data_ptr(), self.vm.data_ptr()
        s.perm, s.cell_hmax, s.order = self.perm.data_ptr(), self.cell_hmax.data_ptr(), self.order.data_ptr()
        s.slot_cell = self.slot_cell.data_ptr()
        s.cell_nhome = self.cell_nhome.data_ptr()
        s.disp, s.cell_dx = self.disp.data_ptr(), self.cell_dx.data_ptr()
        return s

    def order_np(self):
        """(13, capacity) int64 numpy copy of the sorted lists (in-cell indices)."""
        return self.order.cpu().numpy().view("uint16").astype("int64")


FIELDS = ("rho", "wcount", "rho_dh", "wcount_dh", "div_v", "curl_x", "curl_y", "curl_z", "nngb")


@dataclass
class Out:
    n_out: int
    rho: torch.Tensor
    rho_dh: torch.Tensor
    wcount: torch.Tensor
    wcount_dh: torch.Tensor
    div_v: torch.Tensor
    curl_v: torch.Tensor        # (3, n_out)
    nngb: torch.Tensor

    @staticmethod
    def alloc(n_out: int, device="cuda", zero=False) -> "Out":
        n = max(int(n_out), 1)
        f = (torch.zeros if zero else torch.empty)
        return Out(int(n_out), *(f(n, dtype=torch.float32, device=device) for _ in range(5)),
                   f((3, n), dtype=torch.float32, device=device), f(n, dtype=torch.int32, device=device))

    def zero_(self) -> "Out":
        for t in (self.rho, self.rho_dh, self.wcount, self.wcount_dh, self.div_v, self.curl_v, self.nngb):
            t.zero_()
        return self

    def struct(self) -> SphOut:
        s = SphOut()
        s.n_out = self.n_out
        s.rho, s.rho_dh, s.wcount = self.rho.data_ptr(), self.rho_dh.data_ptr(), self.wcount.data_ptr()
        s.wcount_dh, s.div_v, s.curl_v = self.wcount_dh.data_ptr(), self.div_v.data_ptr(), self.curl_v.data_ptr()
        s.nngb = self.nngb.data_ptr()
        return s

    def to_numpy(self) -> dict:
        n = self.n_out
        d = {"rho": self.rho[:n], "wcount": self.wcount[:n], "rho_dh": self.rho_dh[:n],
             "wcount_dh": self.wcount_dh[:n], "div_v": self.div_v[:n], "curl_x": self.curl_v[0, :n],
             "curl_y": self.curl_v[1, :n], "curl_z": self.curl_v[2, :n], "nngb": self.nngb[:n]}
        return {k: v.cpu().numpy() for k, v in d.items()}


class Stats:
    def __init__(self, device="cuda"):
        self.buf = torch.zeros(9, dtype=torch.int64, device=device)   # sph_stats: cand[4], hits[4], band

    def ptr(self):
        return _ptr(self.buf)

    def read(self) -> dict:
        v = self.buf.cpu().tolist()
        return {"cand": v[:4], "hits": v[4:8], "band": v[8]}


def alloc_workspace(grid: SphGrid, capacity: int, device="cuda") -> torch.Tensor:
    return torch.zeros(workspace_bytes(grid, capacity), dtype=torch.uint8, device=device)


# ---- the C ABI calls ---------------------------------------------------------
def sph_build_cells(grid: SphGrid, xyzh_in: torch.Tensor, vm_in: torch.Tensor, cells: Cells, ws: torch.Tensor,
                    n_own: int | None = None, n_ghost: int = 0, stream=None) -> None:
    n_total = xyzh_in.shape[0] if n_own is None else int(n_own) + int(n_ghost)
    n_own = n_total - int(n_ghost) if n_own is None else int(n_own)
    assert xyzh_in.is_contiguous() and vm_in.is_contiguous()
    s = cells.struct()
    _check(_lib.load().sph_build_cells(ctypes.byref(grid), n_own, int(n_ghost), _ptr(xyzh_in), _ptr(vm_in),
                                       ctypes.byref(s), _ptr(ws), ws.numel(), _stream(stream)), "sph_build_cells")
    cells.n = int(s.n)


def sph_build_sort_cells(grid: SphGrid, xyzh_in: torch.Tensor, vm_in: torch.Tensor, cells: Cells, ws: torch.Tensor,
                         n_own: int | None = None, n_ghost: int = 0, stream=None) -> None:
    """sph_build_cells + sph_sort_cells over all cells in one call (ABI v7; the small cells'
    lists come out of the build's placement pass on a single grid)."""
    n_total = xyzh_in.shape[0] if n_own is None else int(n_own) + int(n_ghost)
    n_own = n_total - int(n_ghost) if n_own is None else int(n_own)
    assert xyzh_in.is_contiguous() and vm_in.is_contiguous()
    s = cells.struct()
    _check(_lib.load().sph_build_sort_cells(ctypes.byref(grid), n_own, int(n_ghost), _ptr(xyzh_in), _ptr(vm_in),
                                            ctypes.byref(s), _ptr(ws), ws.numel(), _stream(stream)),
           "sph_build_sort_cells")
    cells.n = int(s.n)


def sph_sort_cells(grid: SphGrid, cells: Cells, ws: torch.Tensor, cell_begin: int = 0, cell_end: int = -1,
                   stream=None) -> None:
    s = cells.struct()
    _check(_lib.load().sph_sort_cells(ctypes.byref(grid), ctypes.byref(s), int(cell_begin), int(cell_end),
                                      _ptr(ws), ws.numel(), _stream(stream)), "sph_sort_cells")


def sph_density_self(grid: SphGrid, cells: Cells, cell_list: torch.Tensor, acc: Out, ws: torch.Tensor,
                     stats: Stats | None = None, stream=None) -> None:
    s, o = cells.struct(), acc.struct()
    _check(_lib.load().sph_density_self(ctypes.byref(grid), ctypes.byref(s), _ptr(cell_list), cell_list.numel(),
                                        ctypes.byref(o), stats.ptr() if stats else None, _ptr(ws), ws.numel(),
                                        _stream(stream)), "sph_density_self")


def sph_density_pair(grid: SphGrid, cells: Cells, pairs: torch.Tensor, acc: Out, ws: torch.Tensor,
                     stats: Stats | None = None, stream=None) -> None:
    assert pairs.dtype == torch.int32 and pairs.is_contiguous() and (pairs.numel() == 0 or pairs.shape[-1] == 2)
    s, o = cells.struct(), acc.struct()
    _check(_lib.load().sph_density_pair(ctypes.byref(grid), ctypes.byref(s), _ptr(pairs), pairs.numel() // 2,
                                        ctypes.byref(o), stats.ptr() if stats else None, _ptr(ws), ws.numel(),
                                        _stream(stream)), "sph_density_pair")


def sph_density_pair_sym(grid: SphGrid, cells: Cells, pairs: torch.Tensor, acc: Out, ws: torch.Tensor,
                         stats: Stats | None = None, stream=None) -> None:
    """Symmetric pairs (include/sph.h): each unordered (ci, cj) listed once, both sides updated."""
    assert pairs.dtype == torch.int32 and pairs.is_contiguous() and (pairs.numel() == 0 or pairs.shape[-1] == 2)
    s, o = cells.struct(), acc.struct()
    _check(_lib.load().sph_density_pair_sym(ctypes.byref(grid), ctypes.byref(s), _ptr(pairs), pairs.numel() // 2,
                                            ctypes.byref(o), stats.ptr() if stats else None, _ptr(ws), ws.numel(),
                                            _stream(stream)), "sph_density_pair_sym")


def sph_drift(grid: SphGrid, cells: Cells, dt: float, max_disp: torch.Tensor | None = None, stream=None) -> None:
    """List reuse: x <- x + v dt for the stored particles (include/sph.h), accumulating each
    particle's displacement bound and the per-cell max_dx; max_disp: a (1,) float32
    device tensor receiving the largest displacement bound since the build (atomic max)."""
    s = cells.struct()
    _check(_lib.load().sph_drift(ctypes.byref(grid), ctypes.byref(s), float(dt),
                                 _ptr(max_disp) if max_disp is not None else None, _stream(stream)), "sph_drift")


def sph_gather_positions(grid: SphGrid, cells: Cells, xyzh_out: torch.Tensor, n_out: int, stream=None) -> None:
    """The stored (drifted) positions back in input order, wrapped into the box (include/sph.h)."""
    assert xyzh_out.is_contiguous() and xyzh_out.dtype == torch.float32
    s = cells.struct()
    _check(_lib.load().sph_gather_positions(ctypes.byref(grid), ctypes.byref(s), _ptr(xyzh_out), int(n_out),
                                            _stream(stream)), "sph_gather_positions")


def sph_select_planes(grid: SphGrid, xyzh: torch.Tensor, vm: torch.Tensor, n_own: int, sel_x: torch.Tensor,
                      sel_v: torch.Tensor, counts: torch.Tensor, ws: torch.Tensor, stream=None) -> None:
    """x-slab ghost exchange: the owned particles of planes x_lo (list 0) and x_hi - 1 (list 1)
    in input order into sel_x/sel_v ((2, cap, 4) float32); counts: (2,) int64 device tensor."""
    assert sel_x.shape[0] == 2 and sel_x.shape == sel_v.shape and counts.dtype == torch.int64
    _check(_lib.load().sph_select_planes(ctypes.byref(grid), int(n_own), _ptr(xyzh), _ptr(vm), _ptr(sel_x),
                                         _ptr(sel_v), sel_x.shape[1], _ptr(counts), _ptr(ws), ws.numel(),
                                         _stream(stream)), "sph_select_planes")


def sph_mask_ghost_rows(recv_x: torch.Tensor, recv_v: torch.Tensor, counts: torch.Tensor, dead_x, dead_v,
                        stream=None) -> None:
    """Rows past counts[k] of the received ghost blocks recv_x/recv_v ((2, cap, 4) float32,
    device) become the dead particle (dead_x, dead_v: 4 host floats each); counts: (2,) int64
    device tensor, read on the device."""
    assert recv_x.shape[0] == 2 and recv_x.shape == recv_v.shape and counts.dtype == torch.int64
    assert recv_x.is_contiguous() and recv_v.is_contiguous()
    fx = (ctypes.c_float * 4)(*[float(a) for a in dead_x])
    fv = (ctypes.c_float * 4)(*[float(a) for a in dead_v])
    _check(_lib.load().sph_mask_ghost_rows(_ptr(recv_x), _ptr(recv_v), recv_x.shape[1], _ptr(counts), fx, fv,
                                           _stream(stream)), "sph_mask_ghost_rows")


def sph_partition_migrants(grid: SphGrid, n: int, xyzh: torch.Tensor, vm: torch.Tensor, gid: torch.Tensor,
                           lo, hi, keep, counts: torch.Tensor, ws: torch.Tensor, stream=None) -> None:
    """Stable three-way split of the n owned particles (wrapped positions, ascending gid) by x
    plane: lo / hi / keep = [xyzh (cap, 4), vm (cap, 4), gid (cap,) int64] buffers; counts:
    (3,) int64 device tensor."""
    assert counts.dtype == torch.int64 and counts.numel() >= 3 and gid.dtype == torch.int64
    args = []
    for b in (lo, hi, keep):
        assert b[2].dtype == torch.int64 and b[0].shape[0] == b[1].shape[0] == b[2].shape[0]
        args += [_ptr(b[0]), _ptr(b[1]), _ptr(b[2]), int(b[0].shape[0])]
    _check(_lib.load().sph_partition_migrants(ctypes.byref(grid), int(n), _ptr(xyzh), _ptr(vm), _ptr(gid), *args,
                                              _ptr(counts), _ptr(ws), ws.numel(), _stream(stream)),
           "sph_partition_migrants")


def sph_merge_by_id(lists, out_x: torch.Tensor, out_v: torch.Tensor, out_g: torch.Tensor, stream=None) -> None:
    """Merge of three (xyzh, vm, gid, n) lists, each ascending in gid, into out_* (n total)."""
    assert len(lists) == 3
    args = []
    for x, v, g, n in lists:
        assert g.dtype == torch.int64
        args += [int(n), _ptr(x), _ptr(v), _ptr(g)]
    _check(_lib.load().sph_merge_by_id(*args, _ptr(out_x), _ptr(out_v), _ptr(out_g), _stream(stream)),
           "sph_merge_by_id")


def sph_max_speed(vm: torch.Tensor, n: int | None = None, stream=None) -> float:
    """max |v| over the first n rows of vm ((N, 4) float32, device), fp64; one host sync."""
    n = vm.shape[0] if n is None else int(n)
    out = torch.zeros(1, dtype=torch.float64, device=vm.device)
    _check(_lib.load().sph_max_speed(_ptr(vm), n, _ptr(out), _stream(stream)), "sph_max_speed")
    return float(out.item())


def sph_density_finalize(acc: Out, n: int | None = None, stream=None) -> None:
    o = acc.struct()
    _check(_lib.load().sph_density_finalize(ctypes.byref(o), acc.n_out if n is None else int(n), _stream(stream)),
           "sph_density_finalize")


def sph_density_all(grid: SphGrid, cells: Cells, out: Out, ws: torch.Tensor, stats: Stats | None = None,
                    stream=None) -> None:
    s, o = cells.struct(), out.struct()
    _check(_lib.load().sph_density_all(ctypes.byref(grid), ctypes.byref(s), ctypes.byref(o),
                                       stats.ptr() if stats else None, _ptr(ws), ws.numel(), _stream(stream)),
           "sph_density_all")


def sph_density_all_sym(grid: SphGrid, cells: Cells, out: Out, ws: torch.Tensor, stats: Stats | None = None,
                        stream=None) -> None:
    """The symmetric sweep over the whole pass, conflict-free by colour phases (include/sph.h)."""
    s, o = cells.struct(), out.struct()
    _check(_lib.load().sph_density_all_sym(ctypes.byref(grid), ctypes.byref(s), ctypes.byref(o),
                                           stats.ptr() if stats else None, _ptr(ws), ws.numel(), _stream(stream)),
           "sph_density_all_sym")


def sph_status(ws: torch.Tensor, stream=None) -> int:
    return int(_lib.load().sph_status(_ptr(ws), _stream(stream)))


def sph_status_reset(ws: torch.Tensor, stream=None) -> None:
    _check(_lib.load().sph_status_reset(_ptr(ws), _stream(stream)), "sph_status_reset")


def check_status(ws: torch.Tensor, stream=None) -> None:
    _check(sph_status(ws, stream), "sph_status")


# ---- convenience: one full density pass ---------------------------------------
class DensityPass:
    """Owns the device buffers of one configuration and runs
    build_cells + sort_cells (one fused call) -> density_all (the hot path)."""

    def __init__(self, nc, n_own: int, box=1.0, gamma=GAMMA, capacity: int | None = None, device="cuda",
                 x_lo=0, x_hi=None, ghost_x=0, h_home=None, skin=0.0):
        self.grid = make_grid(nc, box, gamma, x_lo, x_hi, ghost_x, h_home, skin)
        self.n_own = int(n_own)
        cap = int(capacity if capacity is not None else n_own)
        self.cells = Cells.alloc(self.grid, cap, device)
        self.ws = alloc_workspace(self.grid, self.cells.capacity, device)
        self.out = Out.alloc(self.n_own, device)
        self.device = device

    def run(self, xyzh: torch.Tensor, vm: torch.Tensor, n_ghost: int = 0, stats: Stats | None = None,
            stream=None, out: Out | None = None) -> Out:
        out = self.out if out is None else out
        sph_build_sort_cells(self.grid, xyzh, vm, self.cells, self.ws, n_own=self.n_own, n_ghost=n_ghost,
                             stream=stream)
        sph_density_all(self.grid, self.cells, out, self.ws, stats=stats, stream=stream)
        return out

    def check(self, stream=None) -> None:
        check_status(self.ws, stream)


class ReuseLoop:
    """Time loop with pseudo-Verlet list reuse ("max_dx").

    Cells and sorted lists are built on a grid with a skin s.  Every step drifts the stored
    particles (sph_drift: each particle's displacement bound and the per-cell max_dx grow) and
    runs sph_density_all, whose window in a neighbour cell c is widened by 2 max_dx(c).  Before a
    drift that could take any particle's accumulated displacement past s, the loop rebuilds:
    the current positions are gathered back to input order and wrapped into the box
    (sph_gather_positions), then sph_build_cells + sph_sort_cells.  The decision is made on the
    host from a bound (largest |v| dt per step, measured once at start(), plus rounding), so a
    step needs no host synchronisation."""

    def __init__(self, nc, n: int, skin: float, box=1.0, gamma=GAMMA, device="cuda"):
        self.dp = DensityPass(nc, n, box, gamma, device=device, skin=skin)
        self.skin = float(skin)
        self.n = int(n)
        self.x = torch.empty((max(self.n, 1), 4), dtype=torch.float32, device=device)   # input order
        self.v = None
        self.vmax = 0.0
        self.bound = 0.0                     # host bound of the displacement since the last build
        self.rebuilds = 0
        self.rebuild_steps = []
        self.steps = 0
        self.max_disp = torch.zeros(1, dtype=torch.float32, device=device)

    def _build(self, stream=None):
        sph_build_sort_cells(self.dp.grid, self.x, self.v, self.dp.cells, self.dp.ws, n_own=self.n, stream=stream)
        self.bound = 0.0
        self.max_disp.zero_()

    def start(self, xyzh: torch.Tensor, vm: torch.Tensor, stream=None) -> None:
        """Initial state (input order, device) and the first build; one host sync for max |v|."""
        self.x[:self.n].copy_(xyzh)
        self.v = vm
        self.vmax = sph_max_speed(vm, self.n, stream) if self.n else 0.0
        self._build(stream)

    def step_bound(self, dt: float) -> float:
        """Upper bound of one drift's stored increment: |v| dt with both fp32 roundings (v dt,
        then the position sum: <= 2^-24 |x| per component, |x| < box + skin)."""
        box = max(self.dp.grid.box[0], self.dp.grid.box[1], self.dp.grid.box[2])
        return self.vmax * abs(dt) * (1.0 + 2.0 ** -20) + 3.0 ** 0.5 * 2.0 ** -24 * (box + self.skin) * 1.01

    def step(self, dt: float, stats: Stats | None = None, stream=None, events=None) -> Out:
        """events (optional): two CUDA events recorded around sph_density_all (timing only)."""
        inc = self.step_bound(dt)
        if inc > self.skin:
            raise ValueError(f"one drift ({inc}) exceeds the skin ({self.skin}): smaller dt or a larger skin")
        if self.bound + inc > self.skin:     # this drift could leave the skin: rebuild from the current state
            sph_gather_positions(self.dp.grid, self.dp.cells, self.x, self.n, stream=stream)
            self._build(stream)
            self.rebuilds += 1
            self.rebuild_steps.append(self.steps)
        sph_drift(self.dp.grid, self.dp.cells, dt, self.max_disp, stream=stream)
        self.bound += inc
        self.steps += 1
        if events:
            events[0].record(torch.cuda.current_stream() if stream is None else stream)
        sph_density_all(self.dp.grid, self.dp.cells, self.dp.out, self.dp.ws, stats=stats, stream=stream)
        if events:
            events[1].record(torch.cuda.current_stream() if stream is None else stream)
        return self.dp.out

    def check(self, stream=None) -> None:
        """Raise on errors; also verifies the device displacement against the host bound."""
        self.dp.check(stream)
        md = float(self.max_disp.item())
        if md > self.skin:
            raise RuntimeError(f"displacement {md} since the build exceeds the skin {self.skin}")


def level_grids(h, nc0: int, box=1.0, gamma=GAMMA, max_levels: int = 3):
    """Level passes for clustered data: cell grids nc0, 2 nc0, 4 nc0, ...
    Level k is home to the particles whose support fits its cells but not the next finer
    ones: h_max(k) = the largest fp32 h with gamma h <= box / nc_k, h_min(k) = h_max(k + 1)
    (0 for the finest).  Levels without particles are dropped.  Returns [(nc, h_min, h_max)]."""
    import numpy as np

    def hcap(nc):
        c = float(box) / nc
        v = np.float32(c / gamma)
        while float(gamma) * float(v) > c:
            v = np.nextafter(v, np.float32(0))
        return float(v)

    h = np.asarray(h, np.float32)
    ncs = [nc0 * 2 ** k for k in range(max_levels)]
    caps = [hcap(n) for n in ncs]
    if h.size and float(h.max()) > caps[0]:
        # such a particle would be home on no level (its outputs never written): the coarsest
        # grid itself is too fine (sph_build_cells reports SPH_EH_RANGE for a single grid)
        raise ValueError(f"h = {float(h.max())} exceeds the coarsest level's limit {caps[0]} (gamma h > box/nc0)")
    out = []
    for k, n in enumerate(ncs):
        lo = caps[k + 1] if k + 1 < len(ncs) else 0.0
        if np.any((h > lo) & (h <= caps[k])):
            out.append((n, lo, caps[k]))
    return out


class LevelPasses:
    """One density pass per level grid, all writing the same outputs: each
    particle is home on exactly one level; every level bins all particles as neighbours."""

    def __init__(self, levels, n: int, box=1.0, gamma=GAMMA, device="cuda"):
        self.levels = list(levels)
        self.passes = [DensityPass(nc, n, box, gamma, device=device,
                                   h_home=(lo, hi) if len(self.levels) > 1 else None)
                       for nc, lo, hi in self.levels]
        self.out = self.passes[0].out

    def run(self, xyzh: torch.Tensor, vm: torch.Tensor, stats: Stats | None = None, stream=None) -> Out:
        for dp in self.passes:
            dp.run(xyzh, vm, stats=stats, stream=stream, out=self.out)
        return self.out

    def check(self, stream=None) -> None:
        for dp in self.passes:
            dp.check(stream)


def density_levels(xyzh, vm, levels, box=1.0, gamma=GAMMA, stats: bool = False):
    """Like density(), through level passes [(nc, h_min, h_max)] (level_grids())."""
    xyzh = torch.as_tensor(xyzh, dtype=torch.float32).cuda().contiguous()
    vm = torch.as_tensor(vm, dtype=torch.float32).cuda().contiguous()
    lp = LevelPasses(levels, xyzh.shape[0], box, gamma)
    st = Stats() if stats else None
    out = lp.run(xyzh, vm, stats=st)
    lp.check()
    res = out.to_numpy()
    if stats:
        res["stats"] = st.read()
    return res


def density(xyzh, vm, nc, box=1.0, gamma=GAMMA, stats: bool = False):
    """One-shot helper: host or device float32 (N,4) arrays -> dict of numpy outputs."""
    xyzh = torch.as_tensor(xyzh, dtype=torch.float32).cuda().contiguous()
    vm = torch.as_tensor(vm, dtype=torch.float32).cuda().contiguous()
    dp = DensityPass(nc, xyzh.shape[0], box, gamma)
    st = Stats() if stats else None
    out = dp.run(xyzh, vm, stats=st)
    dp.check()
    res = out.to_numpy()
    if stats:
        res["stats"] = st.read()
    return res
