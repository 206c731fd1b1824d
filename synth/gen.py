"""Seeded synthetic workloads c1..c5 (BASELINE.json `configs`).

Input recipe (the readings are listed in DESIGN.md §2):

* periodic unit cube, L = 1; equal masses m = 1/N (exact in fp32, N is a
  power of two);
* every position lies on the 2^-24 grid, x = k·2^-24 with k in [0, 2^24),
  so it is exact in fp32, never rounds to 1.0f, and a translation by a
  dyadic amount is exact;
* particles are drawn in chunks of 2^20 consecutive particles; chunk c draws
  from its own stream ``Generator(PCG64(SeedSequence([seed, c])))`` in the
  fixed order positions -> h jitter -> velocities.  Chunks are independent,
  so large sets are generated in parallel with identical results;
* arrays are returned as ``xyzh = (x, y, z, h)`` and ``vm = (vx, vy, vz, m)``,
  float32, shape (N, 4), in the config's input order.

Nothing here evaluates the SPH kernel, searches neighbours or sums anything
the density method computes; c4's analytic Plummer density only sets the
input smoothing lengths (BASELINE.json configs[3]).
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

GAMMA = 1.825742          # kernel support / smoothing length (BASELINE.json configs)
ETA = 1.2348              # smoothing length / mean inter-particle spacing (BASELINE.json configs)
GRID = 1 << 24            # position grid: x = k * 2^-24
CHUNK = 1 << 20           # particles per independent random stream


@dataclass
class ParticleSet:
    name: str
    seed: int
    xyzh: np.ndarray       # (N, 4) float32: x, y, z, h
    vm: np.ndarray         # (N, 4) float32: vx, vy, vz, m
    nc: int                # cells per dimension of the cell grid (cube)
    box: float = 1.0
    gamma: float = GAMMA
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.xyzh.shape[0])

    @property
    def cell_edge(self) -> float:
        return self.box / self.nc

    def subset(self, idx) -> "ParticleSet":
        return ParticleSet(self.name + "-sub", self.seed, np.ascontiguousarray(self.xyzh[idx]),
                           np.ascontiguousarray(self.vm[idx]), self.nc, self.box, self.gamma,
                           dict(self.meta))


def _rng(seed: int, chunk: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), int(chunk)])))


def _grid_from_float(x: np.ndarray) -> np.ndarray:
    """Wrap into [0,1) and snap onto the 2^-24 grid (returns float32)."""
    k = np.floor(np.mod(x, 1.0) * GRID).astype(np.int64) % GRID
    return (k.astype(np.float64) / GRID).astype(np.float32)


def _inv_cbrt(n: int) -> float:
    side = round(n ** (1.0 / 3.0))
    if side ** 3 == n:
        return 1.0 / side
    return n ** (-1.0 / 3.0)


def _nthreads() -> int:
    return max(1, min(16, os.cpu_count() or 1))


def _run_chunks(n: int, fn) -> None:
    nchunk = (n + CHUNK - 1) // CHUNK
    if nchunk <= 1:
        for c in range(nchunk):
            fn(c)
        return
    with ThreadPoolExecutor(max_workers=_nthreads()) as ex:
        list(ex.map(fn, range(nchunk)))


def uniform_set(name: str, seed: int, n: int, nc: int, h_jitter: float, v_sigma: float,
                h_mean: float | None = None) -> ParticleSet:
    """Uniform random positions on the 2^-24 grid (configs c1, c3, c5).

    h_i = h_mean * (1 + U(-h_jitter, h_jitter)), h_mean = ETA * N^(-1/3) by default;
    with h_jitter == 0 the jitter draw is skipped (c1: all h equal)."""
    if h_mean is None:
        h_mean = ETA * _inv_cbrt(n)
    xyzh = np.empty((n, 4), np.float32)
    vm = np.empty((n, 4), np.float32)
    m = np.float32(1.0 / n)

    def chunk(c):
        lo, hi = c * CHUNK, min(n, (c + 1) * CHUNK)
        k = hi - lo
        g = _rng(seed, c)
        pos = g.integers(0, GRID, size=(k, 3), dtype=np.int64)
        xyzh[lo:hi, 0:3] = (pos.astype(np.float64) / GRID).astype(np.float32)
        if h_jitter > 0:
            u = g.uniform(-h_jitter, h_jitter, size=k)
            xyzh[lo:hi, 3] = (h_mean * (1.0 + u)).astype(np.float32)
        else:
            xyzh[lo:hi, 3] = np.float32(h_mean)
        vm[lo:hi, 0:3] = (v_sigma * g.standard_normal((k, 3))).astype(np.float32)
        vm[lo:hi, 3] = m

    _run_chunks(n, chunk)
    return ParticleSet(name, seed, xyzh, vm, nc)


def lattice_set(name: str, seed: int, side: int, jitter: float, h_jitter: float, v_sigma: float,
                nc: int | None = None) -> ParticleSet:
    """Jittered cubic lattice (config c2): sites (i + 1/2)/side, i-major order
    (x index slowest), plus independent U(-jitter, jitter)/side per component,
    wrapped into [0,1); h = ETA/side * (1 + U(-h_jitter, h_jitter)).
    nc defaults to floor(L / max_i(GAMMA*h_i)) (reading B20 in DESIGN.md)."""
    n = side ** 3
    xyzh = np.empty((n, 4), np.float32)
    vm = np.empty((n, 4), np.float32)
    m = np.float32(1.0 / n)
    h_mean = ETA / side

    def chunk(c):
        lo, hi = c * CHUNK, min(n, (c + 1) * CHUNK)
        k = hi - lo
        g = _rng(seed, c)
        idx = np.arange(lo, hi, dtype=np.int64)
        ix, iy, iz = idx // (side * side), (idx // side) % side, idx % side
        site = (np.stack([ix, iy, iz], 1).astype(np.float64) + 0.5) / side
        if jitter > 0:
            site = site + g.uniform(-jitter, jitter, size=(k, 3)) / side
        xyzh[lo:hi, 0:3] = _grid_from_float(site)
        if h_jitter > 0:
            xyzh[lo:hi, 3] = (h_mean * (1.0 + g.uniform(-h_jitter, h_jitter, size=k))).astype(np.float32)
        else:
            xyzh[lo:hi, 3] = np.float32(h_mean)
        vm[lo:hi, 0:3] = (v_sigma * g.standard_normal((k, 3))).astype(np.float32)
        vm[lo:hi, 3] = m

    _run_chunks(n, chunk)
    if nc is None:
        hmax = float(np.max(xyzh[:, 3].astype(np.float64)))
        nc = int(math.floor(1.0 / (GAMMA * hmax)))
    return ParticleSet(name, seed, xyzh, vm, nc)


def clustered_set(name: str, seed: int, n: int, nc: int, n_spheres: int = 512,
                  frac_plummer: float = 0.6, v_sigma: float = 1.0) -> ParticleSet:
    """Config c4 (reading B22 in DESIGN.md): round(0.6 N) particles split evenly
    over 512 Plummer spheres (centres U[0,1)^3, scale radii U(0.002, 0.02)),
    the rest uniform background; h_i = ETA (m / rho_analytic(x_i))^(1/3),
    clamped to <= C_l / GAMMA.  Plummer particles first (sphere order), then
    background; no shuffle."""
    setup = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), 0xFFFFFFFF])))
    centres = setup.random((n_spheres, 3))
    radii = setup.uniform(0.002, 0.02, n_spheres)
    n_p = int(round(frac_plummer * n))
    counts = np.full(n_spheres, n_p // n_spheres, np.int64)
    counts[: n_p % n_spheres] += 1
    first = np.concatenate([[0], np.cumsum(counts)])
    xyzh = np.empty((n, 4), np.float32)
    vm = np.empty((n, 4), np.float32)
    m = 1.0 / n

    def chunk(c):
        lo, hi = c * CHUNK, min(n, (c + 1) * CHUNK)
        g = _rng(seed, c)
        plo, phi = lo, min(hi, n_p)
        if phi > plo:
            k = phi - plo
            sph = np.searchsorted(first, np.arange(plo, phi), side="right") - 1
            x = g.random(k)
            d = g.standard_normal((k, 3))
            d /= np.linalg.norm(d, axis=1, keepdims=True)
            with np.errstate(divide="ignore", invalid="ignore"):
                r = radii[sph] / np.sqrt(np.power(x, -2.0 / 3.0) - 1.0)
            r = np.where(np.isfinite(r), r, 0.0)
            xyzh[plo:phi, 0:3] = _grid_from_float(centres[sph] + r[:, None] * d)
        blo = max(lo, n_p)
        if hi > blo:
            k = hi - blo
            pos = g.integers(0, GRID, size=(k, 3), dtype=np.int64)
            xyzh[blo:hi, 0:3] = (pos.astype(np.float64) / GRID).astype(np.float32)
        vm[lo:hi, 0:3] = (v_sigma * g.standard_normal((hi - lo, 3))).astype(np.float32)
        vm[lo:hi, 3] = np.float32(m)

    _run_chunks(n, chunk)
    rho = _plummer_density(xyzh[:, 0:3], centres, radii, counts * m, 1.0 - n_p * m)
    h = ETA * np.cbrt(m / rho)
    h = np.minimum(h, (1.0 / nc) / GAMMA)
    xyzh[:, 3] = h.astype(np.float32)
    # fp32 rounding of h could exceed the clamp by an ulp; pull it back.
    while True:
        bad = (xyzh[:, 3].astype(np.float64) * GAMMA) > (1.0 / nc)
        if not bad.any():
            break
        xyzh[bad, 3] = np.nextafter(xyzh[bad, 3], np.float32(0))
    return ParticleSet(name, seed, xyzh, vm, nc,
                       meta={"n_plummer": n_p, "centres": centres, "radii": radii})


PLUMMER_RCUT = 0.125   # sphere contributions summed within this minimum-image distance (reading R12)


def _plummer_density(pos32, centres, radii, masses, background) -> np.ndarray:
    """Analytic total density: background + sum_s 3M_s/(4 pi a_s^3) (1 + d_s^2/a_s^2)^(-5/2),
    d_s the minimum-image distance, each sphere summed where d_s < PLUMMER_RCUT (input recipe
    only; beyond it a sphere adds < 1 % of the background).  Spheres are added in index order
    (fp64), each over the particles of the coarse grid cells within reach, so the result does
    not depend on the machine or the thread count."""
    n = pos32.shape[0]
    pos = pos32.astype(np.float64)
    g = 16                                         # coarse grid, cell 1/16 >= PLUMMER_RCUT / 2
    cell = np.clip(np.floor(pos * g).astype(np.int64), 0, g - 1)
    key = (cell[:, 0] * g + cell[:, 1]) * g + cell[:, 2]
    order = np.argsort(key, kind="stable")
    start = np.searchsorted(key[order], np.arange(g ** 3 + 1))
    rho = np.full(n, background, np.float64)
    reach = int(np.ceil(PLUMMER_RCUT * g))
    offs = np.arange(-reach, reach + 1)
    amp = 3.0 * masses / (4.0 * np.pi * radii ** 3)
    for s in range(centres.shape[0]):
        cc = np.floor(centres[s] * g).astype(np.int64)
        cx, cy, cz = [(cc[k] + offs) % g for k in range(3)]
        cells = ((cx[:, None, None] * g + cy[None, :, None]) * g + cz[None, None, :]).ravel()
        idx = np.concatenate([order[start[c]:start[c + 1]] for c in np.unique(cells)])
        d = pos[idx] - centres[s]
        d -= np.round(d)
        d2 = (d * d).sum(1)
        near = d2 < PLUMMER_RCUT ** 2
        rho[idx[near]] += amp[s] * (1.0 + d2[near] / radii[s] ** 2) ** -2.5
    return rho


def tiny_random_set(seed: int, n: int, nc: int, h_frac: float = 0.8, h_jitter: float = 0.3,
                    v_sigma: float = 1.0) -> ParticleSet:
    """Small random set for property tests: uniform positions on the 2^-24 grid,
    h_i = h_frac * C_l / GAMMA * (1 - U(0, h_jitter)) (so GAMMA*h_i <= C_l),
    random masses in [0.5, 1.5)/n."""
    g = _rng(seed, 0x7777)
    xyzh = np.empty((n, 4), np.float32)
    vm = np.empty((n, 4), np.float32)
    pos = g.integers(0, GRID, size=(n, 3), dtype=np.int64)
    xyzh[:, 0:3] = (pos.astype(np.float64) / GRID).astype(np.float32)
    hmax = h_frac * (1.0 / nc) / GAMMA
    xyzh[:, 3] = (hmax * (1.0 - g.uniform(0.0, h_jitter, n))).astype(np.float32)
    vm[:, 0:3] = (v_sigma * g.standard_normal((n, 3))).astype(np.float32)
    vm[:, 3] = (g.uniform(0.5, 1.5, n) / n).astype(np.float32)
    return ParticleSet(f"tiny-{seed}-{n}", seed, xyzh, vm, nc)


def test27cells_set(seed: int, nc: int, per_cell: int = 216, eta: float = ETA, v_sigma: float = 1.0) -> ParticleSet:
    """Batched test27cells instances: a periodic nc^3 grid whose
    every cell holds exactly `per_cell` particles placed uniformly at random inside it (on the
    2^-24 position grid, so fp64 binning puts each in its own cell); every cell is the centre
    of one 27-cell instance.  h = eta * C_l / per_cell^(1/3) for all particles (the mean
    inter-particle spacing times eta), masses 1/N, velocities N(0, v_sigma).  Particles are
    written cell by cell in x-major cell order."""
    ncell = nc ** 3
    n = ncell * per_cell
    g = _rng(seed, 0x2727)
    # grid-unit bounds of cell c along an axis: [ceil(c G / nc), ceil((c + 1) G / nc))
    lo = -((-np.arange(nc + 1, dtype=np.int64) * GRID) // nc)
    cell = np.repeat(np.arange(ncell, dtype=np.int64), per_cell)
    ix, iy, iz = cell // (nc * nc), (cell // nc) % nc, cell % nc
    xyzh = np.empty((n, 4), np.float32)
    for a, ia in enumerate((ix, iy, iz)):
        k = lo[ia] + (g.random(n) * (lo[ia + 1] - lo[ia])).astype(np.int64)
        xyzh[:, a] = (k.astype(np.float64) / GRID).astype(np.float32)
    h = eta * (1.0 / nc) / per_cell ** (1.0 / 3.0)
    xyzh[:, 3] = np.float32(h)
    vm = np.empty((n, 4), np.float32)
    vm[:, 0:3] = (v_sigma * g.standard_normal((n, 3))).astype(np.float32)
    vm[:, 3] = np.float32(1.0 / n)
    return ParticleSet(f"test27cells-{nc}-{per_cell}", seed, xyzh, vm, nc,
                       meta={"per_cell": per_cell, "eta": eta})


# ---------------------------------------------------------------------------
# The five BASELINE.json configurations (DESIGN.md §3 gives the readings).
# ---------------------------------------------------------------------------
CONFIGS = {
    "c1": dict(kind="uniform", seed=0, n=4096, nc=5, h_jitter=0.0, v_sigma=0.1),
    "c2": dict(kind="lattice", seed=1, side=32, jitter=0.3, h_jitter=0.1, v_sigma=0.1),
    "c3": dict(kind="uniform", seed=2, n=128 ** 3, nc=47, h_jitter=0.2, v_sigma=1.0),
    "c4": dict(kind="clustered", seed=3, n=256 ** 3, nc=83),
    "c5": dict(kind="uniform", seed=4, n=512 ** 3, nc=184, h_jitter=0.2, v_sigma=1.0),
}


def make_config(name: str) -> ParticleSet:
    cfg = dict(CONFIGS[name])
    kind = cfg.pop("kind")
    if kind == "uniform":
        return uniform_set(name, **cfg)
    if kind == "lattice":
        return lattice_set(name, **cfg)
    if kind == "clustered":
        return clustered_set(name, **cfg)
    raise ValueError(kind)


make = make_config
