"""pvsph: the pseudo-Verlet SPH density loop of arXiv:1804.06231 on B200.

CUDA kernels for sm_100a behind the C ABI of include/sph.h (libpvsph.so,
built in-tree by ``__graft_entry__.build()``); this package is the thin
ctypes binding plus the x-slab multi-GPU plumbing.  No CPU fallback.
"""
from ._lib import LibraryMissing, load  # noqa: F401
from .api import (GAMMA, Cells, DensityPass, LevelPasses, Out, ReuseLoop, density_levels, level_grids, SphError, Stats, alloc_workspace, check_status, density,  # noqa: F401
                  make_grid, ncell, sph_build_cells, sph_build_sort_cells, sph_density_all, sph_density_all_sym, sph_density_finalize, sph_density_pair,
                  sph_density_self, sph_density_pair_sym, sph_drift, sph_gather_positions, sph_mask_ghost_rows, sph_max_speed, sph_merge_by_id, sph_partition_migrants,
                  sph_select_planes, sph_sort_cells,
                  sph_status, sph_status_reset, workspace_bytes)
