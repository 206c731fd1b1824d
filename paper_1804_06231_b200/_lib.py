"""ctypes view of include/sph.h (argument marshalling only; no arithmetic)."""
from __future__ import annotations

import ctypes
import os

from ._build import LIB

c_i32, c_i64, c_f32, c_f64, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double, ctypes.c_void_p

SPH_OK, SPH_EINVAL, SPH_EH_RANGE, SPH_ECAPACITY, SPH_EDOMAIN, SPH_ECUDA = range(6)
SPH_MAX_CELL = 65535
SPH_NDIR = 13
SPH_DELTA_FRAC = 1.0 / 65536.0
ERROR_NAMES = {0: "SPH_OK", 1: "SPH_EINVAL", 2: "SPH_EH_RANGE", 3: "SPH_ECAPACITY", 4: "SPH_EDOMAIN", 5: "SPH_ECUDA"}

# Every function declared in include/sph.h (checked by tests/test_abi.py); sph_calibrate is
# declared in include/sph_calib.h.
EXPORTS = ("sph_abi_version", "sph_ncell", "sph_workspace_bytes", "sph_build_cells", "sph_sort_cells", "sph_build_sort_cells",
           "sph_density_self", "sph_density_pair", "sph_density_pair_sym", "sph_drift", "sph_gather_positions",
           "sph_select_planes", "sph_mask_ghost_rows", "sph_partition_migrants", "sph_merge_by_id",
           "sph_max_speed", "sph_density_finalize", "sph_density_all", "sph_density_all_sym", "sph_status",
           "sph_status_reset", "sph_strerror")


class SphGrid(ctypes.Structure):
    _fields_ = [("nc", c_i32 * 3), ("x_lo", c_i32), ("x_hi", c_i32), ("ghost_x", c_i32), ("reserved", c_i32),
                ("box", c_f64 * 3), ("gamma", c_f32), ("h_home_min", c_f32), ("h_home_max", c_f32),
                ("skin", c_f32)]


class SphCells(ctypes.Structure):
    _fields_ = [("capacity", c_i64), ("n", c_i64), ("cell_start", c_vp), ("xyzh", c_vp), ("vm", c_vp),
                ("perm", c_vp), ("cell_hmax", c_vp), ("order", c_vp), ("slot_cell", c_vp),
                ("cell_nhome", c_vp), ("disp", c_vp), ("cell_dx", c_vp)]


class SphOut(ctypes.Structure):
    _fields_ = [("n_out", c_i64), ("rho", c_vp), ("rho_dh", c_vp), ("wcount", c_vp), ("wcount_dh", c_vp),
                ("div_v", c_vp), ("curl_v", c_vp), ("nngb", c_vp)]


class SphStats(ctypes.Structure):
    _fields_ = [("cand", ctypes.c_uint64 * 4), ("hits", ctypes.c_uint64 * 4), ("band", ctypes.c_uint64)]


_lib = None


class LibraryMissing(RuntimeError):
    pass


def load(path: str = LIB):
    """Load libpvsph.so.  Raises LibraryMissing (no fallback exists).  PVSPH_LIB names another build
    of the same library (A/B measurements of compile-time variants, scripts/)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("PVSPH_LIB", path)
    if not os.path.exists(path):
        raise LibraryMissing(f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    G, C, O, S = ctypes.POINTER(SphGrid), ctypes.POINTER(SphCells), ctypes.POINTER(SphOut), c_vp
    L.sph_abi_version.restype = ctypes.c_int
    L.sph_ncell.argtypes = [G]
    L.sph_ncell.restype = c_i64
    L.sph_workspace_bytes.argtypes = [G, c_i64]
    L.sph_workspace_bytes.restype = ctypes.c_size_t
    L.sph_build_cells.argtypes = [G, c_i64, c_i64, c_vp, c_vp, C, c_vp, ctypes.c_size_t, c_vp]
    L.sph_sort_cells.argtypes = [G, C, c_i64, c_i64, c_vp, ctypes.c_size_t, c_vp]
    L.sph_build_sort_cells.argtypes = [G, c_i64, c_i64, c_vp, c_vp, C, c_vp, ctypes.c_size_t, c_vp]
    L.sph_density_self.argtypes = [G, C, c_vp, c_i64, O, S, c_vp, ctypes.c_size_t, c_vp]
    L.sph_density_pair.argtypes = [G, C, c_vp, c_i64, O, S, c_vp, ctypes.c_size_t, c_vp]
    L.sph_density_pair_sym.argtypes = [G, C, c_vp, c_i64, O, S, c_vp, ctypes.c_size_t, c_vp]
    L.sph_drift.argtypes = [G, C, ctypes.c_float, c_vp, c_vp]
    L.sph_gather_positions.argtypes = [G, C, c_vp, c_i64, c_vp]
    L.sph_select_planes.argtypes = [G, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, ctypes.c_size_t, c_vp]
    L.sph_mask_ghost_rows.argtypes = [c_vp, c_vp, c_i64, c_vp, ctypes.POINTER(ctypes.c_float),
                                      ctypes.POINTER(ctypes.c_float), c_vp]
    L.sph_partition_migrants.argtypes = [G, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64,
                                         c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, ctypes.c_size_t, c_vp]
    L.sph_merge_by_id.argtypes = [c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp,
                                  c_vp, c_vp, c_vp, c_vp]
    L.sph_max_speed.argtypes = [c_vp, c_i64, c_vp, c_vp]
    L.sph_density_finalize.argtypes = [O, c_i64, c_vp]
    L.sph_density_all.argtypes = [G, C, O, S, c_vp, ctypes.c_size_t, c_vp]
    L.sph_density_all_sym.argtypes = [G, C, O, S, c_vp, ctypes.c_size_t, c_vp]
    L.sph_status.argtypes = [c_vp, c_vp]
    L.sph_status_reset.argtypes = [c_vp, c_vp]
    L.sph_calibrate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vp, c_vp]
    L.sph_calibrate.restype = ctypes.c_int
    L.sph_strerror.argtypes = [ctypes.c_int]
    L.sph_strerror.restype = ctypes.c_char_p
    for f in ("sph_build_cells", "sph_sort_cells", "sph_build_sort_cells", "sph_density_self", "sph_density_pair", "sph_density_pair_sym",
              "sph_drift", "sph_gather_positions", "sph_select_planes", "sph_mask_ghost_rows",
              "sph_partition_migrants", "sph_merge_by_id", "sph_max_speed",
              "sph_density_finalize",
              "sph_density_all", "sph_density_all_sym", "sph_status", "sph_status_reset"):
        getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L
