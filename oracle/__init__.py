"""CPU fp64 oracle for the pseudo-Verlet SPH density loop (arXiv:1804.06231).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_1804_06231_b200`` and never imports
it.  The arithmetic lives in ``oracle/oracle.c`` (plain C, fp64, OpenMP);
this module only marshals numpy arrays through ctypes.

Parity status: every output is pinned by tests/test_oracle_pins.py (see the
table in DESIGN.md §5); nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SRC_PATH = os.path.join(_HERE, "oracle.c")

FIELDS = ("rho", "wcount", "rho_dh", "wcount_dh", "div_v", "curl_x", "curl_y", "curl_z",
          "nngb", "band", "a_rho_dh", "a_wcount_dh", "a_div", "a_curl", "c_div", "c_curl")
KINDS = ("self", "face", "edge", "corner")
DELTA_FRAC = 2.0 ** -16      # window margin delta = 2^-16 C_l (reading R5)


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc -O2 -fopenmp, fp64, no fast-math)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-fno-fast-math",
               "-ffp-contract=off", "-o", LIB_PATH, SRC_PATH, "-lm"]
        subprocess.check_call(cmd)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        i64, f64, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_int
        vp = ctypes.c_void_p
        L.oracle_kernel.argtypes = [f64, f64, f64, ctypes.POINTER(f64), ctypes.POINTER(f64), ctypes.POINTER(f64)]
        L.oracle_kernel.restype = None
        L.oracle_bruteforce.argtypes = [i64, vp, vp, f64, f64, vp, i64, vp]
        L.oracle_celllist.argtypes = [i64, vp, vp, f64, f64, i32, vp, i64, vp]
        L.oracle_pv_counts.argtypes = [i64, vp, f64, f64, i32, f64, vp, i64, vp, vp]
        L.oracle_bin_cells.argtypes = [i64, vp, f64, i32, vp, vp, vp]
        L.oracle_cell_keys.argtypes = [i64, vp, f64, i32, vp]
        L.oracle_directions.argtypes = [vp]
        L.oracle_set_num_threads.argtypes = [i32]
        for f in ("oracle_bruteforce", "oracle_celllist", "oracle_pv_counts", "oracle_bin_cells",
                  "oracle_cell_keys", "oracle_directions", "oracle_num_threads", "oracle_nout"):
            getattr(L, f).restype = i32
        assert L.oracle_nout() == len(FIELDS)
        _lib = L
    return _lib


def _f32x4(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    assert a.ndim == 2 and a.shape[1] == 4
    return a


def _targets(targets):
    if targets is None:
        return None, 0
    t = np.ascontiguousarray(targets, dtype=np.int64)
    return t, t.size


def _ptr(a):
    return None if a is None else a.ctypes.data


def _as_dict(out):
    return {f: out[:, k].copy() for k, f in enumerate(FIELDS)}


def kernel(r, h, gamma):
    """(W, dW/dr, dW/dh) of the cubic spline at separation r, smoothing length h."""
    W, dr, dh = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().oracle_kernel(float(r), float(h), float(gamma), ctypes.byref(W), ctypes.byref(dr), ctypes.byref(dh))
    return W.value, dr.value, dh.value


def bruteforce(xyzh, vm, box=1.0, gamma=1.825742, targets=None):
    """O1: O(N^2) minimum-image density sums, fp64.  Returns dict of arrays."""
    xyzh, vm = _f32x4(xyzh), _f32x4(vm)
    t, nt = _targets(targets)
    n = xyzh.shape[0]
    out = np.zeros((nt if t is not None else n, len(FIELDS)), np.float64)
    rc = lib().oracle_bruteforce(n, _ptr(xyzh), _ptr(vm), float(box), float(gamma), _ptr(t), nt, _ptr(out))
    if rc:
        raise RuntimeError(f"oracle_bruteforce failed ({rc})")
    return _as_dict(out)


def celllist(xyzh, vm, nc, box=1.0, gamma=1.825742, targets=None):
    """O2: plain cell list over the 27-cell block (Code 1), fp64."""
    xyzh, vm = _f32x4(xyzh), _f32x4(vm)
    t, nt = _targets(targets)
    n = xyzh.shape[0]
    out = np.zeros((nt if t is not None else n, len(FIELDS)), np.float64)
    rc = lib().oracle_celllist(n, _ptr(xyzh), _ptr(vm), float(box), float(gamma), int(nc), _ptr(t), nt, _ptr(out))
    if rc:
        raise RuntimeError(f"oracle_celllist failed ({rc})")
    return _as_dict(out)


def pv_counts(xyzh, nc, box=1.0, gamma=1.825742, delta=None, targets=None):
    """Code 2 as a count: per target and kind (self, face, edge, corner) the
    naive candidates, pseudo-Verlet candidates and in-range hits.
    Returns (counts[nt, 4, 3] int64, unsafe) where unsafe must be 0."""
    xyzh = _f32x4(xyzh)
    t, nt = _targets(targets)
    n = xyzh.shape[0]
    if delta is None:
        delta = DELTA_FRAC * box / nc
    m = nt if t is not None else n
    out = np.zeros((m, 4, 3), np.int64)
    unsafe = ctypes.c_int64(0)
    rc = lib().oracle_pv_counts(n, _ptr(xyzh), float(box), float(gamma), int(nc), float(delta), _ptr(t), nt,
                                _ptr(out), ctypes.addressof(unsafe))
    if rc:
        raise RuntimeError(f"oracle_pv_counts failed ({rc})")
    return out, unsafe.value


def bin_cells(xyzh, nc, box=1.0):
    """Cell of every particle, stable cell-sorted order and cell starts."""
    xyzh = _f32x4(xyzh)
    n = xyzh.shape[0]
    cell = np.zeros(n, np.int64)
    order = np.zeros(n, np.int64)
    start = np.zeros(nc ** 3 + 1, np.int64)
    rc = lib().oracle_bin_cells(n, _ptr(xyzh), float(box), int(nc), _ptr(cell), _ptr(order), _ptr(start))
    if rc:
        raise RuntimeError(f"oracle_bin_cells failed ({rc})")
    return cell, order, start


def cell_keys(xyzh, nc, box=1.0):
    """keys[13, N]: fp64 cell-local projection of every particle on the 13 unit sort axes."""
    xyzh = _f32x4(xyzh)
    n = xyzh.shape[0]
    keys = np.zeros((13, n), np.float64)
    rc = lib().oracle_cell_keys(n, _ptr(xyzh), float(box), int(nc), _ptr(keys))
    if rc:
        raise RuntimeError(f"oracle_cell_keys failed ({rc})")
    return keys


def directions():
    o = np.zeros((13, 3), np.int32)
    lib().oracle_directions(_ptr(o))
    return o


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(t: int) -> None:
    lib().oracle_set_num_threads(int(t))
