"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/sph.h declares, and the host-side argument checks work."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sph.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1804_06231_b200 import _build, _lib
    _build.build()
    return _lib.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(sph_[a-z_]+)\s*\(", src, flags=re.M)))


def test_header_declares_the_five_calls():
    names = declared_functions()
    for f in ("sph_build_cells", "sph_sort_cells", "sph_density_self", "sph_density_pair", "sph_density_all"):
        assert f in names


def test_library_exports_every_declared_symbol(lib):
    from paper_1804_06231_b200 import _lib
    names = declared_functions()
    assert set(names) == set(_lib.EXPORTS)
    for f in names:
        assert hasattr(lib, f), f


def test_library_is_sm100a_only():
    from paper_1804_06231_b200 import _build
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def test_abi_version_and_strerror(lib):
    assert lib.sph_abi_version() == 7
    for code in range(6):
        assert len(lib.sph_strerror(code)) > 0


def _grid(nc=(4, 4, 4), box=1.0, x_lo=0, x_hi=None, ghost=0, gamma=1.825742, skin=0.0):
    from paper_1804_06231_b200.api import make_grid
    return make_grid(nc, box, gamma, x_lo, x_hi, ghost, skin=skin)


def test_grid_validation(lib):
    g = _grid()
    assert lib.sph_ncell(ctypes.byref(g)) == 64
    assert lib.sph_ncell(ctypes.byref(_grid(nc=(2, 4, 4)))) < 0          # nc < 3
    assert lib.sph_ncell(ctypes.byref(_grid(x_lo=1, x_hi=3))) < 0        # partial slab needs ghosts
    assert lib.sph_ncell(ctypes.byref(_grid(x_lo=1, x_hi=3, ghost=1))) == 4 * 16
    assert lib.sph_ncell(ctypes.byref(_grid(nc=(8, 4, 4), x_lo=0, x_hi=7, ghost=1))) < 0   # ghost planes coincide
    assert lib.sph_ncell(ctypes.byref(_grid(gamma=0.0))) < 0
    assert lib.sph_ncell(ctypes.byref(_grid(skin=0.01))) == 64                 # list reuse margin
    assert lib.sph_ncell(ctypes.byref(_grid(skin=-0.01))) < 0
    assert lib.sph_ncell(ctypes.byref(_grid(skin=0.125))) < 0                  # 2 skin >= C_l
    assert lib.sph_workspace_bytes(ctypes.byref(g), 1000) > 8000
    assert lib.sph_workspace_bytes(ctypes.byref(_grid(nc=(1, 4, 4))), 10) == 0


def test_host_argument_errors_return_einval(lib):
    from paper_1804_06231_b200 import _lib
    g = _grid()
    cells = _lib.SphCells()          # all-null pointers
    assert lib.sph_build_cells(ctypes.byref(g), 10, 0, None, None, ctypes.byref(cells), None, 0, None) == 1
    assert lib.sph_sort_cells(ctypes.byref(g), ctypes.byref(cells), 0, -1, None, 0, None) == 1
    out = _lib.SphOut()
    assert lib.sph_density_all(ctypes.byref(g), ctypes.byref(cells), ctypes.byref(out), None, None, 0, None) == 1
    assert lib.sph_density_self(None, ctypes.byref(cells), None, 0, ctypes.byref(out), None, None, 0, None) == 1
    assert lib.sph_density_pair(ctypes.byref(g), None, None, 0, ctypes.byref(out), None, None, 0, None) == 1
    assert lib.sph_density_pair_sym(ctypes.byref(g), None, None, 0, ctypes.byref(out), None, None, 0, None) == 1
    assert lib.sph_density_finalize(ctypes.byref(out), 5, None) == 1
    assert lib.sph_status(None, None) == 1


def test_capacity_error_is_host_side(lib):
    """n_own + n_ghost > capacity returns SPH_ECAPACITY before touching the device."""
    from paper_1804_06231_b200 import _lib
    g = _grid()
    c = _lib.SphCells()
    c.capacity = 4
    fake = 256   # aligned non-null fake device addresses: never dereferenced on this path
    c.cell_start = c.xyzh = c.vm = c.perm = c.cell_hmax = c.order = c.slot_cell = c.cell_nhome = fake
    c.disp = c.cell_dx = fake
    assert lib.sph_build_cells(ctypes.byref(g), 5, 0, ctypes.c_void_p(fake), ctypes.c_void_p(fake),
                               ctypes.byref(c), ctypes.c_void_p(fake), 1 << 30, None) == 3
    assert lib.sph_build_cells(ctypes.byref(g), 2, 1, ctypes.c_void_p(fake), ctypes.c_void_p(fake),
                               ctypes.byref(c), ctypes.c_void_p(fake), 1 << 30, None) == 1   # ghosts w/o ghost_x
