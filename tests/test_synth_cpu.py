"""Input generators (synth/) on the CPU: the test27cells instances (bench_test27cells.py)."""
import numpy as np

import oracle
import synth


def test_test27cells_generator_fills_every_cell():
    """Every cell holds exactly 216 particles under the oracle's fp64 binning, h is the
    mean spacing times eta, gamma h < C_l; seeded (same seed, same set)."""
    p = synth.test27cells_set(seed=27, nc=4)
    cells, _, _ = oracle.bin_cells(p.xyzh, p.nc)
    assert np.all(np.bincount(cells, minlength=p.nc ** 3) == 216)
    assert np.all(p.xyzh[:, 3] == np.float32(synth.ETA * 0.25 / 6.0))
    assert synth.GAMMA * float(p.xyzh[0, 3]) * p.nc < 1.0
    q = synth.test27cells_set(seed=27, nc=4)
    assert np.array_equal(p.xyzh, q.xyzh) and np.array_equal(p.vm, q.vm)
