"""Seeded synthetic particle sets (shared by the oracle tests and the CUDA path).

This package holds ONLY input generation (positions, smoothing lengths,
velocities, masses, the cell-grid size of each configuration).  It contains
none of the density method's arithmetic: no kernel, no neighbour search, no
sums.  Both `oracle/` and the CUDA path read what it produces; neither is
imported here.
"""
from .gen import (CONFIGS, GAMMA, ETA, ParticleSet, make, make_config,
                  uniform_set, lattice_set, clustered_set, tiny_random_set, test27cells_set)

__all__ = ["CONFIGS", "GAMMA", "ETA", "ParticleSet", "make", "make_config",
           "uniform_set", "lattice_set", "clustered_set", "tiny_random_set",
           "test27cells_set"]
