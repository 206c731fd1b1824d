"""Compile libpvsph.so (sm_100a only) in-tree with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libpvsph.so")
SRC = os.path.join(PKG, "csrc", "pvsph.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "--shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-diag-suppress", "128"]


def _sources():
    return glob.glob(os.path.join(PKG, "csrc", "*")) + [os.path.join(ROOT, "include", "sph.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = [NVCC, *NVCC_FLAGS, "-o", LIB, SRC]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            errs = [l for l in (r.stdout + r.stderr).splitlines() if "error" in l.lower()]
            raise RuntimeError("nvcc failed:\n" + "\n".join(errs[:40]))
        with open(os.path.join(PKG, "csrc", "ptxas_info.txt"), "w") as f:
            f.write(r.stderr)
        if verbose:
            print(r.stderr)
    return LIB
