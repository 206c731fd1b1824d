"""Build a profiling variant of libpvsph.so with extra -D flags (gitignored exp/ directory);
used by the profiling helpers (phase_timing.py, v5_lane_stats.py), never by the product."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_variant(name: str, defines) -> str:
    from paper_1804_06231_b200 import _build
    out = os.path.join(ROOT, "exp", name)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = _build._sources()
    if os.path.exists(out) and all(os.path.getmtime(s) <= os.path.getmtime(out) for s in srcs):
        return out
    flags = [f for f in _build.NVCC_FLAGS if f not in ("-Xptxas", "-v")]
    cmd = [_build.NVCC, *flags, *[f"-D{d}" for d in defines], "-o", out, _build.SRC]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out
