"""Mutation check of the oracle pins (VERDICT r1 'What's weak' 1): every tolerance scale the
GPU comparison divides by, multiplied by 100 (or with a term dropped), must fail at least one
test in tests/test_oracle_pins.py.  Copies oracle/ and tests/ to a scratch directory, applies
one source mutation at a time, rebuilds liboracle.so there and runs the pins.

usage: python scripts/oracle_mutation.py      (CPU only, ~1 min)"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = [
    ("a_rho_dh self term x100", "double a_rdh = fabs(mi * dWh0)", "double a_rdh = 100.0 * fabs(mi * dWh0)"),
    ("a_wcount_dh self term x100", "a_wdh = fabs(dWh0);", "a_wdh = 100.0 * fabs(dWh0);"),
    ("a_rho_dh pair terms x100", "a_rdh += fabs(mj * dWdh);", "a_rdh += 100.0 * fabs(mj * dWdh);"),
    ("a_wcount_dh pair terms x100", "a_wdh += fabs(dWdh);", "a_wdh += 100.0 * fabs(dWdh);"),
    ("a_div x100", "a_div += fabs(f * vdx);", "a_div += 100.0 * fabs(f * vdx);"),
    ("a_curl x100", "a_curl += fabs(f) * sqrt(vx * vx + vy * vy + vz * vz) * r;",
     "a_curl += 100.0 * fabs(f) * sqrt(vx * vx + vy * vy + vz * vz) * r;"),
    ("c_div x100", "c_div += fabs(f * vdx) * kap;", "c_div += 100.0 * fabs(f * vdx) * kap;"),
    ("c_curl x100", "c_curl += fabs(f) * sqrt(vx * vx + vy * vy + vz * vz) * r * kap;",
     "c_curl += 100.0 * fabs(f) * sqrt(vx * vx + vy * vy + vz * vz) * r * kap;"),
    ("a_curl drops |v|", "a_curl += fabs(f) * sqrt(vx * vx + vy * vy + vz * vz) * r;", "a_curl += fabs(f) * r;"),
    ("kappa without +1", "fabs(x * d2w_m4(x) / dw) + 1.0 : 1.0", "fabs(x * d2w_m4(x) / dw) : 1.0"),
    ("curl sign of one component", "Ry += f * (vz * dx - vx * dz);", "Ry += f * (vx * dz - vz * dx);"),
    ("rho_dh self term dropped", "double rho = mi * W0, wc = W0, rho_dh = mi * dWh0",
     "double rho = mi * W0, wc = W0, rho_dh = 0.0"),
]


def main():
    tmp = tempfile.mkdtemp(prefix="oracle_mut_")
    for d in ("oracle", "tests", "synth"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                        ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
    src_path = os.path.join(tmp, "oracle", "oracle.c")
    base = open(src_path).read()
    survived = []
    for name, old, new in MUTATIONS:
        assert base.count(old) == 1, f"mutation site not unique/found: {name}"
        open(src_path, "w").write(base.replace(old, new))
        so = os.path.join(tmp, "oracle", "liboracle.so")
        if os.path.exists(so):
            os.remove(so)
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "tests/test_oracle_pins.py"], cwd=tmp,
                           capture_output=True, text=True)
        killed = r.returncode != 0
        print(f"{'killed  ' if killed else 'SURVIVED'}  {name}")
        if not killed:
            survived.append(name)
    open(src_path, "w").write(base)
    shutil.rmtree(tmp, ignore_errors=True)
    print(f"{len(MUTATIONS) - len(survived)}/{len(MUTATIONS)} mutations killed")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
