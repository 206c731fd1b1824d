"""Tolerances of the GPU-vs-oracle comparison (readings R13-R15).

* rho, wcount (all terms positive):  |gpu - oracle| <= 1e-5 * oracle
* rho_dh, wcount_dh, div_v, curl_v (signed, can cancel):
      |gpu - oracle| <= 1e-4 * A_i,  A_i = sum_j |term_ij| (oracle, same normalisation)
  and for div_v, curl_v additionally + 2^-22 * C_i, C_i = sum_j |term_ij| (|x w''/w'| + 1),
  the first-order effect of a 4-ulp (x in [1/2, 1)) fp32 rounding of x = r/H (reading R14);
  the report counts the particles that pass ONLY because of that term (`r14_active`);
* nngb: |gpu - oracle| <= band_i, band_i = #{j : |r^2 - H_i^2| < 1e-6 H_i^2}
  (BASELINE north_star: exact except for pairs in that band).
"""
import json
import os

import numpy as np

TOL_POS = 1e-5
TOL_SIGNED = 1e-4
EPS_X = 2.0 ** -22


def compare(gpu: dict, ref: dict, idx=None, label: str = "") -> dict:
    """gpu: dict of arrays over all particles (input order); ref: oracle dict for the
    particles idx (all if None).  Raises AssertionError with a report; returns the report."""
    sel = (lambda a: a) if idx is None else (lambda a: a[idx])
    rep = {}
    r14 = np.zeros(len(ref["rho"]), bool)
    for f in ("rho", "wcount"):
        err = np.abs(sel(gpu[f]).astype(np.float64) - ref[f]) / ref[f]
        rep[f] = float(err.max()) if err.size else 0.0
    for f, a, c in (("rho_dh", "a_rho_dh", None), ("wcount_dh", "a_wcount_dh", None), ("div_v", "a_div", "c_div"),
                    ("curl_x", "a_curl", "c_curl"), ("curl_y", "a_curl", "c_curl"), ("curl_z", "a_curl", "c_curl")):
        scale = ref[a] + (EPS_X / TOL_SIGNED) * ref[c] if c else ref[a]
        scale = np.where(scale > 0, scale, 1.0)
        diff = np.abs(sel(gpu[f]).astype(np.float64) - ref[f])
        err = diff / scale
        rep[f] = float(err.max()) if err.size else 0.0
        if c:
            plain = np.where(ref[a] > 0, ref[a], 1.0)
            r14 |= (diff > TOL_SIGNED * plain) & (err <= TOL_SIGNED)
    dn = np.abs(sel(gpu["nngb"]).astype(np.int64) - ref["nngb"].astype(np.int64))
    bad = dn > ref["band"].astype(np.int64)
    rep["nngb_mismatch_outside_band"] = int(bad.sum())
    rep["band_total"] = int(ref["band"].sum())
    rep["nngb_diff_total"] = int(dn.sum())
    rep["checked"] = int(ref["rho"].size)
    rep["r14_active"] = int(r14.sum())
    ok = (rep["rho"] <= TOL_POS and rep["wcount"] <= TOL_POS and rep["nngb_mismatch_outside_band"] == 0 and
          all(rep[f] <= TOL_SIGNED for f in ("rho_dh", "wcount_dh", "div_v", "curl_x", "curl_y", "curl_z")))
    log = os.environ.get("PVSPH_PARITY_LOG")
    if log:                                   # per-comparison record (DESIGN.md §5 table, R14 activation)
        with open(log, "a") as fh:
            fh.write(json.dumps({"label": label, "ok": bool(ok), **rep}) + "\n")
    assert ok, f"parity failure {label}: {rep}"
    return rep
