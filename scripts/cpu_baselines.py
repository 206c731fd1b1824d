#!/usr/bin/env python
"""CPU baselines of SURVEY.md §8(d) beside bench.py's all-core cpu_baseline: the fp64 oracle's
cell-list pass (O2, Code-1 loops) on ONE thread for c1-c3 and on all cores, and the brute-force
O1 for c1 and c2, each as a median of repetitions (the paper's protocol is the median of 5,
P:220).  c3's one-thread O2 runs on a random sample of targets (the call still bins all N).
Rates are in-range interactions per second (the oracle's own neighbour counts / wall time).
Test infrastructure: runs the oracle only.  Prints one JSON object.

usage: python scripts/cpu_baselines.py [--reps 5]"""
import argparse
import json
import os
import platform
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def timed(fn, reps):
    ts, out = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), min(ts), max(ts), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    oracle.build()
    all_cores = oracle.num_threads()
    res = {"cpu_model": cpu_model(), "host_threads": os.cpu_count(), "oracle_threads_all": all_cores,
           "protocol": f"median of {args.reps} (min, max); fp64 oracle (oracle/oracle.c, gcc -O2)", "runs": []}
    rng = np.random.default_rng(11)
    for cfg in ("c1", "c2", "c3"):
        p = synth.make(cfg)
        targets, sample = None, "full pass"
        if cfg == "c3":
            targets = np.sort(rng.choice(p.n, 100_000, replace=False)).astype(np.int64)
            sample = "100000 random targets (binning of all N included)"
        for threads in (1, all_cores):
            oracle.set_num_threads(threads)
            reps = args.reps if (cfg != "c3" or threads > 1) else 3
            med, lo, hi, out = timed(lambda: oracle.celllist(p.xyzh, p.vm, p.nc, targets=targets), reps)
            inter = int(np.asarray(out["nngb"], dtype=np.int64).sum())
            res["runs"].append({"config": cfg, "variant": "O2 celllist", "threads": threads, "sample": sample,
                                "seconds": {"median": med, "min": lo, "max": hi}, "reps": reps,
                                "interactions": inter, "interactions_per_s": inter / med})
        if cfg in ("c1", "c2"):
            oracle.set_num_threads(1)
            reps = args.reps if cfg == "c1" else 1
            med, lo, hi, out = timed(lambda: oracle.bruteforce(p.xyzh, p.vm), reps)
            inter = int(np.asarray(out["nngb"], dtype=np.int64).sum())
            res["runs"].append({"config": cfg, "variant": "O1 brute force", "threads": 1, "sample": "full pass",
                                "pairs": p.n * (p.n - 1), "seconds": {"median": med, "min": lo, "max": hi},
                                "reps": reps, "interactions": inter, "interactions_per_s": inter / med})
    oracle.set_num_threads(all_cores)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
