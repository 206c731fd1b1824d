#!/bin/bash
# Iteration helper for gpurun: [tests] + c3/c5 bench lines + optional ncu capture of the density kernel.
# usage: scripts/gpu_iter.sh TAG [tests] [c5] [ncu]
TAG=$1; shift
mkdir -p gpurun_out
for a in "$@"; do
  case $a in
    tests) timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log;;
  esac
done
timeout 300 python bench.py --config c3 --no-cpu --no-e2e > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err
for a in "$@"; do
  case $a in
    c5) timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err;;
    ncu) timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:k_density --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_$TAG python bench.py --config c3 --no-cpu --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_$TAG.log 2>&1;;
  esac
done
python - "$TAG" <<'PY'
import json, sys, glob
tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/bench_c*_{tag}.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "ms/step", round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d["stage_ms"].items()}, "frac", round(d["roofline"]["frac"], 4))
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-800:])
PY
