#!/bin/bash
# iteration helper: gpu tests (v5 default) + bench c3/c5 lines for v5 and v4
TAG=$1; shift
mkdir -p gpurun_out
export PVSPH_PARITY_LOG=gpurun_out/parity_$TAG.jsonl
rm -f $PVSPH_PARITY_LOG
if [[ " $* " == *" tests "* ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
fi
for C in c3 c5; do
  timeout 300 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err; echo "bench $C rc=$?"
done
if [[ " $* " == *" v4 "* ]]; then
  PVSPH_ENGINE=v4 timeout 300 python bench.py --config c5 --no-cpu --no-e2e > gpurun_out/bench_c5v4_$TAG.json 2> gpurun_out/bench_c5v4_$TAG.err
fi
python - "$TAG" <<'PY'
import json, sys, glob
tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/bench_c*_{tag}.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "ms/step", round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d["stage_ms"].items()}, "frac", round(d["roofline"]["frac"], 4))
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-1500:])
PY
