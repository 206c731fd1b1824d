#!/bin/bash
# Round-end measurement on one B200 (run under gpurun): bench lines for c5 (default), c3, c4,
# the c5 launch list (gpu__time_duration, cold-cache, serialised) and one --set full capture
# of the density kernel at c5.  Outputs under gpurun_out/$TAG_*; summarised here with
# scripts/ncu_summary.py, scripts/ncu_blocks.py and scripts/ncu_lines.py.
# usage: scripts/round_profile.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
echo "bench c5 rc=$?"
timeout 300 python bench.py --config c3 > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
echo "bench c3 rc=$?"
timeout 600 python bench.py --config c4 --no-cpu > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
echo "bench c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/${TAG}_launches_c5.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:k_density_v4 \
    --launch-skip 3 --launch-count 1 -o gpurun_out/${TAG}_prof_c5 \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_prof_c5.log 2>&1
echo "ncu full rc=$?"
