#!/bin/bash
# Round-2 measurement on one B200 (run under gpurun from the repo root).  Every ncu command
# runs only after the same command has exited 0 without ncu.  Outputs: gpurun_out/${TAG}_*;
# scripts/make_profile_r2.py TAG turns them into profiles/r2/.
# usage: scripts/round2_measure.sh TAG [notests]
TAG=${1:-r2f}
mkdir -p gpurun_out
O=gpurun_out/${TAG}
if [[ "$2" != "notests" ]]; then
  timeout 1500 python -m pytest tests -m gpu -q > ${O}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 ${O}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc=$?"
fi
# bench lines: the default (c5, cpu_baseline + e2e), c3, c4 (three level grids), the reuse loop,
# the symmetric whole pass, the reference arm
timeout 900 python bench.py > ${O}_bench_c5.json 2> ${O}_bench_c5.err; echo "bench c5 rc=$?"
timeout 600 python bench.py --config c3 > ${O}_bench_c3.json 2> ${O}_bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --config c4 > ${O}_bench_c4.json 2> ${O}_bench_c4.err; echo "bench c4 rc=$?"
timeout 900 python bench.py --reuse --no-cpu > ${O}_bench_reuse_c5.json 2> ${O}_bench_reuse_c5.err; echo "bench reuse rc=$?"
timeout 600 python bench.py --config c3 --engine sym --no-cpu --no-e2e > ${O}_bench_sym_c3.json 2> ${O}_bench_sym_c3.err; echo "bench sym rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > ${O}_bench_ref_c5.json 2> ${O}_bench_ref_c5.err; echo "bench ref rc=$?"
timeout 600 python bench_test27cells.py > ${O}_test27cells.json 2> ${O}_test27cells.err; echo "test27cells rc=$?"
timeout 300 python scripts/calibrate.py > ${O}_calib.json 2> ${O}_calib.err; echo "calibrate rc=$?"
timeout 900 python scripts/cpu_baselines.py > ${O}_cpu_baselines.json 2> ${O}_cpu_baselines.err; echo "cpu baselines rc=$?"
# measured FP32 counters of the density kernel (c3, c4, c5)
bash scripts/ncu_fp32.sh ${TAG} k_density_v5 c3 c4 c5
# the same counters summed over one symmetric whole pass at c3 (78 launches)
bash scripts/ncu_sym.sh ${TAG}
# c5 launch list with DRAM bytes per launch (cold-cache, serialised)
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > ${O}_launchplain.json 2>&1 &&
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file ${O}_launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e \
    > ${O}_launches_c5.log 2>&1
echo "launch list rc=$?"
timeout 300 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e > ${O}_launchplain_c4.json 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 600 --csv --log-file ${O}_launches_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-e2e \
    > ${O}_launches_c4.log 2>&1
echo "launch list c4 rc=$?"
# one --set full capture of the density kernel at c5
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name regex:k_density_v5 \
    --launch-skip 3 --launch-count 1 -o ${O}_prof_c5 \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > ${O}_prof_c5.log 2>&1
echo "ncu full rc=$?"
