#!/bin/bash
# Measured FP32 of the symmetric whole pass (sph_density_all_sym): the FP32 counters of every
# k_density_pair_sym launch of ONE pass at c3 (13 directions x 3 colours x 2 kernels), summed
# by scripts/parse_fp32.py parse_multi.  The plain command runs first (must exit 0).
# usage: scripts/ncu_sym.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
M=sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_ffma_pred_on.sum.peak_sustained,sm__cycles_elapsed.avg.per_second
M=$M,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
# bench: 1 counted + 3 warm-up passes before the timed one; 78 pair-kernel launches per pass at c3
timeout 300 python bench.py --config c3 --engine sym --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_symplain.json 2>&1 &&
timeout 900 ncu --metrics $M --clock-control none --kernel-name regex:k_density_pair_sym --launch-skip 312 --launch-count 78 \
    --csv --log-file gpurun_out/${TAG}_sym_fp32_c3.csv python bench.py --config c3 --engine sym --steps 1 --warmup 3 \
    --no-cpu --no-e2e > gpurun_out/${TAG}_sym_fp32.log 2>&1
echo "sym fp32 counters rc=$?"
