#!/bin/bash
# Measured-FP32 roofline counters of the density kernel, one launch
# per config, under gpurun.  The plain command runs first (must exit 0) and only then ncu.
# usage: scripts/ncu_fp32.sh TAG [KERNEL_REGEX] [configs...]
TAG=${1:-r2}; KRE=${2:-k_density_v}; shift 2; CFGS=${@:-c3 c5}
mkdir -p gpurun_out
M=sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum
M=$M,sm__sass_thread_inst_executed_op_ffma_pred_on.sum.peak_sustained,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum.peak_sustained
M=$M,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum
M=$M,smsp__thread_inst_executed_per_inst_executed.ratio,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
M=$M,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
M=$M,smsp__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,gpu__time_duration.sum
M=$M,launch__registers_per_thread,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
for C in $CFGS; do
  timeout 600 python bench.py --config $C --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_fp32plain_$C.json 2>&1 &&
  timeout 900 ncu --metrics $M --clock-control none --kernel-name regex:$KRE --launch-skip 3 --launch-count 1 --csv \
      --log-file gpurun_out/${TAG}_fp32_$C.csv python bench.py --config $C --steps 1 --warmup 3 --no-cpu --no-e2e \
      > gpurun_out/${TAG}_fp32_$C.log 2>&1
  echo "fp32 counters $C rc=$?"
done
