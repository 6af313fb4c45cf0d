#!/bin/bash
# Counter evidence for the dominant kernel itself: one
# steady-state ensemble_kernel launch of the default bench workload (C3,
# 296 slots, segment 3 after 3 warm-up launches), with the FP64 / DMMA pipe,
# issue, eligibility, stall and DRAM counters.  Runs the plain command first
# (the recipe's rule), then ncu on the same command line.
set -e
TAG=${1:-r02}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,\
sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,\
sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,\
sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,\
sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,\
sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_fp64_pred_on.sum,\
smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.per_cycle_active,\
smsp__warps_eligible.avg.per_cycle_active,smsp__warps_active.avg.per_cycle_active,\
smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_membar_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_selected_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,\
smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,\
l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__sass_inst_executed_op_shared_ld.sum,sm__sass_inst_executed_op_shared_st.sum,\
dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread
ncu --metrics $M --clock-control none -k regex:ensemble_kernel -s 3 -c 1 --csv \
    --log-file gpurun_out/${TAG}_ensemble_metrics.csv $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo done
