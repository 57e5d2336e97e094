#!/bin/bash
# Key rollout-kernel counters for each libbssmppi_<name>.so variant (C3).
M=smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,gpu__time_duration.sum
for n in "$@"; do
  echo "== $n"
  BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_$n.so ncu --metrics $M --clock-control none -k regex:bss_rollout -s 1 -c 1 python tools/profile_iter.py --iters 2 2>&1 | grep -E "^\s+(smsp|sm__|gpu__)" 
done
