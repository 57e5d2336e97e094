#!/bin/bash
# Key rollout-kernel counters of each libbssmppi_<name>.so variant at C3 on a
# LATE iteration (the 30th control step on the fixed state: the warm-started
# plan has drifted to the regime quick_bench / bench.py time).
M=smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__thread_inst_executed_per_inst_executed.ratio,gpu__time_duration.sum
for n in "$@"; do
  echo "== $n"
  BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_$n.so ncu --metrics $M --clock-control none -k regex:bss_rollout -s 29 -c 1 python tools/profile_iter.py --iters 31 2>&1 | grep -E "^\s+(smsp|sm__|gpu__|l1tex)"
done
