#!/bin/bash
# FMA sub-pipe balance of the C3 rollout kernel: which FMA-pipe metrics the
# device exposes, and the heavy / lite split of a launch.
#   tools/ncu_pipes.sh [name]   (libbssmppi_<name>.so; default the product library)
cd "$(dirname "$0")/.."
[ -n "$1" ] && export BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_$1.so
ncu --query-metrics 2>/dev/null | grep -iE "pipe_fma|pipe_fp|pipe_alu|pipe_xu|fmaheavy|fmalite|pipe_fp64|inst_executed_pipe" | awk '{print $1}' | sort -u > gpurun_out/pipe_metric_names.txt
wc -l gpurun_out/pipe_metric_names.txt
M=$(grep -E "^(sm__inst_executed_pipe_[a-z0-9_]+|sm__pipe_[a-z0-9_]+_cycles_active)$" gpurun_out/pipe_metric_names.txt | sed 's/$/.avg.pct_of_peak_sustained_active/' | paste -sd, -)
M2=$(grep -E "^sm__inst_executed_pipe_[a-z0-9_]+$" gpurun_out/pipe_metric_names.txt | sed 's/$/.sum/' | paste -sd, -)
ncu --metrics "$M,$M2,smsp__inst_executed.sum,gpu__time_duration.sum" --clock-control none -k regex:bss_rollout -s 1 -c 1 python tools/profile_iter.py --iters 2 2>&1 | grep -E "^\s+(smsp|sm__|gpu__)" | tee gpurun_out/pipes_c3.txt
