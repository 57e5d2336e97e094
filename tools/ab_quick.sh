#!/bin/bash
# One GPU call for an A/B round: interleaved quick_bench timing of the given
# libbssmppi_<name>.so variants, then the key ncu counters of each at C3.
#   tools/ab_quick.sh ROUNDS name ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rounds=$1; shift
timeout 1200 tools/ab_bench.sh "$rounds" "$@" > gpurun_out/ab.log 2>&1
timeout 900 tools/ncu_ab.sh "$@" > gpurun_out/ncu_ab.log 2>&1
cat gpurun_out/ab.log; cat gpurun_out/ncu_ab.log
