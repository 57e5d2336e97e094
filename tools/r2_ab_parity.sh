#!/bin/bash
# One GPU call for a kernel variant: the full-size Philox parity tests
# (device vs the FP64 C oracle, the same counters) against
# libbssmppi_<new>.so, then interleaved A/B timing and the ncu counters of
# <base> and <new> (tools/ab_quick.sh).
#   tools/r2_ab_parity.sh ROUNDS base new
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rounds=$1; base=$2; new=$3
BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_$new.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider > gpurun_out/ab_parity.log 2>&1
tail -5 gpurun_out/ab_parity.log
tools/ab_quick.sh "$rounds" "$base" "$new"
