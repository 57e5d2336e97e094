#!/bin/bash
# Interleaved A/B timing of libbssmppi_<name>.so variants on one box:
#   tools/ab_bench.sh ROUNDS name ...
# Each round runs quick_bench.py once per variant (C1, C2, C3, C5a, C5b), so
# box drift affects every variant alike.
cd "$(dirname "$0")/.."
rounds=$1; shift
for r in $(seq "$rounds"); do
  for n in "$@"; do
    BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_$n.so timeout 300 python tools/quick_bench.py 2>&1 \
      | grep -E "^[CS]" | sed "s/^/$n r$r /"
  done
done
