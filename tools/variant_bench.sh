#!/bin/bash
# time each libbssmppi_<name>.so variant at C3 / C1 / C5b with quick_bench-like loop
for n in "$@"; do
  echo "== $n"; BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_$n.so timeout 300 python tools/quick_bench.py 2>&1 | grep -E "^C(1|3|5b)"
done
