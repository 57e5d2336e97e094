#!/bin/bash
# A/B of libbssmppi_<name>.so variants at the small shapes (the 8-GPU C3
# shard, C1, C2) and at C1 / C3 / C5 via variant_bench.sh:
#   bash tools/peel_bench.sh base candidate
for v in "$@" "$@"; do for shape in "2048 256 50" "256 32 20" "4096 128 40"; do
  BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_$v.so timeout 120 python tools/g_sweep.py $shape 2>&1 | tail -1 | sed "s/^/$v /"
done; done
bash tools/variant_bench.sh "$@"
