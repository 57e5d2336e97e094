#!/bin/bash
# Device time vs belief-kernel block size (BSSMPPI_FORCE_BLOCK) over shard
# and config shapes; the 128 / 512 rule in bssmppi.cu rollout_block_threads
# is fitted to it.
cd "$(dirname "$0")/.."
for shape in "256 32 20" "1024 256 50" "2048 256 50" "4096 128 40" "4096 64 60" "4096 256 50" \
             "8192 256 50" "16384 256 50" "8192 64 50" "16384 64 50" "4096 512 60" "2048 128 50"; do
  for b in 128 512; do
    echo -n "B=$b "; BSSMPPI_FORCE_BLOCK=$b timeout 120 python tools/g_sweep.py $shape 2>&1 | tail -1
  done
done
