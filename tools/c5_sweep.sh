#!/bin/bash
# BASELINE config 5 sweep + C1/C2 single iterations (1 GPU); one JSON line each
for K in 4096 32768 131072; do for M in 64 256 512; do
  python bench.py --workload C5:$K:$M --steps 20 --warmup 3 --e2e-steps 5 --no-cpu-baseline
done; done
for w in C1 C2; do python bench.py --workload $w --steps 100 --warmup 5 --e2e-steps 50 --no-cpu-baseline; done
