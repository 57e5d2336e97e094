#!/bin/bash
# Build libbssmppi variants for A/B timing: name:flags
# (-DBSS_AB_ONLY: only the Philox re-projection kernels with the diagonal
# process noise and the short tire sine -- what tools/quick_bench.py runs --
# so a variant builds in well under a minute; persist / oracle-noise calls
# fail with cudaErrorNotSupported)
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -Xptxas -v -DBSS_AB_ONLY -I include $flags \
    paper_2408_00494_b200/csrc/bssmppi.cu -o paper_2408_00494_b200/libbssmppi_$name.so 2> /tmp/ptx_$name.log &
done
wait
for spec in "$@"; do name="${spec%%:*}"; echo "$name: $(grep -A2 'ILi8ELb0ELb0ELi128' /tmp/ptx_$name.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"; done
