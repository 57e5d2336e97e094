#!/bin/bash
# One-call GPU check: parity tests, parity dump, quick timing.
set -o pipefail
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/parity_dump.py gpurun_out/dump.npz > /dev/null 2>&1
timeout 300 python tools/quick_bench.py > gpurun_out/qb.log 2>&1
tail -6 gpurun_out/pytest_gpu.log; cat gpurun_out/qb.log
