#!/bin/bash
# One-call GPU check: parity tests (no -x: every failure is listed), parity
# dump at the policy and forced lane-group widths, interleaved A/B timing of
# the given library variants (libbssmppi_<name>.so).
#   tools/gpu_check.sh [variant ...]
mkdir -p gpurun_out
python -m pytest tests -q -s -m gpu -rA 2>&1 | grep -E "PASSED|FAILED|ERROR|passed|failed|^K=|^  G=|moments|err" > gpurun_out/pytest_gpu.log
echo "pytest rc=${PIPESTATUS[0]}" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/parity_dump.py gpurun_out/dump.npz > gpurun_out/dump.log 2>&1
if [ $# -gt 0 ]; then timeout 900 tools/ab_bench.sh 2 "$@" > gpurun_out/ab.log 2>&1; fi
tail -5 gpurun_out/pytest_gpu.log; grep -E "FAILED|ERROR" gpurun_out/pytest_gpu.log | head -30; cat gpurun_out/ab.log 2>/dev/null
