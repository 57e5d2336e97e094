bash tools/r2_check.sh
timeout 900 tools/ab_bench.sh 2 opq mrg > gpurun_out/ab5.log 2>&1
grep -E "C3|S8|C2" gpurun_out/ab5.log
