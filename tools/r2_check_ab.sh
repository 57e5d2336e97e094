bash tools/r2_check.sh
timeout 900 tools/ab_bench.sh 2 p1 tire > gpurun_out/ab3.log 2>&1
timeout 600 tools/ncu_ab.sh tire > gpurun_out/ncu_ab3.log 2>&1
grep -E "C3|S8|C2" gpurun_out/ab3.log
