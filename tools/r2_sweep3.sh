mkdir -p gpurun_out
bash tools/r2_check.sh
for g in 8 16 32; do timeout 300 python tools/g_sweep.py 4096 128 40 $g; done > gpurun_out/gs3.log 2>&1
cat gpurun_out/gs3.log
