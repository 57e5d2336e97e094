mkdir -p gpurun_out
for g in 4 8 16; do timeout 300 python tools/g_sweep.py 16384 256 50 $g; done > gpurun_out/gs2.log 2>&1
for b in 128 512; do BSSMPPI_FORCE_BLOCK=$b timeout 300 python tools/g_sweep.py 16384 256 50 8; done >> gpurun_out/gs2.log 2>&1
for b in 128 512; do BSSMPPI_FORCE_BLOCK=$b timeout 300 python tools/g_sweep.py 2048 256 50 32; done >> gpurun_out/gs2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bss_rollout -s 1 -c 1 -o /tmp/s8_full python tools/profile_iter.py --K 2048 --iters 2 > gpurun_out/s8_full.log 2>&1
ncu -i /tmp/s8_full.ncu-rep --page source --csv --print-source sass > gpurun_out/s8_src.csv 2>/dev/null
ncu -i /tmp/s8_full.ncu-rep --page raw --csv > gpurun_out/s8_raw.csv 2>/dev/null
cat gpurun_out/gs2.log
