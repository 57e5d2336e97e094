mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:bss_rollout -s 1 -c 1 -o /tmp/s8_full python tools/profile_iter.py --K 2048 --iters 2 > gpurun_out/s8_full.log 2>&1
ncu -i /tmp/s8_full.ncu-rep --page source --csv --print-source sass > gpurun_out/s8_src.csv 2>/dev/null
ncu -i /tmp/s8_full.ncu-rep --page raw --csv > gpurun_out/s8_raw.csv 2>/dev/null
ls -la gpurun_out/s8_*
