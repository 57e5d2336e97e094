mkdir -p gpurun_out
BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_${1:-new}.so ncu --set full --clock-control none --import-source on -k regex:bss_rollout -s 1 -c 1 -o gpurun_out/${1:-new}_full python tools/profile_iter.py --iters 2 > gpurun_out/${1:-new}_full.log 2>&1
ncu -i gpurun_out/${1:-new}_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${1:-new}_src.csv 2>/dev/null
ncu -i gpurun_out/${1:-new}_full.ncu-rep --page raw --csv > gpurun_out/${1:-new}_raw.csv 2>/dev/null
ls -la gpurun_out
