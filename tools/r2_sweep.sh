mkdir -p gpurun_out
timeout 900 tools/ab_bench.sh 1 p1 p1mb5 p1mb3 > gpurun_out/ab2.log 2>&1
for g in 4 8 16; do BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_p1.so timeout 300 python tools/g_sweep.py 16384 256 50 $g; done > gpurun_out/gs.log 2>&1
for g in 8 16 32; do BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_p1.so timeout 300 python tools/g_sweep.py 2048 256 50 $g; done >> gpurun_out/gs.log 2>&1
cat gpurun_out/ab2.log gpurun_out/gs.log
