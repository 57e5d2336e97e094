mkdir -p gpurun_out
python tools/diag_case.py low_speed 0 > gpurun_out/diag.log 2>&1
BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_exact.so python tools/diag_case.py low_speed 0 >> gpurun_out/diag.log 2>&1
cat gpurun_out/diag.log
