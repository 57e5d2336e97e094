# The GPU suite against the bounds-checked build (-DBSS_CHECKED: device
# asserts on array, table and noise indices).  Build it first (here):
#   nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a \
#     -Xcompiler -fPIC,-O2 -shared -DBSS_CHECKED -I include \
#     paper_2408_00494_b200/csrc/bssmppi.cu -o paper_2408_00494_b200/libbssmppi_checked.so
mkdir -p gpurun_out
BSSMPPI_LIB=$PWD/paper_2408_00494_b200/libbssmppi_checked.so timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -k "not acceptance" > gpurun_out/pytest_checked.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_checked.log
tail -4 gpurun_out/pytest_checked.log
