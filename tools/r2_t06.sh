mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_acceptance.py -q -s -m gpu -k test_06 -p no:cacheprovider > gpurun_out/t06.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -5 gpurun_out/t06.log
