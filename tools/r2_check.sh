# One-call GPU check: the -m gpu suite, smoke(), the default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rf -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_acceptance.py -q -s -m gpu -k test_06 -p no:cacheprovider 2>&1 | grep "acceptance 06" > gpurun_out/t06.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/t06.log; tail -2 gpurun_out/smoke.log; tail -c 300 gpurun_out/bench.log
