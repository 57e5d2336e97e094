set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r_bench_c3.json 2> gpurun_out/r_bench_c3.err
python bench.py --workload C4 > gpurun_out/r_bench_c4.json 2> gpurun_out/r_bench_c4.err
bash tools/c5_sweep.sh > gpurun_out/r_sweep.jsonl 2> gpurun_out/r_sweep.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r_launches_c3.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bss_rollout -s 1 -c 1 -o gpurun_out/prof_c3_v15 python tools/profile_iter.py --iters 2 > gpurun_out/ncu_v11.log 2>&1
tail -c 300 gpurun_out/r_bench_c3.json
