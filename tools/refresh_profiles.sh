# Full GPU refresh of the measured evidence (one gpurun call):
#   bench lines (C3, C4, reference arm), the C5/C1/C2 sweep, the shard
#   projection, the C2 closed loops, the ncu launch list and the --set full
#   capture of the C3 rollout kernel.  Outputs land in gpurun_out/r_*.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r_bench_c3.json 2> gpurun_out/r_bench_c3.err
python bench.py --workload C4 > gpurun_out/r_bench_c4.json 2> gpurun_out/r_bench_c4.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r_bench_ref.json 2> gpurun_out/r_bench_ref.err
bash tools/c5_sweep.sh > gpurun_out/r_sweep.jsonl 2> gpurun_out/r_sweep.err
python tools/shard_sizes.py C3 C4 C5:131072:512 C5:32768:256 C5:4096:64 C2 > gpurun_out/r_shard.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r_launches_c3.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r_ncu_launch.log 2>&1
# the report itself stays on the box (the full library's source import is
# tens of MB): the summary and the source page travel back
ncu --set full --clock-control none --import-source on -k regex:bss_rollout -s 1 -c 1 -o /tmp/r_prof_c3 python tools/profile_iter.py --iters 2 > gpurun_out/r_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/r_prof_c3.ncu-rep 209715200 \
  "${P:-r2} ncu summary — bss_rollout_kernel<8,false,false> (G=8: 4 rollouts per warp, 32 particles per lane), C3 (K=16384, M=256, T=50)" \
  "ncu --set full --clock-control none --import-source on -k regex:bss_rollout -s 1 -c 1 python tools/profile_iter.py --iters 2" \
  > gpurun_out/r_ncu_c3.md
ncu -i /tmp/r_prof_c3.ncu-rep --page source --csv --print-source sass > gpurun_out/r_src_c3.csv 2> /dev/null
python tools/closed_loop_c2.py --oracle --out gpurun_out/r_closed_loop_c2.json > gpurun_out/r_closed_loop.log 2>&1
tail -c 400 gpurun_out/r_bench_c3.json
