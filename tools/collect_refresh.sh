#!/bin/bash
# Copy a tools/refresh_profiles.sh run (gpurun_out/r_*) into profiles/<P>_*
# (P = round prefix, default r2): bench lines, sweep, launch list, shard
# projection, closed loops, the ncu summary, the per-line instruction
# breakdown of the C3 rollout kernel and its FMA-pipe evidence
# (profiles/rollout_pipes.json, read by bench.py into roofline.fma_pipe).
set -e
cd "$(dirname "$0")/.."
P=${1:-r2}
tmp=$(mktemp -d)
(cd "$tmp" && cuobjdump -xelf all "$OLDPWD/paper_2408_00494_b200/libbssmppi.so" > /dev/null && nvdisasm -g bssmppi.sm_100a.cubin > all.sass)
# the C3 launch: G = 8, Philox noise, 128-thread blocks
K=$(grep -o '^\.text\._ZN3bss18bss_rollout_kernelILi8ELb0ELb0ELi128EEEvNS_10RollParamsE' "$tmp/all.sass" | head -1 | sed 's/^\.text\.//')
cp gpurun_out/r_ncu_c3.md profiles/${P}_rollout_ncu_c3.md
cp gpurun_out/r_src_c3.csv "$tmp/k.csv"
{ echo "# Executed lane-instructions per particle-step of bss_rollout_kernel<8,false,false> at C3, by SASS opcode and by CUDA source line"
  echo "# (ncu source page of r_prof_c3.ncu-rep joined with nvdisasm -g line info: python tools/sass_exec.py k.csv all.sass <kernel> 209715200)"
  python tools/sass_exec.py "$tmp/k.csv" "$tmp/all.sass" $K 209715200; } > profiles/${P}_rollout_lines_c3.txt
cp gpurun_out/r_bench_c3.json profiles/${P}_bench_c3.json
cp gpurun_out/r_bench_c4.json profiles/${P}_bench_c4.json
cp gpurun_out/r_bench_ref.json profiles/${P}_bench_reference_arm.json
cp gpurun_out/r_sweep.jsonl profiles/${P}_sweep_c5_c1_c2.jsonl
cp gpurun_out/r_launches_c3.csv profiles/${P}_launches_c3.csv
cp gpurun_out/shard_sizes.json profiles/${P}_shard_projection.json
cp gpurun_out/r_closed_loop_c2.json profiles/${P}_closed_loop_c2.json
dram=$(grep -E "dram__bytes_(read|write)" profiles/${P}_rollout_ncu_c3.md | sed -E 's/.*\| ([0-9.]+) (K?byte|Kbyte|byte) \|/\1 \2/' | awk '{v=$1; if ($2=="Kbyte") v*=1000; s+=v} END {print s}')
python - "$dram" <<'PY'
import json, sys
d = json.load(open("profiles/rollout_traffic.json"))
d["C3"] = float(sys.argv[1])
json.dump(d, open("profiles/rollout_traffic.json", "w"), indent=1)
PY
python tools/fma_cycles.py "$tmp/k.csv" "$tmp/all.sass" $K 209715200 > profiles/${P}_rollout_fma_cycles_c3.txt
python - "$P" <<'PY'
import json, re, sys
P = sys.argv[1]
md = open(f"profiles/{P}_rollout_ncu_c3.md").read()
def metric(name):
    m = re.search(r"`" + re.escape(name) + r"` \| ([0-9.]+)", md)
    return float(m.group(1)) if m else None
lines = open(f"profiles/{P}_rollout_lines_c3.txt").read()
fma = open(f"profiles/{P}_rollout_fma_cycles_c3.txt").read()
m = re.search(r"FMA-pipe cycles per particle-step \(warp\): ([0-9.]+)", fma)
m2 = re.search(r"\*\*([0-9.]+) lane-instructions per particle-step\*\*", md)
d = json.load(open("profiles/rollout_pipes.json")) if __import__("os").path.exists("profiles/rollout_pipes.json") else {}
d["C3"] = {"source": f"profiles/{P}_rollout_ncu_c3.md (ncu --set full, C3 rollout kernel)",
           "fma_pipe_active_pct": metric("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
           "issue_active_pct": metric("smsp__issue_active.avg.pct_of_peak_sustained_active"),
           "xu_pipe_pct": metric("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
           "lane_instructions_per_particle_step": float(m2.group(1)) if m2 else None,
           "fma_pipe_cycles_per_particle_step_per_warp": float(m.group(1)) if m else None}
json.dump(d, open("profiles/rollout_pipes.json", "w"), indent=1)
print(d["C3"])
PY
rm -rf "$tmp"
head -3 profiles/${P}_rollout_lines_c3.txt | tail -1
grep -E "dram__bytes|issue_active|fma_cycles|pipe_xu|registers" profiles/${P}_rollout_ncu_c3.md
