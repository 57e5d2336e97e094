"""Print the headline numbers of profiles/r1_* (for DESIGN.md / README.md)."""
import collections
import csv
import json
import subprocess
import sys

sys.path.insert(0, ".")


def line(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


for name in ("c3", "c4"):
    d = line(f"profiles/r1_bench_{name}.json")
    r = d["roofline"]
    print(f"{name}: {d['ms_per_step']:.3f} ms  {d['value'] / 1e9:.1f} G/s  e2e {d['e2e']['ms_per_step']:.3f} ms "
          f"{d['e2e']['value'] / 1e9:.1f} G/s  rollout {r['rollout_ms']:.3f} ms  sfu {r['sfu']['frac']:.3f} "
          f"fp32 {r['fp32']['frac']:.3f} ({r['fp32']['achieved']:.1f} TF/s, {r['sfu']['achieved']:.2f} Tops/s)  "
          f"cpu {d.get('cpu_baseline', {}).get('value', 0) / 1e6:.1f} M/s")
ref = line("profiles/r1_bench_reference_arm.json")
print(f"reference arm: {ref['value'] / 1e6:.1f} M/s")
for l in open("profiles/r1_sweep_c5_c1_c2.jsonl"):
    d = json.loads(l)
    print(f"  {d['config']['workload'].split(':')[0]:14s} K={d['config']['K']:6d} M={d['config']['M']:3d} "
          f"{d['ms_per_step']:.3f} ms {d['value'] / 1e9:.1f} e2e {d['e2e']['value'] / 1e9:.1f}")
for d in json.load(open("profiles/r1_shard_projection.json")):
    print(f"  shard {d['workload']:14s} N={d['n_gpus']} {d['device_ms']:.3f} ms eff {d['efficiency'] * 100:.0f}%")
cl = json.load(open("profiles/r1_closed_loop_c2.json"))
for r in cl["runs"]:
    g, o = r["gpu"], r["oracle"]
    print(f"  C2 seed {r['seed']}: p50 {g['latency_ms_p50']:.3f} ms dev {g['device_ms_p50']:.3f}; viol {g['violation_rate']} / "
          f"{o['violation_rate']}; speed {g['mean_speed']:.4f} / {o['mean_speed']:.4f}")
rows = [r for r in csv.reader(open("profiles/r1_launches_c3.csv")) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
t = collections.defaultdict(list)
for r in rows[1:]:
    try:
        t[r[ki][:40]].append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
for k, v in t.items():
    print(f"  launch {k:40s} n={len(v)} mean {sum(v) / len(v) / 1e3:.1f} us")
