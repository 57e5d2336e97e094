"""Markdown summary of the rollout kernel from an `ncu --set full` report.

    python tools/ncu_summary.py rep.ncu-rep <particle-steps> "<title>" "<command>" > profiles/...md
"""

import csv
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
]
STALLS = ["wait", "not_selected", "selected", "math_pipe_throttle", "dispatch_stall", "short_scoreboard",
          "branch_resolving", "no_instruction", "mio_throttle", "long_scoreboard"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main():
    rep, units, title, cmd = sys.argv[1], float(sys.argv[2]), sys.argv[3], sys.argv[4]
    v, u = raw(rep)
    print(f"# {title}\n")
    print(f"Command: `{cmd}` (B200, driver 580.159).\n")
    print("| metric | value |\n|---|---|")
    for m in METRICS:
        if m in v:
            print(f"| `{m}` | {v[m]} {u.get(m, '')} |")
    print("\nWarp stall reasons (warps per issue-active cycle):\n")
    print("| reason | ratio |\n|---|---|")
    for s in STALLS:
        k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if k in v:
            print(f"| {s} | {v[k]} |")
    inst = float(v["smsp__inst_executed.sum"].replace(",", ""))
    rd = float(v["dram__bytes_read.sum"].replace(",", ""))
    wr = float(v["dram__bytes_write.sum"].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic = rd * scale.get(u["dram__bytes_read.sum"], 1) + wr * scale.get(u["dram__bytes_write.sum"], 1)
    print(f"\nDerived: {inst:.4g} warp-instructions x 32 / {units:.4g} particle-steps = "
          f"**{inst * 32 / units:.0f} lane-instructions per particle-step**; "
          f"DRAM traffic per launch {traffic:.0f} B.")


if __name__ == "__main__":
    main()
