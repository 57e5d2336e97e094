"""Executed-instruction breakdown of one kernel from an ncu report, joined
with nvdisasm line info of the same binary (instruction order matches).

    nvdisasm -g <cubin> > all.sass
    ncu -i rep.ncu-rep --page source --csv --print-source sass > k.csv
    python tools/sass_exec.py k.csv all.sass <mangled-kernel> <units>

Prints lane-instructions per unit by opcode and by CUDA source line.
"""

import collections
import csv
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_census import parse  # noqa: E402


def main():
    csv_path, sass_path, fn, units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    rows = list(csv.reader(open(csv_path)))
    hdr = next(r for r in rows if "Address" in r)
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    i_thr = hdr.index("Thread Instructions Executed")
    body = [r for r in rows[rows.index(hdr) + 1:] if len(r) > i_ex and r[0].startswith("0x")]
    ins, _ = parse(sass_path, fn)
    if len(ins) != len(body):
        print(f"warning: {len(ins)} disassembled vs {len(body)} profiled instructions")
    by_op, by_line, by_op_thr = collections.Counter(), collections.Counter(), collections.Counter()
    total = 0
    for j, r in enumerate(body):
        n = float(r[i_ex]) * 32.0 / units
        op = r[i_src].split()[0]
        if op.startswith("@"):
            op = r[i_src].split()[1]
        op = op.split(".")[0]
        by_op[op] += n
        by_op_thr[op] += float(r[i_thr]) / units
        total += n
        if j < len(ins):
            by_line[ins[j][2]] += n
    print(f"lane-instruction slots per unit: {total:.1f}")
    print("by opcode (slots, active-thread inst):")
    for k, v in by_op.most_common(40):
        print(f"  {v:7.2f}  {by_op_thr[k]:7.2f}  {k}")
    print("by source line:")
    for k, v in by_line.most_common(70):
        if v < 0.5:
            break
        print(f"  {v:7.2f}  {k}")
    # stall samples (all samples, per reason), by reason and by source line
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = {h: hdr.index(h) for h in reasons}
    tot = collections.Counter()
    line_r = collections.defaultdict(collections.Counter)
    for j, r in enumerate(body):
        src = ins[j][2] if j < len(ins) else "?"
        for h, i in idx.items():
            try:
                v = float(r[i])
            except ValueError:
                continue
            tot[h] += v
            line_r[src][h] += v
    allv = sum(tot.values())
    print("stall samples by reason:")
    for h, v in tot.most_common():
        if v > 0:
            print(f"  {100 * v / allv:5.1f}%  {h}")
    print("stall samples by source line (non-selected reasons):")
    busy = {k: sum(v for h, v in c.items() if h not in ("stall_selected", "stall_not_selected"))
            for k, c in line_r.items()}
    for k, v in sorted(busy.items(), key=lambda kv: -kv[1])[:40]:
        top = ", ".join(f"{h[6:]} {100 * n / allv:.1f}" for h, n in line_r[k].most_common(3)
                        if h not in ("stall_selected", "stall_not_selected"))
        print(f"  {100 * v / allv:5.1f}%  {k:24s} {top}")


if __name__ == "__main__":
    main()
