"""FMA-pipe cycles per particle-step (per warp) of the rollout kernel, by
CUDA source line: the executed opcodes of an ncu source page weighted by the
measured pipe occupancy (tools/microbench_pipes.cu: IMAD.WIDE 4, IMAD 2,
FFMA2/FMUL2/FADD2 2, FFMA/FMUL/FADD/HFMA2/FRND 1 cycle of one shared pipe).

    python tools/fma_cycles.py k.csv all.sass <mangled-kernel> <particle-steps>
"""
import collections
import csv
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_census import parse  # noqa: E402

W = {"FFMA2": 2, "FMUL2": 2, "FADD2": 2, "FFMA": 1, "FMUL": 1, "FADD": 1, "HFMA2": 1, "FRND": 1}


def main():
    csv_path, sass_path, fn, units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    rows = list(csv.reader(open(csv_path)))
    hdr = next(r for r in rows if "Address" in r)
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    body = [r for r in rows[rows.index(hdr) + 1:] if len(r) > i_ex and r[0].startswith("0x")]
    ins, _ = parse(sass_path, fn)
    by_line, by_op = collections.Counter(), collections.Counter()
    for j, r in enumerate(body):
        toks = r[i_src].split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        base = op.split(".")[0]
        w = W.get(base, 0)
        if base == "IMAD":
            w = 4 if ".WIDE" in op else 2
        c = float(r[i_ex]) * 32.0 / units * w
        by_line[ins[j][2] if j < len(ins) else None] += c
        by_op[base] += c
    print(f"FMA-pipe cycles per particle-step (warp): {sum(by_line.values()):.1f}")
    print("by opcode:", ", ".join(f"{k} {v:.1f}" for k, v in by_op.most_common() if v > 0.05))
    for k, v in by_line.most_common(30):
        print(f"  {v:6.2f}  {k}")


if __name__ == "__main__":
    main()
