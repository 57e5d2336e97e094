"""Static SASS census of one kernel: loops (backward branches), and for a
chosen loop the opcode and source-line histograms.

    nvdisasm -g <cubin> > all.sass
    python tools/sass_census.py all.sass <mangled-kernel> [loop-index]
"""

import collections
import re
import sys

INS = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)(.*);")
LINE = re.compile(r'//## File "([^"]+)", line (\d+)')
LABEL = re.compile(r"^(\.L_x_\d+):")


def parse(path, fn):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{fn}:"))
    ins, labels, src = [], {}, None
    for l in lines[start + 1:]:
        if l.startswith(".text.") or l.startswith("//------"):
            break
        m = LABEL.match(l)
        if m:
            labels[m.group(1)] = len(ins)
            continue
        m = LINE.search(l)
        if m:
            src = f"{m.group(1).rsplit('/', 1)[-1]}:{m.group(2)}"
            continue
        m = INS.search(l)
        if m:
            ins.append((m.group(3), m.group(4), src))
    return ins, labels


def main():
    path, fn = sys.argv[1], sys.argv[2]
    pick = int(sys.argv[3]) if len(sys.argv) > 3 else None
    ins, labels = parse(path, fn)
    loops = []
    for i, (op, rest, _) in enumerate(ins):
        if op.startswith("BRA"):
            m = re.search(r"`\((\.L_x_\d+)\)", rest)
            if m and labels.get(m.group(1), i + 1) <= i:
                loops.append((labels[m.group(1)], i))
    print(f"{fn}: {len(ins)} instructions")
    for j, (a, b) in enumerate(loops):
        mufu = sum(1 for op, _, _ in ins[a:b + 1] if op.startswith("MUFU"))
        print(f"  loop {j}: [{a}, {b}] {b - a + 1} instructions, {mufu} MUFU")
    if pick is None:
        return
    a, b = loops[pick]
    body = ins[a:b + 1]
    ops = collections.Counter(op.split(".")[0] for op, _, _ in body)
    print("opcodes:", ", ".join(f"{k} {v}" for k, v in ops.most_common()))
    srcs = collections.Counter(s for _, _, s in body)
    for s, n in srcs.most_common(60):
        print(f"  {n:4d}  {s}")


if __name__ == "__main__":
    main()
