"""Aggregate an ncu source page (--print-source cuda,sass) per CUDA source
line: instructions executed per particle-step and stall-sample share."""
import csv, sys, subprocess
rep, units = sys.argv[1], float(sys.argv[2])     # units = particle-steps in the launch
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
items = []; path = None; hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": path = r[1].split('/')[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or r[0] == "" or r[0] == "Function Name": continue
    try:
        n = float(r[hdr.index("Instructions Executed")]); s = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except Exception:
        continue
    if n > 0 or s > 0: items.append((n, s, f"{path}:{r[0]}", r[1][:90]))
tot = sum(x[0] for x in items); tots = sum(x[1] for x in items)
print(f"total warp-inst {tot:.4g}  lane-inst per unit {tot*32/units:.1f}")
key = sys.argv[3] if len(sys.argv) > 3 else "inst"
for n, s, loc, src in sorted(items, key=lambda x: -(x[0] if key == "inst" else x[1]))[:int(sys.argv[4]) if len(sys.argv) > 4 else 50]:
    print(f"{n*32/units:7.2f} {100*s/tots:5.1f}%  {loc:22s} {src}")
