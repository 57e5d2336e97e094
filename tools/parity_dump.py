"""Dump GPU rollout costs + moments for every golden case (oracle-noise
mode) into gpurun_out/parity_dump.npz for analysis in the build container:
at the launch policy's lane-group width and at every forced width G in
{4, 8, 16, 32} (the widths the production shapes use)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from cases import CASES
from helpers import Inputs
from test_gpu_parity import _gpu_rollout

out = {}
for c in CASES:
    inp = Inputs(c["name"])
    if inp.kind == "bss":
        for g in (0, 4, 8, 16, 32):
            costs, mom = _gpu_rollout(inp, moments=True, group_width=g)
            out[f"{c['name']}__mom__g{g}"] = mom
            out[f"{c['name']}__costs__g{g}"] = costs
        out[c["name"] + "__mom"] = out[f"{c['name']}__mom__g0"]
    else:
        costs = _gpu_rollout(inp)
    out[c["name"] + "__costs"] = costs
np.savez_compressed(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_dump.npz", **out)
print("dumped", len(out))
