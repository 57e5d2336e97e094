"""Dump GPU rollout costs + moments for every golden case (oracle-noise
mode) into gpurun_out/parity_dump.npz for analysis in the build container."""
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
        costs, mom = _gpu_rollout(inp, moments=True)
        out[c["name"] + "__mom"] = mom
    else:
        costs = _gpu_rollout(inp)
    out[c["name"] + "__costs"] = costs
np.savez_compressed(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_dump.npz", **out)
print("dumped", len(out))
