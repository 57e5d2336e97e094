"""Reference statistics of the acceptance suite's closed-loop batches
(reference test_acceptance.py:37-57, 204-247), run with the REFERENCE
controller in the build container (minutes of CPU):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_acceptance.py [workers]

Writes tests/golden/acceptance_reference.json; tests/test_gpu_acceptance.py
compares the same batches run by the reference's own harness with this
repo's device Controller swapped in."""

import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

from belief_mppi import sim  # noqa: E402

from acceptance_spec import BATCHES, RUNS, config, key, summary  # noqa: E402

workers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
out = {"runs": RUNS, "generator": "reference belief_mppi.sim.monte_carlo (numba controller)", "batches": {}}
for b in BATCHES:
    t0 = time.time()
    rep = sim.monte_carlo(config(sim, b, workers=workers))
    out["batches"][key(b)] = summary(rep)
    print(f"{key(b)}: crash {rep.crash_ratio:.2f} sat {rep.mean_satisfaction:.3f} "
          f"({time.time() - t0:.0f} s)", flush=True)
(HERE / "acceptance_reference.json").write_text(json.dumps(out, indent=1))
