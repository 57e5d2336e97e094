"""Analyse gpurun_out/parity_dump.npz against the golden fixtures."""
import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from cases import CASES
from helpers import Inputs, moments_rel_err

d = np.load(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/parity_dump.npz')


def unpack(mom):
    mean = mom[..., :8].astype(float); up = mom[..., 8:].astype(float)
    cov = np.empty(mean.shape[:-1] + (4, 4)); q = 0
    for a in range(4):
        for b in range(a, 4):
            cov[..., a, b] = cov[..., b, a] = up[..., q]; q += 1
    return mean, cov


for c in CASES:
    name = c['name']
    inp = Inputs(name); g = inp.gold
    costs = d[name + '__costs']; ref = g['costs']; fin = np.isfinite(ref)
    rel = np.abs(costs[fin] - ref[fin]) / np.abs(ref[fin]) if fin.any() else np.zeros(1)
    line = f"{name:14s} cost rel max {rel.max():.2e} med {np.median(rel):.1e}"
    if name + '__mom' in d:
        # the test's own metric (tests/test_gpu_parity.py test_belief_moments)
        ks = g['ks']
        mean, cov = unpack(d[name + '__mom'][:, ks])
        alive = np.broadcast_to(np.isfinite(g['costs'][ks])[None, :], mean.shape[:2])
        floor = 1e-2 * np.abs(g['means']).max(axis=0, keepdims=True)
        em, ec = moments_rel_err(mean[alive], cov[alive], g['means'][alive], g['covs'][alive],
                                 floor=np.broadcast_to(floor, mean.shape)[alive])
        line += f" | mean {em:.2e} | cov {ec:.2e} (M={inp.M})"
    print(line)
