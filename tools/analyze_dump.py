"""Analyse gpurun_out/parity_dump.npz against the golden fixtures."""
import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from cases import CASES
from helpers import Inputs

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
        ks = g['ks']
        mean, cov = unpack(d[name + '__mom'][:, ks])
        alive = np.cumprod(g['oks'][:, ks], axis=0).astype(bool)
        gm, gc = g['means'], g['covs']
        sig = np.sqrt(np.clip(np.diagonal(gc, axis1=-2, axis2=-1), 0, None))
        sub = [1, 2, 5, 6]
        scale = np.abs(gm).copy(); scale[..., sub] = np.maximum(scale[..., sub], sig)
        em = np.abs(mean - gm) / np.where(scale > 0, scale, 1); em[~alive] = 0
        i = np.unravel_index(np.argmax(em), em.shape)
        denom = np.sqrt(np.einsum('...i,...j->...ij', sig ** 2, sig ** 2))
        ec = np.abs(cov - gc) / np.where(denom > 0, denom, 1); ec[~alive] = 0
        j = np.unravel_index(np.argmax(ec), ec.shape)
        line += f" | mean {em[i]:.2e} @t{i[0]} c{i[2]} | cov {ec[j]:.2e} @t{j[0]} {j[2]}{j[3]}"
    print(line)
