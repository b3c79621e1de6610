"""Diagnose conditioned float32 per-sample mismatches (tests/test_f32_parity.py):
run a case several times and print the worst samples' details."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_f32_parity as F  # noqa: E402
from oracle import gridsurf_oracle as O  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
for rep in range(reps):
    r = F.run_case(case)
    M, N = r["M"], r["N"]
    dg = r["dev"]["gphi"][:M * N]
    og = r["R"]["gphi"].reshape(-1, 3)
    scale = np.abs(og).max()
    err = np.abs(dg - og).max(axis=1) / scale
    dphi = np.abs(r["dev"]["phi"][:M * N] - r["R"]["phi"].reshape(-1)) / np.abs(r["R"]["phi"]).max()
    worst = np.argsort(-err)[:6]
    print(f"rep {rep}: max gphi err {err.max():.3e}, n>1e-5: {(err > 1e-5).sum()}, max phi err {dphi.max():.3e}")
    xf = r["R"]["xf"]
    for s in worst:
        if err[s] <= 1e-5:
            break
        x = xf[s]
        locs = []
        model = r["model"]
        for lev in model.grid.levels:
            g = lev.geom
            loc = (x - g.origin) / g.voxel_size
            locs.append(np.round(loc - np.floor(loc), 8).tolist())
        print(f"  s={s} ray={s // N} j={s % N} err={err[s]:.3e} phi_err={dphi[s]:.2e} dev={dg[s]} ora={og[s]}"
              f" x={x.tolist()} fracs={locs}")
