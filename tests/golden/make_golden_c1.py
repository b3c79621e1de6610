"""Golden vectors at BASELINE configs[0] (c1), by running the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_golden_c1.py

c1 = sphere-in-box room, 20 RGB-D frames 160x120 (FOV 70, gs/cli.py:144-147),
default 4-level grid (0.96/0.24/0.06/0.03 m, derived bounds, P = 8.66 M),
M = 1024 rays, 96 + 3x12 samples, iteration 0, build_model(skip_init=True).

The full gradients (8.66 M per precision) are too large to commit, so each
tensor's gradient is stored as checksums (f64 sum, sum of squares, max |g|)
plus 4096 sampled entries at fixed indices; loss parts, extras, the sampled
depths and the rendering weights are stored whole.
"""

from __future__ import annotations

import json
import os

import numpy as np

from gridsurf import diffcore as dc
from gridsurf import optimizer, renderer, sampler, scenegen, seeds
from gridsurf.camera import Intrinsics

HERE = os.path.dirname(os.path.abspath(__file__))
NSAMP = 4096


def main():
    f = 0.5 * 160 / np.tan(np.radians(35.0))
    intr = Intrinsics(fx=f, fy=f, cx=80.0, cy=60.0, width=160, height=120)
    ds = scenegen.render_dataset(scenegen.sphere_in_box(), scenegen.orbit_trajectory(20), intr,
                                 max_t=8.0, seed=0)
    colors_u8 = np.round(ds.colors * 255.0).astype(np.uint8)
    depths_u16 = np.round(ds.depths * 1000.0).astype(np.uint16)
    assert np.array_equal(colors_u8.astype(np.float64) / 255.0, ds.colors)
    assert np.array_equal(depths_u16.astype(np.float64) / 1000.0, ds.depths)
    for precision in ("double", "single"):
        cfg = optimizer.TrainConfig(precision=precision, batch_rays=1024, seed=0)
        dc.set_finite_checks(precision == "double")
        model = optimizer.build_model(ds, cfg, skip_init=True)
        names = optimizer._param_names(model)
        it = 0
        batch = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, it), cfg.batch_rays,
                                       near=cfg.near, far=cfg.max_depth)
        total, parts, extras = renderer.train_objective(model, ds, batch, it, cfg)
        grads = dc.grad(total, list(model.parameters()))
        arrays = dict(colors_u8=colors_u8, depths_u16=depths_u16, poses=ds.poses,
                      depths=extras["depths"], weights=extras["weights"].data)
        rng = np.random.default_rng(123)
        for n, g in zip(names, grads):
            a = g.data.reshape(-1).astype(np.float64)
            idx = np.sort(rng.choice(a.size, size=min(a.size, NSAMP), replace=False)).astype(np.int64)
            arrays[f"gsum_{n}"] = np.array([a.sum(), (a * a).sum(), np.abs(a).max()])
            arrays[f"gidx_{n}"] = idx
            arrays[f"gval_{n}"] = a[idx]
        meta = dict(precision=precision, intr=[f, f, 80.0, 60.0, 160, 120], names=names,
                    parts={k: float(v) for k, v in parts.items()},
                    extras={k: (int(v) if isinstance(v, (int, np.integer, bool, np.bool_)) else float(v))
                            for k, v in extras.items() if k not in ("depths", "weights")},
                    lo=list(map(float, model.grid.lo)), hi=list(map(float, model.grid.hi)),
                    n_params=int(sum(p.data.size for p in model.parameters())))
        arrays["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
        path = os.path.join(HERE, f"c1_{precision}.npz")
        np.savez_compressed(path, **arrays)
        print(path, meta["parts"], meta["n_params"])


if __name__ == "__main__":
    main()
