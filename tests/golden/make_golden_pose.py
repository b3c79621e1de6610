"""Golden vectors for pose refinement, by running the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_golden_pose.py

The "small" case of make_golden.py (sphere-in-box, 6 frames 32x24, 4 levels,
48 rays x 132 samples) with ``refine_poses=True`` (frame 0 frozen,
gs/optimizer.py:203) and ``pose_refresh_every=2``, trained for 4 iterations
through the reference's own loop body (gs/optimizer.py:362-376): draw,
train_objective, dc.grad, Adam.step, refresh.  Iteration 0 runs at nu = 0
(series branch of exp_so3), later iterations at |nu| > 1e-4 (closed form),
and the refresh after iterations 1 and 3 folds nu into R0.

Stored per iteration: loss parts, extras, every gradient (the case is small:
all tensors whole), and after the last iteration every parameter, R0, nu, t.
"""

from __future__ import annotations

import json
import os

import numpy as np

from gridsurf import diffcore as dc
from gridsurf import optimizer, renderer, sampler, scenegen, seeds
from gridsurf.camera import Intrinsics

HERE = os.path.dirname(os.path.abspath(__file__))
ITERS = 4


def main():
    f = 0.5 * 32 / np.tan(np.radians(35.0))
    intr = Intrinsics(fx=f, fy=f, cx=16.0, cy=12.0, width=32, height=24)
    ds = scenegen.render_dataset(scenegen.sphere_in_box(), scenegen.orbit_trajectory(6), intr,
                                 max_t=8.0, seed=0)
    colors_u8 = np.round(ds.colors * 255.0).astype(np.uint8)
    depths_u16 = np.round(ds.depths * 1000.0).astype(np.uint16)
    assert np.array_equal(colors_u8.astype(np.float64) / 255.0, ds.colors)
    assert np.array_equal(depths_u16.astype(np.float64) / 1000.0, ds.depths)
    case = dict(seed=3, batch_rays=48, voxel_sizes=(0.96, 0.48, 0.24, 0.16), refine_poses=True,
                pose_refresh_every=2)
    for precision in ("double", "single"):
        cfg = optimizer.TrainConfig(precision=precision, **case)
        cfg.weights.smooth_count = 256
        dc.set_finite_checks(precision == "double")
        model = optimizer.build_model(ds, cfg, skip_init=True)
        opt = optimizer.make_optimizer(model, cfg)
        names = optimizer._param_names(model)
        arrays = dict(colors_u8=colors_u8, depths_u16=depths_u16, poses=ds.poses)
        for n, p in zip(names, model.parameters()):
            arrays[f"init_{n}"] = p.data.copy()
        meta = dict(precision=precision, intr=[f, f, 16.0, 12.0, 32, 24], names=names,
                    cfg={k: (list(v) if isinstance(v, tuple) else v) for k, v in case.items()},
                    smooth_count=256, iters=ITERS, parts=[], extras=[],
                    lo=list(map(float, model.grid.lo)), hi=list(map(float, model.grid.hi)))
        for it in range(ITERS):
            batch = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, it), cfg.batch_rays,
                                           near=cfg.near, far=cfg.max_depth)
            total, parts, extras = renderer.train_objective(model, ds, batch, it, cfg)
            grads = dc.grad(total, opt.params)
            for n, g in zip(names, grads):
                arrays[f"it{it}_grad_{n}"] = g.data.copy()
            arrays[f"it{it}_depths"] = extras["depths"]
            meta["parts"].append({k: float(v) for k, v in parts.items()})
            meta["extras"].append({k: (int(v) if isinstance(v, (int, np.integer, bool, np.bool_))
                                       else float(v))
                                   for k, v in extras.items() if k not in ("depths", "weights")})
            opt.step(grads)
            if cfg.refine_poses and (it + 1) % cfg.pose_refresh_every == 0:
                for p in model.poses:
                    p.refresh()
        for n, p in zip(names, model.parameters()):
            arrays[f"final_{n}"] = p.data.copy()
        arrays["final_R0"] = np.stack([p.R0 for p in model.poses])
        arrays["final_nu"] = np.stack([np.asarray(p.nu.data, dtype=np.float64) for p in model.poses])
        arrays["final_t"] = np.stack([np.asarray(p.t.data, dtype=np.float64) for p in model.poses])
        arrays["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
        path = os.path.join(HERE, f"pose_small_{precision}.npz")
        np.savez_compressed(path, **arrays)
        pg = {n: arrays[f"it0_grad_{n}"] for n in names if n[:2] in ("nu", "t1", "t2")}
        print(path, os.path.getsize(path) / 1e6, "MB", meta["parts"][0], {k: v[:2] for k, v in pg.items()})


if __name__ == "__main__":
    main()
