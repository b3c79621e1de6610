"""Generate golden vectors by running the REFERENCE package (gridsurf).

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

For each case it renders the reference synthetic scene, builds the model
with the reference's own ``build_model(skip_init=True)``, runs two full
training iterations exactly as ``gs/optimizer.py:362-373`` does and stores:
the dataset (u8 colour / u16 depth, exactly the reference's quantisation),
poses, intrinsics, config, the first iteration's ray batch, per-round
importance inputs/outputs (recorded by wrapping the reference's sampler),
depths, weights, loss parts/extras, every parameter gradient, and the
parameters + Adam moments after the second iteration.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

from gridsurf import diffcore as dc
from gridsurf import optimizer, renderer, sampler, scenegen, seeds
from gridsurf.camera import Intrinsics

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # mirrors pkg/tests/test_renderer.py:11-26 (make_tiny)
    "tiny": dict(
        intr=(6.0, 6.0, 4.0, 3.0, 8, 6), frames=4, scene="sphere_in_box",
        cfg=dict(seed=0, batch_rays=8, coarse_samples=12, importance_rounds=1,
                 importance_add=4, voxel_sizes=(0.96, 0.48), geom_feat_dim=2,
                 color_feat_dim=2, fixed_far=2.0,
                 bounds=((-1.7, -1.7, -1.7), (1.7, 1.7, 1.3))),
        smooth_count=32, iteration=0),
    # full sampling schedule (96 + 3x12 = 132), 4 levels, default widths,
    # derived bounds, smoothness on
    "small": dict(
        intr=(0.5 * 32 / np.tan(np.radians(35.0)), 0.5 * 32 / np.tan(np.radians(35.0)),
              16.0, 12.0, 32, 24), frames=6, scene="sphere_in_box",
        cfg=dict(seed=3, batch_rays=48, voxel_sizes=(0.96, 0.48, 0.24, 0.16)),
        smooth_count=256, iteration=5),
}


def render(case):
    fx, fy, cx, cy, w, h = case["intr"]
    intr = Intrinsics(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))
    scene = getattr(scenegen, case["scene"])()
    traj = scenegen.orbit_trajectory(case["frames"])
    return scenegen.render_dataset(scene, traj, intr, max_t=8.0, seed=0)


def main():
    out_files = []
    for name, case in CASES.items():
        ds = render(case)
        colors_u8 = np.round(ds.colors * 255.0).astype(np.uint8)
        depths_u16 = np.round(ds.depths * 1000.0).astype(np.uint16)
        assert np.array_equal(colors_u8.astype(np.float64) / 255.0, ds.colors)
        assert np.array_equal(depths_u16.astype(np.float64) / 1000.0, ds.depths)
        for precision in ("double", "single"):
            cfg = optimizer.TrainConfig(precision=precision, **case["cfg"])
            cfg.weights.smooth_count = case["smooth_count"]
            dc.set_finite_checks(precision == "double")
            model = optimizer.build_model(ds, cfg, skip_init=True)
            opt = optimizer.make_optimizer(model, cfg)
            names = optimizer._param_names(model)
            init = {n: p.data.copy() for n, p in zip(names, model.parameters())}

            rounds = []
            orig = sampler.importance_refine_with_sources

            def spy(depths, weights, near, far, uniforms):
                out, src = orig(depths, weights, near, far, uniforms)
                rounds.append(dict(depths_in=np.array(depths), weights=np.array(weights),
                                   uniforms=np.array(uniforms), depths=out, src=src))
                return out, src

            rec = {}
            it0 = case["iteration"]
            for it in (it0, it0 + 1):
                rounds.clear()
                sampler.importance_refine_with_sources = spy
                try:
                    batch = sampler.draw_ray_batch(
                        ds, seeds.substream(cfg.seed, seeds.RAYS, it), cfg.batch_rays,
                        near=cfg.near, far=cfg.max_depth)
                    total, parts, extras = renderer.train_objective(model, ds, batch, it, cfg)
                finally:
                    sampler.importance_refine_with_sources = orig
                grads = dc.grad(total, opt.params)
                if it == it0:
                    rec["batch"] = batch
                    rec["parts"] = parts
                    rec["extras"] = {k: v for k, v in extras.items()
                                     if k not in ("depths", "weights")}
                    rec["depths"] = extras["depths"]
                    rec["weights"] = extras["weights"].data
                    rec["grads"] = {n: g.data.copy() for n, g in zip(names, grads)}
                    rec["rounds"] = [dict(r) for r in rounds]
                else:
                    rec["parts1"] = parts
                opt.step(grads)
                if it == it0:
                    rec["step1"] = {n: q.data.copy() for n, q in zip(names, model.parameters())}
                    rec["step1_m"] = [x.copy() for x in opt.m]
                    rec["step1_v"] = [x.copy() for x in opt.v]
            arrays = {}
            arrays["colors_u8"] = colors_u8
            arrays["depths_u16"] = depths_u16
            arrays["poses"] = ds.poses
            b = rec["batch"]
            for k in ("frame_ids", "pixels", "color", "depth_ray", "valid", "dir_cam"):
                arrays[f"batch_{k}"] = getattr(b, k)
            arrays["depths"] = rec["depths"]
            arrays["weights"] = rec["weights"]
            for i, r in enumerate(rec["rounds"]):
                for k, v in r.items():
                    arrays[f"round{i}_{k}"] = v
            for n in names:
                arrays[f"init_{n}"] = init[n]
                arrays[f"grad_{n}"] = rec["grads"][n]
                arrays[f"final_{n}"] = [p for nn, p in zip(names, model.parameters())
                                        if nn == n][0].data
            for i, n in enumerate(names):
                arrays[f"step1_{n}"] = rec["step1"][n]
                arrays[f"step1_m_{n}"] = rec["step1_m"][i]
                arrays[f"step1_v_{n}"] = rec["step1_v"][i]
            for n, m_, v_ in zip(names, opt.m, opt.v):
                arrays[f"adam_m_{n}"] = m_
                arrays[f"adam_v_{n}"] = v_
            meta = dict(
                case=name, precision=precision, intr=list(map(float, case["intr"])),
                frames=case["frames"], cfg={k: (list(map(list, v)) if k == "bounds" else
                                                 (list(v) if isinstance(v, tuple) else v))
                                            for k, v in case["cfg"].items()},
                smooth_count=case["smooth_count"], iteration=case["iteration"],
                parts=rec["parts"], parts1=rec["parts1"], extras=rec["extras"],
                names=names, lo=list(map(float, model.grid.lo)), hi=list(map(float, model.grid.hi)),
                adam_t=opt.t, skipped=opt.skipped,
                numpy=np.__version__,
            )
            arrays["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
            path = os.path.join(HERE, f"{name}_{precision}.npz")
            np.savez_compressed(path, **arrays)
            out_files.append(path)
            print(f"{path}: {os.path.getsize(path) / 1e6:.2f} MB  parts={rec['parts']}")
    return out_files


if __name__ == "__main__":
    sys.exit(0 if main() else 1)
