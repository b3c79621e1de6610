"""Reference arm of bench.py: the UNMODIFIED reference package (`gridsurf`,
installed once into baseline/_ref with

    cp -r /root/reference/pkg /tmp/gsref
    python -m pip install --no-index --no-build-isolation --no-deps \
        --find-links /opt/wheelhouse --target baseline/_ref /tmp/gsref

) timed on the host cores through its own public API and stock code path:
the body of `gs/optimizer.py:train` (`:362-373`), i.e.

    batch = sampler.draw_ray_batch(ds, seeds.substream(seed, RAYS, it), M)
    total, parts, extras = renderer.train_objective(model, ds, batch, it, cfg)
    grads = dc.grad(total, opt.params)
    opt.step(grads)

on the same workload as the B200 arm: the config-2 scene rendered by the
reference's own `scenegen.render_dataset` (no repo code, no repo .so), the
same frames, pinned bounds, grid, batch and samples, float32.

Runs as its own process (bench.py spawns it) so that OpenBLAS / numba see
the thread count before numpy is imported and nothing of this repository is
loaded.  Prints one JSON object on stdout.
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--rays", type=int, default=6144)
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--precision", default="single")
    args = ap.parse_args()
    sys.path.insert(0, REF)
    import numpy as np
    from gridsurf import camera, optimizer, renderer, sampler, scenegen, seeds
    from gridsurf import diffcore as dc

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    if args.config == 1:
        # gs/cli.py:144-147 intrinsics (70 deg FOV), sphere_in_box, 20-frame orbit
        w, h = 160, 120
        f = 0.5 * w / np.tan(np.radians(35.0))
        intr = camera.Intrinsics(f, f, w / 2.0, h / 2.0, w, h)
        scene = scenegen.sphere_in_box()
        traj = scenegen.orbit_trajectory(args.frames)
        bounds = None
    else:
        # ScanNet intrinsics, the 6 x 6 x 3 m room, pinned box
        intr = camera.Intrinsics(577.87, 577.87, 319.5, 239.5, 640, 480)
        room = scenegen.Complement(scenegen.Box((0.0, 0.0, 1.5), (3.0, 3.0, 1.5),
                                                albedo=(0.75, 0.72, 0.65), checker=0.25))
        parts = [room, scenegen.Sphere((1.2, 0.8, 0.5), 0.5),
                 scenegen.Sphere((-1.5, -1.0, 0.35), 0.35, albedo=(0.2, 0.5, 0.8)),
                 scenegen.Box((0.0, -1.8, 0.4), (0.6, 0.4, 0.4), albedo=(0.3, 0.7, 0.3),
                              checker=0.1)]
        light = np.array([0.3, 0.5, -0.8])
        scene = scenegen.AnalyticScene(scenegen.Union(*parts), light / np.linalg.norm(light),
                                       np.array([0.1, 0.1, 0.12]))
        traj = scenegen.orbit_trajectory(args.frames, target=(0.0, 0.0, 0.8), radius=1.8,
                                         height=1.5, height_amp=0.3)
        bounds = ((-3.5, -3.5, -0.5), (3.5, 3.5, 2.75))
    ds = scenegen.render_dataset(scene, traj, intr, threads=threads)
    t_render = time.perf_counter() - t0

    cfg = optimizer.TrainConfig(precision=args.precision, batch_rays=args.rays, bounds=bounds,
                                iterations=10 ** 6)
    dc.set_finite_checks(cfg.precision == "double")  # as train() does
    model = optimizer.build_model(ds, cfg, skip_init=True)
    opt = optimizer.make_optimizer(model, cfg)
    P = int(sum(p.data.size for p in model.parameters()))

    def step(it):
        batch = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, it),
                                       cfg.batch_rays, near=cfg.near, far=cfg.max_depth)
        total, parts, extras = renderer.train_objective(model, ds, batch, it, cfg)
        grads = dc.grad(total, opt.params)
        opt.step(grads)
        return parts

    for it in range(args.warmup):  # numba JIT + first-touch allocations
        step(it)
    times = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        parts = step(args.warmup + k)
        times.append(time.perf_counter() - t0)
    tot = float(sum(times))
    print(json.dumps({"value": args.rays * args.steps / tot, "ms_per_step": 1e3 * tot / args.steps,
                      "median_step_s": float(np.median(times)), "steps": args.steps,
                      "warmup": args.warmup, "threads": threads, "params": P,
                      "render_s": t_render, "rays": args.rays, "frames": args.frames,
                      "total": parts["total"], "config": args.config}), flush=True)


if __name__ == "__main__":
    main()
