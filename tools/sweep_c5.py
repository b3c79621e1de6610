"""BASELINE configs[4] (c5): ray-batch sweep 1K-256K rays x 64-192 samples
per ray, smoothness on and off, on the c2 scene/grid.  One process: the
scene and model are built once; each point is W warm-up + K device-timed
steps (objective + backward + Adam), inputs resident in HBM."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2206_14735_b200 import engine, optimizer, scenes
from paper_2206_14735_b200.renderer import engine_for

ap = argparse.ArgumentParser()
ap.add_argument("--rays", default="1024,4096,16384,65536,262144")
ap.add_argument("--samples", default="64,96,132,192")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda", 0)
ds = scenes.config2(frames=8, threads=8)
base = bench.make_cfg()
model = optimizer.build_model(ds, base, skip_init=True, device=dev)
opt = optimizer.make_optimizer(model, base)
eng = engine_for(model, ds)
rows = []
for smooth in (True, False):
    for N in (int(x) for x in a.samples.split(",")):
        for M in (int(x) for x in a.rays.split(",")):
            cfg = bench.make_cfg(batch=M, coarse=N - 36, smooth=smooth)
            pre = []
            for it in range(a.warmup + a.steps):
                d = engine.host_draws(model, ds, cfg, it)
                pre.append((d, *eng.upload(d)))

            def step(d, ids, sm):
                eng.launch(cfg, d, ids, sm)
                opt.t = [t + 1 for t in opt.t]
                opt._launch()

            for p in pre[:a.warmup]:
                step(*p)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for p in pre[a.warmup:]:
                step(*p)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            r = dict(rays=M, samples=N, smooth=smooth, ms_per_step=ms, rays_per_s=M / ms * 1e3,
                     samples_per_s=M * N / ms * 1e3)
            rows.append(r)
            print(json.dumps(r), flush=True)
            del pre
            eng._ws.clear()
            torch.cuda.empty_cache()
