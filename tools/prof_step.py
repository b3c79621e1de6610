"""Short config-2 step loop for profiling (ncu / timing): 2 frames, M rays."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2206_14735_b200 import engine, optimizer, scenes
from paper_2206_14735_b200.renderer import engine_for

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--rays", type=int, default=6144)
ap.add_argument("--frames", type=int, default=2)
ap.add_argument("--precision", default="single")
a = ap.parse_args()
dev = torch.device("cuda", 0)
cfg = optimizer.TrainConfig(precision=a.precision, batch_rays=a.rays, bounds=scenes.CONFIG2_BOUNDS)
ds = scenes.config2(frames=a.frames, threads=8)
model = optimizer.build_model(ds, cfg, skip_init=True, device=dev)
opt = optimizer.make_optimizer(model, cfg)
eng = engine_for(model, ds)
for it in range(a.steps):
    d = engine.host_draws(model, ds, cfg, it)
    ids, sm = eng.upload(d)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ws = eng.launch(cfg, d, ids, sm)
    opt.t = [t + 1 for t in opt.t]
    opt._launch()
    torch.cuda.synchronize()
    print(f"step {it}: {1e3 * (time.perf_counter() - t0):.2f} ms total={ws['parts'][0].item():.5f}")
