"""Host-side cost of one training iteration (c2): draws, upload, launch."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2206_14735_b200 import engine, optimizer, scenes
from paper_2206_14735_b200.renderer import engine_for

cfg = bench.make_cfg()
ds = scenes.config2(frames=8, threads=8)
dev = torch.device("cuda", 0)
model = optimizer.build_model(ds, cfg, skip_init=True, device=dev)
opt = optimizer.make_optimizer(model, cfg)
eng = engine_for(model, ds)
T = optimizer.Trainer(model, ds, cfg, opt)
acc = {}


def tick(name, t0):
    acc.setdefault(name, []).append(time.perf_counter() - t0)


for it in range(60):
    t0 = time.perf_counter()
    d = engine.host_draws(model, ds, cfg, it)
    tick("host_draws", t0)
    t0 = time.perf_counter()
    ids, sm = eng.upload(d)
    tick("upload", t0)
    t0 = time.perf_counter()
    ws = eng.launch(cfg, d, ids, sm)
    tick("engine.launch", t0)
    t0 = time.perf_counter()
    opt.t = [t + 1 for t in opt.t]
    opt._launch(guard=ws["parts"], guard_threshold=cfg.divergence_threshold)
    tick("adam launch", t0)
    t0 = time.perf_counter()
    torch.cuda.synchronize()
    tick("gpu wait", t0)
for k, v in acc.items():
    print(f"{k:16s} {1e3 * np.median(v[10:]):7.3f} ms")
