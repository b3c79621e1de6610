"""Where does the e2e loop lose time vs the device-timed loop?  GPU-event
time of the Trainer loop vs wall time, and host time per phase."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2206_14735_b200 import optimizer, scenes

cfg = bench.make_cfg()
ds = scenes.config2(frames=8, threads=8)
dev = torch.device("cuda", 0)
model = optimizer.build_model(ds, cfg, skip_init=True, device=dev)
opt = optimizer.make_optimizer(model, cfg)
T = optimizer.Trainer(model, ds, cfg, opt)
for it in range(5):
    T.launch(it, slot=it % 2)
torch.cuda.synchronize()
K = 100
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
host_launch, host_wait = [], []
t0 = time.perf_counter()
e0.record()
pending = None
for k in range(K):
    a = time.perf_counter()
    T.launch(5 + k, slot=k % 2)
    b = time.perf_counter()
    if pending is not None:
        T.parts(pending)
    c = time.perf_counter()
    host_launch.append(b - a)
    host_wait.append(c - b)
    pending = k % 2
T.parts(pending)
e1.record()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"wall/step {1e3 * wall / K:.3f} ms  gpu/step {e0.elapsed_time(e1) / K:.3f} ms  "
      f"host launch {1e3 * np.median(host_launch):.3f} ms  host wait {1e3 * np.median(host_wait):.3f} ms")
