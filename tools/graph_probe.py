"""How much of the c2 step is launch overhead?  Time the same step (objective +
backward + Adam, fixed inputs) issued eagerly and replayed from a CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2206_14735_b200 import engine, optimizer, scenes
from paper_2206_14735_b200.renderer import engine_for

cfg = bench.make_cfg()
ds = scenes.config2(frames=8)
dev = torch.device("cuda", 0)
model = optimizer.build_model(ds, cfg, skip_init=True, device=dev)
opt = optimizer.make_optimizer(model, cfg)
eng = engine_for(model, ds)
d = engine.host_draws(model, ds, cfg, 0)
ids, sm = eng.upload(d)
torch.cuda.synchronize()


def step():
    eng.launch(cfg, d, ids, sm)
    opt.t = [1 for _ in opt.t]
    opt._launch()


s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        step()
    b.record()
    b.synchronize()
    eager = a.elapsed_time(b) / 50
    g = torch.cuda.CUDAGraph()
    import ctypes
    from paper_2206_14735_b200 import _lib
    with torch.cuda.graph(g, stream=s):
        step()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(50):
        g.replay()
    b.record()
    b.synchronize()
    graph = a.elapsed_time(b) / 50
print(f"eager {eager:.4f} ms/step, graph replay {graph:.4f} ms/step, launch overhead {eager - graph:.4f} ms")
