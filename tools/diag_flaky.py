"""Run-to-run check of the float32 device step: the same model, batch and
iteration stepped R times; per-tensor max |g_r - g_0| / max|g_0|.  float32
atomics alone give ~1e-6; anything larger is a race.  Usage (GPU box):
python tools/diag_flaky.py [case] [R]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
import test_f32_parity as T  # noqa: E402
from paper_2206_14735_b200 import optimizer, renderer, sampler, seeds  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c1"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ds, kw = T._dataset(case)
smooth_count = kw.pop("smooth_count", None)
cfg = optimizer.TrainConfig(precision="single", **kw)
if smooth_count is not None:
    cfg.weights.smooth_count = smooth_count
model = optimizer.build_model(ds, cfg, skip_init=False, device=torch.device("cuda", 0))
it = 3
batch = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, it), cfg.batch_rays,
                               near=cfg.near, far=cfg.max_depth)
runs = []
for r in range(R):
    total, parts, extras = renderer.train_objective(model, ds, batch, it, cfg)
    grads = renderer.grad(total, model.parameters())
    g = {n: t.cpu().numpy().copy() for n, t in zip(model.param_names(), grads)}
    eng = renderer.engine_for(model, ds)
    M = cfg.batch_rays
    ws = eng.workspace(M, cfg.coarse_samples, cfg.importance_rounds, cfg.importance_add,
                       cfg.weights.smooth_count)
    dev = {k: ws[k].cpu().numpy().copy() for k in ("phi", "gphi", "color", "depths", "pbar", "ubar", "cbar")}
    runs.append((float(total), g, dev))
t0, g0, d0 = runs[0]
for r, (t, g, d) in enumerate(runs[1:], 1):
    ge = {n: float(np.abs(g[n] - g0[n]).max() / max(np.abs(g0[n]).max(), 1e-30)) for n in g0}
    de = {k: float(np.abs(d[k] - d0[k]).max()) for k in d0}
    bad = {n: v for n, v in ge.items() if v > 1e-5}
    print(r, "total", t - t0, "per-sample max diffs", de, "grads >1e-5:", bad, flush=True)
    for n in bad:
        diff = np.abs(g[n] - g0[n]).reshape(-1)
        idx = np.argsort(diff)[::-1][:8]
        print("   ", n, "shape", g0[n].shape, "top idx", idx.tolist(), "diff", diff[idx].tolist(),
              "g0", g0[n].reshape(-1)[idx].tolist(), flush=True)
