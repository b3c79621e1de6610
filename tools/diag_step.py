import sys, os
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np, torch
from _golden import load, oracle_params, rel_maxnorm
from oracle import gridsurf_oracle as O
from paper_2206_14735_b200 import data, optimizer, renderer, sampler, seeds
dev = torch.device("cuda", 0)
for case in ("tiny", "small"):
  for prec in ("double", "single"):
    G = load(case, prec)
    cfg = optimizer.TrainConfig(precision=prec, **{k: v for k, v in G.meta["cfg"].items() if k not in ("bounds", "voxel_sizes")}, voxel_sizes=G.cfg.voxel_sizes, bounds=G.cfg.bounds)
    cfg.weights.smooth_count = G.meta["smooth_count"]
    ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"], G.ds.intrinsics)
    model = optimizer.build_model(ds, cfg, skip_init=True, device=dev)
    it = G.meta["iteration"]
    b = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, it), cfg.batch_rays, near=cfg.near, far=cfg.max_depth)
    total, parts, extras = renderer.train_objective(model, ds, b, it, cfg)
    g = renderer.grad(total, model.parameters())
    print(f"== {case} {prec}")
    print(" parts rel:", {k: f"{(parts[k]-v)/max(abs(v),1e-30):.2e}" for k, v in G.meta["parts"].items()})
    print(" extras:", {k: (extras[k], G.meta["extras"][k]) for k in ("n_valid_rays","n_tr","n_fs","n_eik","n_smooth")})
    d = extras["depths"]; print(" depths maxabs", np.abs(d - G.a["depths"]).max(), " weights maxabs", np.abs(extras["weights"] - G.a["weights"]).max())
    print(" grads:", {n: f"{rel_maxnorm(t.cpu().numpy(), G.a['grad_'+n]):.1e}" for n, t in zip(model.param_names(), g)})
