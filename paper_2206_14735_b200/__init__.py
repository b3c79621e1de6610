"""B200-native GO-Surf training step (arXiv 2206.14735).

Drop-in for the reference ``gridsurf`` package's optimisation path:

    from paper_2206_14735_b200 import optimizer, renderer, sampler, seeds
    model = optimizer.build_model(dataset, cfg, skip_init=True)
    opt = optimizer.make_optimizer(model, cfg)
    batch = sampler.draw_ray_batch(dataset, seeds.substream(cfg.seed, seeds.RAYS, it),
                                   cfg.batch_rays, near=cfg.near, far=cfg.max_depth)
    total, parts, extras = renderer.train_objective(model, dataset, batch, it, cfg)
    grads = renderer.grad(total, opt.params)
    opt.step(grads)

The step runs as hand-written sm_100a CUDA kernels behind the C ABI in
include/gsb.h (``_gsb.so``, loaded with ctypes).  There is no CPU fallback.
"""

from . import camera, checkpoint, data, seeds  # noqa: F401

__all__ = ["camera", "checkpoint", "data", "seeds", "model", "sampler", "renderer",
           "optimizer", "engine"]


def __getattr__(name):
    import importlib
    if name in ("model", "sampler", "renderer", "optimizer", "engine", "geometry", "scenes",
                "dist"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
