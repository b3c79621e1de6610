"""Edge cases of the step against the oracle (the oracle itself is pinned to
the reference, tests/test_oracle_golden.py): missing depth (invalid rays:
eikonal over the whole ray, no depth / sdf / fs terms), a frame with no valid
pixel at all, ragged batch sizes (1 ray, a partial warp, a partial 128-tile),
all samples in free space (fixed far in front of the surface), and a dataset
where every depth is missing (n_valid = 0: normalisers clamp at 1, the
smoothness point set is empty).  float64 device step, losses and gradients to
1e-9."""

import numpy as np
import pytest

from _golden import load, oracle_params
from oracle import gridsurf_oracle as O

PART_KEYS = ("total", "rgb", "depth", "sdf", "fs", "eik", "smooth", "s")


def variant(name):
    """(golden handle with modified dataset, batch size, cfg overrides)."""
    G = load("small", "double")
    dep = G.a["depths_u16"].copy()
    over = {}
    m = 48
    if name == "holes":          # rectangle of missing depth in every frame + one empty frame
        dep[:, 4:14, 6:20] = 0
        dep[2] = 0
    elif name == "ragged1":
        m = 1
    elif name == "ragged37":
        m = 37
    elif name == "ragged130":
        m = 130
    elif name == "freespace":     # every sample in front of the surface
        over = dict(fixed_far=0.05)
    elif name == "nodepth":
        dep[:] = 0
    return G, dep, m, over


def oracle_step(G, dep, m, over):
    ds = O_dataset(G, dep)
    cfg = G.cfg
    for k, v in over.items():
        setattr(cfg, k, v)
    cfg.batch_rays = m
    P = oracle_params(G)
    it = G.meta["iteration"]
    b = O.draw_ray_batch(ds, O.substream(cfg.seed, O.RAYS, it), m, near=cfg.near, far=cfg.max_depth)
    return O.train_objective(P, ds, b, it, cfg), P


def O_dataset(G, dep):
    from _golden import OracleDataset
    return OracleDataset(G.a["colors_u8"], dep, G.a["poses"], G.ds.intrinsics)


@pytest.mark.parametrize("name", ["holes", "ragged1", "ragged37", "nodepth"])
def test_oracle_edge_case_runs(name):
    """CPU: the restatement handles each case (finite parts, sane counts)."""
    G, dep, m, over = variant(name)
    R, _ = oracle_step(G, dep, m, over)
    assert all(np.isfinite(v) for v in R["parts"].values())
    e = R["extras"]
    if name == "nodepth":
        assert e["n_valid_rays"] == 0 and e["n_tr"] == 0 and e["n_fs"] == 0
        assert R["parts"]["depth"] == 0.0 and R["parts"]["sdf"] == 0.0 and R["parts"]["smooth"] == 0.0
        assert e["n_eik"] == m * e["samples_per_ray"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["holes", "ragged1", "ragged37", "ragged130", "freespace", "nodepth"])
def test_device_edge_case_matches_oracle(name):
    import torch
    from paper_2206_14735_b200 import data, optimizer, renderer, sampler, seeds
    G, dep, m, over = variant(name)
    R, P = oracle_step(G, dep, m, over)
    cfg = optimizer.TrainConfig(precision="double", **{
        k: v for k, v in G.meta["cfg"].items() if k not in ("bounds", "voxel_sizes")},
        voxel_sizes=G.cfg.voxel_sizes, bounds=G.cfg.bounds)
    cfg.weights.smooth_count = G.meta["smooth_count"]
    cfg.batch_rays = m
    cfg.bounds = (tuple(G.meta["lo"]), tuple(G.meta["hi"]))  # the oracle's box (not re-derived)
    for k, v in over.items():
        setattr(cfg, k, v)
    ds = data.Dataset(G.a["colors_u8"], dep, G.a["poses"], G.ds.intrinsics)
    model = optimizer.build_model(ds, cfg, skip_init=True, device=torch.device("cuda", 0))
    it = G.meta["iteration"]
    batch = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, it), m, near=cfg.near,
                                   far=cfg.max_depth)
    total, parts, extras = renderer.train_objective(model, ds, batch, it, cfg)
    grads = renderer.grad(total, model.parameters())
    bad = {k: (parts[k], R["parts"][k]) for k in PART_KEYS
           if not abs(parts[k] - R["parts"][k]) <= 1e-9 * max(abs(R["parts"][k]), 1e-12)}
    assert not bad, bad
    for k in ("n_valid_rays", "n_tr", "n_fs", "n_eik", "n_smooth"):
        assert extras[k] == R["extras"][k], k
    # device exp vs numpy's SIMD exp (<= 1 ulp) moves importance depths at 1e-12
    np.testing.assert_allclose(extras["depths"], R["depths"], rtol=1e-10, atol=1e-11)
    for n, g in zip(model.param_names(), grads):
        ref = R["grads"][n]
        scale = max(np.abs(ref).max(), 1e-300)
        assert np.abs(g.detach().cpu().numpy() - ref).max() <= 1e-9 * scale, n
