"""Sphere pre-fit (decoders.geometric_init, gs/decoders.py:102-177): the
oracle (CPU) and the device implementation against golden vectors produced by
running the reference (tests/golden/make_golden_init.py), plus the
reference's own known-answer checks (pkg/tests/test_decoders.py:114-142)."""

import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from _golden import load, oracle_params, rel_maxnorm  # noqa: E402

NAMES_NET = [f"geom_{k}{i}" for i in range(3) for k in ("w", "b")]


def init_golden(precision):
    z = np.load(os.path.join(HERE, "golden", f"init_small_{precision}.npz"))
    arrays = {k: z[k] for k in z.files}
    meta = json.loads(arrays.pop("meta_json").tobytes().decode())
    return arrays, meta


def ref_errors(name):
    """The reference's own float32-vs-float64 distance after K steps."""
    d, _ = init_golden("double")
    s, _ = init_golden("single")
    return rel_maxnorm(s[name], d[name])


def compare(params, precision, floor):
    ref, meta = init_golden(precision)
    errs = {}
    for n, a in ref.items():
        e = rel_maxnorm(params[n], a)
        budget = 1e-9 if precision == "double" else max(4 * ref_errors(n), floor)
        errs[n] = (e, budget)
    bad = {n: v for n, v in errs.items() if not v[0] <= v[1]}
    assert not bad, bad
    return meta


@pytest.mark.parametrize("precision", ["double", "single"])
def test_oracle_init_k_steps_matches_reference(precision):
    from oracle import gridsurf_oracle as O
    G = load("small", precision)
    P = oracle_params(G)
    _, meta = init_golden(precision)
    rmse = O.geometric_init(P, meta["center"], meta["radius"], seed=meta["seed"],
                            max_steps=meta["K"], tol=1e9)
    params = {f"level{i}": P.levels[i].feat for i in range(len(P.levels))}
    params.update({f"geom_{k}{i}": P.geom[i][j] for i in range(3) for j, k in ((0, "w"), (1, "b"))})
    compare(params, precision, 1e-4)
    assert abs(rmse - meta["rmse_k"]) <= (1e-12 if precision == "double" else 1e-5) * meta["rmse_k"]


def test_oracle_init_rejects_sphere_outside_box():
    from oracle import gridsurf_oracle as O
    G = load("small", "double")
    P = oracle_params(G)
    with pytest.raises(ValueError):
        O.geometric_init(P, (0.0, 0.0, 0.0), 100.0)
    with pytest.raises(O.InitError):
        O.geometric_init(P, 0.5 * (np.array(G.meta["lo"]) + np.array(G.meta["hi"])), 0.3, max_steps=0)


def _gpu_model(precision):
    import torch
    from paper_2206_14735_b200 import data, optimizer
    G = load("small", precision)
    cfg = optimizer.TrainConfig(precision=precision, **{
        k: v for k, v in G.meta["cfg"].items() if k not in ("bounds", "voxel_sizes")},
        voxel_sizes=G.cfg.voxel_sizes, bounds=G.cfg.bounds)
    ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"], G.ds.intrinsics)
    model = optimizer.build_model(ds, cfg, skip_init=True, device=torch.device("cuda", 0))
    return model


def _params_of(model):
    out = {f"level{i}": l.features.numpy() for i, l in enumerate(model.grid.levels)}
    for i, (W, b) in enumerate(model.geom_net.layers):
        out[f"geom_w{i}"] = W.numpy()
        out[f"geom_b{i}"] = b.numpy()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["double", "single"])
def test_device_init_k_steps_matches_reference(precision):
    from paper_2206_14735_b200.geometry import geometric_init
    model = _gpu_model(precision)
    _, meta = init_golden(precision)
    rmse = geometric_init(model, meta["center"], meta["radius"], seed=meta["seed"],
                          max_steps=meta["K"], tol=1e9)
    compare(_params_of(model), precision, 1e-4)
    assert abs(rmse - meta["rmse_k"]) <= (1e-9 if precision == "double" else 1e-4) * meta["rmse_k"]


@pytest.mark.gpu
def test_device_init_full_run_double_matches_reference_exit():
    """Same early-exit step and final RMSE as the reference's full pre-fit."""
    from paper_2206_14735_b200.geometry import geometric_init
    model = _gpu_model("double")
    _, meta = init_golden("double")
    info = {}
    rmse = geometric_init(model, meta["center"], meta["radius"], seed=meta["seed"], info=info)
    assert info["steps"] == meta["full_steps"]
    assert abs(rmse - meta["rmse_full"]) <= 1e-7 * meta["rmse_full"]


@pytest.mark.gpu
def test_device_init_float32_reaches_sphere_sdf():
    """pkg/tests/test_decoders.py:114-132 on the production (float32) path."""
    from paper_2206_14735_b200.geometry import SdfQuery, geometric_init
    model = _gpu_model("single")
    _, meta = init_golden("double")
    center, radius = np.array(meta["center"]), meta["radius"]
    final = geometric_init(model, center, radius, seed=meta["seed"])
    assert final < 0.01
    q = SdfQuery(model)
    rng = np.random.default_rng(8)
    d = rng.normal(size=(64, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    assert np.max(np.abs(q((center + radius * d).astype(np.float32)))) < 0.03
    assert q(center[None, :].astype(np.float32))[0] == pytest.approx(-radius, abs=0.01)
    two_r = (center + np.array([[2 * radius, 0.0, 0.0]])).astype(np.float32)
    assert q(two_r)[0] == pytest.approx(radius, abs=0.02)


@pytest.mark.gpu
def test_build_model_runs_geometric_init_by_default():
    """build_model(skip_init=False) is the reference default (gs/optimizer.py:206-213)."""
    import torch
    from paper_2206_14735_b200 import data, optimizer
    G = load("small", "single")
    cfg = optimizer.TrainConfig(precision="single", **{
        k: v for k, v in G.meta["cfg"].items() if k not in ("bounds", "voxel_sizes")},
        voxel_sizes=G.cfg.voxel_sizes, bounds=G.cfg.bounds, sphere_radius_scale=0.3)
    ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"], G.ds.intrinsics)
    model = optimizer.build_model(ds, cfg, device=torch.device("cuda", 0))
    lo, hi = np.array(G.meta["lo"]), np.array(G.meta["hi"])
    from paper_2206_14735_b200.geometry import SdfQuery
    c = 0.5 * (lo + hi)
    assert SdfQuery(model)(c[None, :].astype(np.float32))[0] < 0.0
