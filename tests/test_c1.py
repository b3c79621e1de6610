"""Parity at BASELINE configs[0] (c1: sphere-in-box, 20 frames 160x120,
default 4-level grid, P = 8.66 M, M = 1024 rays x 132 samples) against the
reference's own step (tests/golden/make_golden_c1.py): loss parts, extras,
sampled depths and rendering weights whole; each parameter tensor's gradient
through checksums (sum, sum of squares, max |g|) and 4096 sampled entries."""

import json
import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

PART_KEYS = ("total", "rgb", "depth", "sdf", "fs", "eik", "smooth", "s")


def golden(precision):
    z = np.load(os.path.join(HERE, "golden", f"c1_{precision}.npz"))
    a = {k: z[k] for k in z.files}
    return a, json.loads(a.pop("meta_json").tobytes().decode())


def intrinsics(meta):
    fx, fy, cx, cy, w, h = meta["intr"]
    return SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))


def checksums(g):
    a = np.asarray(g, dtype=np.float64).reshape(-1)
    return np.array([a.sum(), (a * a).sum(), np.abs(a).max()]), a


def grad_errors(grads, a, names):
    """Per tensor: relative checksum error and sampled-entry error vs max |g|."""
    out = {}
    for n in names:
        cs, flat = checksums(grads[n])
        ref_cs = a[f"gsum_{n}"]
        scale = max(abs(ref_cs[2]), 1e-300)
        e_sum = abs(cs[0] - ref_cs[0]) / max(abs(ref_cs[0]), scale)
        e_sq = abs(cs[1] - ref_cs[1]) / max(ref_cs[1], 1e-300)
        e_max = abs(cs[2] - ref_cs[2]) / scale
        e_val = np.abs(flat[a[f"gidx_{n}"]] - a[f"gval_{n}"]).max() / scale
        out[n] = max(e_sum, e_sq, e_max, e_val)
    return out


def ref_f32_errors(names):
    """The reference's own float32-vs-float64 distance, per tensor / part."""
    d, md = golden("double")
    s, ms = golden("single")
    gs = {n: None for n in names}
    for n in names:
        cs_s, cs_d = s[f"gsum_{n}"], d[f"gsum_{n}"]
        scale = max(abs(cs_d[2]), 1e-300)
        e_val = np.abs(s[f"gval_{n}"] - d[f"gval_{n}"]).max() / scale
        gs[n] = max(abs(cs_s[0] - cs_d[0]) / max(abs(cs_d[0]), scale),
                    abs(cs_s[1] - cs_d[1]) / max(cs_d[1], 1e-300), abs(cs_s[2] - cs_d[2]) / scale, e_val)
    ps = {k: abs(ms["parts"][k] - md["parts"][k]) / max(abs(md["parts"][k]), 1e-300) for k in PART_KEYS}
    return gs, ps


def test_oracle_c1_double_matches_reference():
    from _golden import OracleDataset, cfg_ns
    from oracle import gridsurf_oracle as O
    a, meta = golden("double")
    ds = OracleDataset(a["colors_u8"], a["depths_u16"], a["poses"], intrinsics(meta))
    cfg = cfg_ns(precision="double", batch_rays=1024, bounds=(tuple(meta["lo"]), tuple(meta["hi"])))
    P = O.create_params(meta["lo"], meta["hi"], ds.poses, seed=0, dtype=np.float64)
    b = O.draw_ray_batch(ds, O.substream(0, O.RAYS, 0), 1024)
    R = O.train_objective(P, ds, b, 0, cfg)
    for k in PART_KEYS:
        assert abs(R["parts"][k] - meta["parts"][k]) <= 1e-14 * max(abs(meta["parts"][k]), 1e-300), k
    np.testing.assert_array_equal(R["depths"], a["depths"])
    errs = grad_errors(R["grads"], a, meta["names"])
    assert max(errs.values()) <= 1e-10, errs


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["double", "single"])
def test_device_c1_step_matches_reference(precision):
    import torch
    from paper_2206_14735_b200 import data, optimizer, renderer, sampler, seeds
    a, meta = golden(precision)
    intr = intrinsics(meta)
    from paper_2206_14735_b200.camera import Intrinsics
    ds = data.Dataset(a["colors_u8"], a["depths_u16"], a["poses"],
                      Intrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
    cfg = optimizer.TrainConfig(precision=precision, batch_rays=1024, seed=0)
    model = optimizer.build_model(ds, cfg, skip_init=True, device=torch.device("cuda", 0))
    np.testing.assert_array_equal(model.grid.lo, meta["lo"])
    np.testing.assert_array_equal(model.grid.hi, meta["hi"])
    assert sum(p.size for p in model.parameters()) == meta["n_params"]
    batch = sampler.draw_ray_batch(ds, seeds.substream(0, seeds.RAYS, 0), 1024, near=cfg.near,
                                   far=cfg.max_depth)
    total, parts, extras = renderer.train_objective(model, ds, batch, 0, cfg)
    grads = renderer.grad(total, model.parameters())
    g = {n: t.detach().cpu().numpy() for n, t in zip(model.param_names(), grads)}
    errs = grad_errors(g, a, meta["names"])
    if precision == "double":
        for k in PART_KEYS:
            assert abs(parts[k] - meta["parts"][k]) <= 1e-12 * max(abs(meta["parts"][k]), 1e-300), k
        for k in ("n_valid_rays", "n_tr", "n_fs", "n_eik"):
            assert extras[k] == meta["extras"][k], k
        assert max(errs.values()) <= 1e-9, errs
    else:
        g_ref, p_ref = ref_f32_errors(meta["names"])
        for k in PART_KEYS:
            e = abs(parts[k] - meta["parts"][k]) / max(abs(meta["parts"][k]), 1e-300)
            assert e <= max(4 * p_ref[k], 1e-5), (k, e, p_ref[k])
        bad = {n: (e, g_ref[n]) for n, e in errs.items() if not e <= max(4 * g_ref[n], 2e-4)}
        assert not bad, bad
