"""Pose refinement against the reference's own run
(tests/golden/make_golden_pose.py): the "small" case with refine_poses=True
(frame 0 frozen) and pose_refresh_every=2, trained 4 iterations through the
reference loop body (draw, train_objective, grad, Adam, refresh).  Every
iteration's loss parts and every gradient -- including d/d nu_f, d/d t_f --
are compared, and after the last iteration every parameter and R0.

* CPU: the oracle restatement (oracle/gridsurf_oracle.py pose_backward,
  exp_so3_adjoint) against the golden; the exp_so3 adjoint against finite
  differences on both branches.
* GPU: the device path (gsb_pose_table / gsb_pose_grad through the
  package's public train_objective / grad / Adam / PoseParam.refresh) against
  the golden, and a checkpoint round trip with trainable poses."""

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
    z = np.load(os.path.join(HERE, "golden", f"pose_small_{precision}.npz"))
    a = {k: z[k] for k in z.files}
    return a, json.loads(a.pop("meta_json").tobytes().decode())


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def ref_f32_budget(names):
    """The reference's own float32-vs-float64 distance per iteration / tensor."""
    d, md = golden("double")
    s, ms = golden("single")
    g = [{n: rel(s[f"it{it}_grad_{n}"], d[f"it{it}_grad_{n}"]) for n in names} for it in range(md["iters"])]
    p = [{k: abs(ms["parts"][it][k] - md["parts"][it][k]) / max(abs(md["parts"][it][k]), 1e-300)
          for k in PART_KEYS} for it in range(md["iters"])]
    return g, p


def is_pose(name):
    return name.startswith("nu") or (name[0] == "t" and name[1:].isdigit())


def _intr(meta):
    fx, fy, cx, cy, w, h = meta["intr"]
    return fx, fy, cx, cy, int(w), int(h)


def test_exp_so3_adjoint_matches_finite_differences():
    from oracle import gridsurf_oracle as O
    rng = np.random.default_rng(0)
    Eb = rng.normal(size=(3, 3))
    for scale in (0.0, 3e-5, 2e-3, 0.7):  # series branch (|nu| < 1e-4) and closed form
        nu = rng.normal(size=3) * scale
        E, aux = O.exp_so3_graph(nu)
        g = O.exp_so3_adjoint(nu, aux, Eb)
        h = 1e-7
        fd = np.zeros(3)
        for a in range(3):
            e = np.zeros(3)
            e[a] = h
            fd[a] = ((O.exp_so3_graph(nu + e)[0] - O.exp_so3_graph(nu - e)[0]) * Eb).sum() / (2 * h)
        assert np.abs(g - fd).max() <= 1e-6 * max(np.abs(fd).max(), 1.0), (scale, g, fd)
        np.testing.assert_allclose(E, O.exp_so3_data(nu), rtol=0, atol=1e-15)


@pytest.mark.parametrize("precision", ["double", "single"])
def test_oracle_pose_refinement_matches_reference(precision):
    from _golden import OracleDataset, cfg_ns
    from oracle import gridsurf_oracle as O
    a, meta = golden(precision)
    fx, fy, cx, cy, w, h = _intr(meta)
    intr = SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)
    ds = OracleDataset(a["colors_u8"], a["depths_u16"], a["poses"], intr)
    c = dict(meta["cfg"])
    c["voxel_sizes"] = tuple(c["voxel_sizes"])
    cfg = cfg_ns(precision=precision, **c)
    cfg.weights.smooth_count = meta["smooth_count"]
    dt = np.float64 if precision == "double" else np.float32
    P = O.create_params(meta["lo"], meta["hi"], ds.poses, seed=cfg.seed, voxel_sizes=cfg.voxel_sizes,
                        dtype=dt, refine_poses=True)
    assert P.names() == meta["names"]
    for n, arr in zip(P.names(), P.arrays()):
        np.testing.assert_array_equal(arr, a[f"init_{n}"])
    opt = O.Adam(P.arrays(), P.lrs())
    if precision == "single":
        g_ref, p_ref = ref_f32_budget(meta["names"])
    for it in range(meta["iters"]):
        R = O.train_step(P, opt, ds, cfg, it)
        for k in PART_KEYS:
            e = abs(R["parts"][k] - meta["parts"][it][k]) / max(abs(meta["parts"][it][k]), 1e-300)
            assert e <= (1e-12 if precision == "double" else max(4 * p_ref[it][k], 1e-5)), (it, k, e)
        for n in meta["names"]:
            e = rel(R["grads"][n], a[f"it{it}_grad_{n}"])
            tol = 1e-11 if precision == "double" else max(4 * g_ref[it][n], 2e-4)
            assert e <= tol, (it, n, e)
    np.testing.assert_allclose(P.R0, a["final_R0"], rtol=0, atol=1e-12 if precision == "double" else 1e-6)
    for n, arr in zip(P.names(), P.arrays()):
        assert rel(arr, a[f"final_{n}"]) <= (1e-11 if precision == "double" else 1e-3), n


# ---------------------------------------------------------------------------
# device


def _device_setup(precision):
    import torch
    from paper_2206_14735_b200 import data, optimizer
    from paper_2206_14735_b200.camera import Intrinsics
    a, meta = golden(precision)
    ds = data.Dataset(a["colors_u8"], a["depths_u16"], a["poses"], Intrinsics(*_intr(meta)))
    c = dict(meta["cfg"])
    c["voxel_sizes"] = tuple(c["voxel_sizes"])
    cfg = optimizer.TrainConfig(precision=precision, **c)
    cfg.weights.smooth_count = meta["smooth_count"]
    model = optimizer.build_model(ds, cfg, skip_init=True, device=torch.device("cuda", 0))
    return a, meta, ds, cfg, model


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["double", "single"])
def test_device_pose_refinement_matches_reference(precision):
    from paper_2206_14735_b200 import optimizer, renderer, sampler, seeds
    a, meta, ds, cfg, model = _device_setup(precision)
    names = model.param_names()
    assert names == meta["names"]
    for n, p in zip(names, model.parameters()):
        np.testing.assert_array_equal(p.numpy(), a[f"init_{n}"])
    opt = optimizer.make_optimizer(model, cfg)
    if precision == "single":
        g_ref, p_ref = ref_f32_budget(names)
    # float32: the pose gradients at this state are ill-conditioned (see
    # test_device_pose_kernels_single), Adam steps the poses by +-lr either way,
    # so float32 trajectories part after the first update: one iteration
    for it in range(meta["iters"] if precision == "double" else 1):
        batch = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, it), cfg.batch_rays,
                                       near=cfg.near, far=cfg.max_depth)
        total, parts, extras = renderer.train_objective(model, ds, batch, it, cfg)
        grads = renderer.grad(total, model.parameters())
        for k in PART_KEYS:
            e = abs(parts[k] - meta["parts"][it][k]) / max(abs(meta["parts"][it][k]), 1e-300)
            assert e <= (1e-11 if precision == "double" else max(4 * p_ref[it][k], 1e-5)), (it, k, e)
        for n, g in zip(names, grads):
            if precision == "single" and is_pose(n):
                continue  # see test_device_pose_kernels_single
            e = rel(g.detach().cpu().numpy(), a[f"it{it}_grad_{n}"])
            tol = 1e-9 if precision == "double" else max(4 * g_ref[it][n], 2e-4)
            assert e <= tol, (it, n, e)
        opt.step(grads)
        if (it + 1) % cfg.pose_refresh_every == 0:
            for p in model.poses:
                p.refresh()
    if precision == "single":
        return
    R0 = np.stack([p.R0 for p in model.poses])
    np.testing.assert_allclose(R0, a["final_R0"], rtol=0, atol=1e-10 if precision == "double" else 1e-5)
    for n, p in zip(names, model.parameters()):
        assert rel(p.numpy(), a[f"final_{n}"]) <= (1e-9 if precision == "double" else 1e-3), n


@pytest.mark.gpu
def test_device_pose_kernels_single():
    """float32 pose gradients, component parity.  At this state (random init,
    phi ~ 1e-5 everywhere) sigma_{i+1}/sigma_i sits at 1 and the clamp gates of
    the rendering adjoint flip with float32 rounding, so the END-TO-END float32
    pose gradient is ill-conditioned: the reference's own single-vs-double
    distance is up to 4% (nu2) and single-vs-single between two float32
    implementations larger.  The double-precision test above pins the
    end-to-end semantics; here the float32 kernels (gsb_pose_grad) are pinned
    given the step's own sampled depths and adjoints, against the oracle's
    restatement evaluated in float64 on the same float32 parameters."""
    import torch
    from oracle import gridsurf_oracle as O
    from paper_2206_14735_b200 import optimizer, renderer, sampler, seeds
    from paper_2206_14735_b200.renderer import engine_for
    a, meta, ds, cfg, model = _device_setup("single")
    opt = optimizer.make_optimizer(model, cfg)
    names = model.param_names()
    for it in range(3):
        batch = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, it), cfg.batch_rays,
                                       near=cfg.near, far=cfg.max_depth)
        # oracle parameters = the device's float32 values, evaluated in float64
        P = O.create_params(meta["lo"], meta["hi"], a["poses"], seed=cfg.seed, voxel_sizes=cfg.voxel_sizes,
                            dtype=np.float64, refine_poses=True)
        for arr, p in zip(P.arrays(), model.parameters()):
            arr[...] = p.numpy().astype(np.float64)
        P.R0 = np.stack([p.R0 for p in model.poses])
        total, parts, extras = renderer.train_objective(model, ds, batch, it, cfg)
        grads = renderer.grad(total, model.parameters())
        ws = [v for k, v in engine_for(model, ds)._ws.items() if not (isinstance(k, tuple) and k[0] == "pose")][0]
        M, N = cfg.batch_rays, extras["samples_per_ray"]
        dep = ws["depths"][:, :N].cpu().numpy()
        pbar = ws["pbar"][:M * N].cpu().numpy().astype(np.float64).reshape(M, N)
        ubar = ws["ubar"][:M * N].cpu().numpy().astype(np.float64).reshape(M, N, 3)
        cbar = ws["cbar"].cpu().numpy().astype(np.float64).reshape(M, N, 3)
        lo, hi = model.grid.clamp_box()
        ref, _ = O.pose_grads_given(P, batch, dep, pbar, ubar, cbar, lo, hi)
        for n, g in zip(names, grads):
            if is_pose(n):
                e = rel(g.detach().cpu().numpy(), ref[n])
                assert e <= 2e-3, (it, n, e)
        opt.step(grads)
        if (it + 1) % cfg.pose_refresh_every == 0:
            for p in model.poses:
                p.refresh()


@pytest.mark.gpu
def test_trainer_pose_refinement_and_checkpoint(tmp_path):
    """The pipelined Trainer (device smoothness points, refresh inside the
    loop) reaches the reference's final state; a GSURFCKPT1 round trip keeps
    R0, nu, t, the trainable flags and the Adam moments."""
    from paper_2206_14735_b200 import optimizer
    a, meta, ds, cfg, model = _device_setup("double")
    opt = optimizer.make_optimizer(model, cfg)
    T = optimizer.Trainer(model, ds, cfg, opt)
    for it in range(meta["iters"]):
        T.launch(it, slot=it % 2)
        T.parts(it % 2)
    np.testing.assert_allclose(np.stack([p.R0 for p in model.poses]), a["final_R0"], rtol=0, atol=1e-10)
    for n, p in zip(model.param_names(), model.parameters()):
        assert rel(p.numpy(), a[f"final_{n}"]) <= 1e-9, n
    path = str(tmp_path / "pose.gsck")
    optimizer.save_model(path, model, cfg, meta["iters"], opt)
    m2, cfg2, it2, opt2 = optimizer.load_model(path)
    assert it2 == meta["iters"] and cfg2.refine_poses
    assert [p.trainable for p in m2.poses] == [p.trainable for p in model.poses]
    np.testing.assert_array_equal(np.stack([p.R0 for p in m2.poses]), np.stack([p.R0 for p in model.poses]))
    for n, p, q in zip(model.param_names(), model.parameters(), m2.parameters()):
        np.testing.assert_array_equal(p.numpy(), q.numpy())
    for m_a, m_b in zip(opt.m, opt2.m):
        np.testing.assert_array_equal(m_a.cpu().numpy(), m_b.cpu().numpy())
