"""The training loop (gs/optimizer.py:331-391) end to end: loss-log CSV
schema and rows, periodic ``ckpt_%06d.gsck`` cadence, the final checkpoint,
resume appending to the log, DivergenceError before the diverging step's
update, and GSURFCKPT1 files the reference's own ``load_model``
(gs/optimizer.py:283-325) reads back."""

import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from _golden import load  # noqa: E402

REF_SRC = "/root/reference/pkg/src"
REF_CSV_HEADER = "iter,total,rgb,depth,sdf,fs,eik,smooth,s\n"  # gs/optimizer.py:331


def small_setup(precision="single", **kw):
    from paper_2206_14735_b200 import camera, data, optimizer
    G = load("small", "double")
    i = G.ds.intrinsics
    ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"],
                      camera.Intrinsics(i.fx, i.fy, i.cx, i.cy, i.width, i.height))
    cfg = optimizer.TrainConfig(precision=precision, bounds=G.cfg.bounds, voxel_sizes=G.cfg.voxel_sizes,
                                batch_rays=64, seed=G.cfg.seed, sphere_radius_scale=0.4, **kw)
    return ds, cfg


def _reference_optimizer():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    from gridsurf import optimizer as RO
    return RO


def test_reference_load_model_reads_our_checkpoint(tmp_path):
    """A checkpoint written by save_model (host arena on the CPU: no compute)
    loads in the reference: parameters, Adam moments and step counts,
    iteration and config."""
    import torch
    from paper_2206_14735_b200 import optimizer
    RO = _reference_optimizer()
    ds, cfg = small_setup()
    model = optimizer.build_model(ds, cfg, skip_init=True, device="cpu")
    opt = optimizer.make_optimizer(model, cfg)
    g = torch.Generator().manual_seed(1)
    opt.m_arena.copy_(torch.randn(opt.m_arena.shape, generator=g))
    opt.v_arena.copy_(torch.rand(opt.v_arena.shape, generator=g))
    opt.t = [7] * len(opt.t)
    path = str(tmp_path / "ours.gsck")
    optimizer.save_model(path, model, cfg, 7, opt)
    rm, rcfg, rit, ropt = RO.load_model(path)
    assert rit == 7 and rcfg.batch_rays == cfg.batch_rays and rcfg.precision == "single"
    for a, b, n in zip(rm.parameters(), model.parameters(), model.param_names()):
        np.testing.assert_array_equal(a.data.reshape(-1), b.numpy().reshape(-1), err_msg=n)
    for i in range(len(opt.t)):
        np.testing.assert_array_equal(ropt.m[i].reshape(-1), opt.m[i].numpy().reshape(-1))
        np.testing.assert_array_equal(ropt.v[i].reshape(-1), opt.v[i].numpy().reshape(-1))
        assert ropt.t[i] == 7
    # and back: the reference's own checkpoint of that model loads here
    path2 = str(tmp_path / "ref.gsck")
    RO.save_model(path2, rm, rcfg, 7, ropt)
    m2, cfg2, it2, opt2 = optimizer.load_model(path2, device="cpu")
    assert it2 == 7
    for a, b in zip(m2.parameters(), model.parameters()):
        np.testing.assert_array_equal(a.numpy(), b.numpy())


def _rows(path):
    with open(path) as f:
        lines = f.readlines()
    return lines[0], [ln.rstrip("\n").split(",") for ln in lines[1:]]


@pytest.mark.gpu
def test_train_csv_checkpoints_resume(tmp_path):
    from paper_2206_14735_b200 import optimizer
    ds, cfg = small_setup(iterations=6, checkpoint_every=2, init_steps=400, init_tol=0.05)
    out = str(tmp_path / "run")
    model, final = optimizer.train(ds, cfg, out)
    header, rows = _rows(os.path.join(out, "loss_log.csv"))
    assert header == REF_CSV_HEADER
    assert [int(r[0]) for r in rows] == list(range(6))
    assert all(len(r) == 9 and all(np.isfinite(float(x)) for x in r[1:]) for r in rows)
    for k in (2, 4, 6):
        assert os.path.exists(os.path.join(out, f"ckpt_{k:06d}.gsck"))
    assert final == os.path.join(out, "ckpt_final.gsck")
    m6, _, it6, opt6 = optimizer.load_model(os.path.join(out, "ckpt_000006.gsck"))
    mf, _, itf, optf = optimizer.load_model(final)
    assert it6 == 6 and itf == 6 and optf.t == [6] * len(optf.t)
    for a, b in zip(mf.parameters(), model.parameters()):
        np.testing.assert_array_equal(a.numpy(), b.numpy())

    # resume from iteration 4 in a copy of the run directory: the log is
    # appended from iteration 4, and iterations 4-5 redo the same steps
    import shutil
    res = str(tmp_path / "resumed")
    shutil.copytree(out, res)
    cfg8 = optimizer.TrainConfig(**{**cfg.__dict__, "iterations": 8})
    model8, final8 = optimizer.train(ds, cfg8, res, resume=os.path.join(res, "ckpt_000004.gsck"))
    header, rows8 = _rows(os.path.join(res, "loss_log.csv"))
    assert [int(r[0]) for r in rows8] == list(range(6)) + list(range(4, 8))
    for a, b in zip(rows8[4:6], rows8[6:8]):  # same iteration, same batch, same state
        np.testing.assert_allclose([float(x) for x in a[1:]], [float(x) for x in b[1:]], rtol=2e-5)
    m6r, _, _, _ = optimizer.load_model(os.path.join(res, "ckpt_000006.gsck"))
    for n, a, b in zip(m6.param_names(), m6r.parameters(), m6.parameters()):
        # float32 atomics make two runs differ in the last bits; Adam can turn
        # a gradient that is rounding noise into a +-lr step, so the bound is
        # on almost every element plus a loose cap
        x, y = a.numpy().astype(np.float64), b.numpy().astype(np.float64)
        d = np.abs(x - y).reshape(-1)
        assert np.quantile(d, 0.999) <= 1e-5 * max(np.abs(y).max(), 1e-12), n
        assert d.max() <= 4 * cfg.lr_grids, n
    _, _, it8, _ = optimizer.load_model(final8)
    assert it8 == 8


@pytest.mark.gpu
def test_train_raises_divergence_before_the_update(tmp_path):
    """A total above divergence_threshold raises DivergenceError at that
    iteration; no row is logged for it and no update is applied (the device
    guard skips the Adam launches already enqueued)."""
    from paper_2206_14735_b200 import optimizer
    ds, cfg = small_setup(iterations=5, checkpoint_every=1000, init_steps=400, init_tol=0.05,
                          divergence_threshold=-1.0)
    out = str(tmp_path / "div")
    with pytest.raises(optimizer.DivergenceError, match="iteration 0"):
        optimizer.train(ds, cfg, out)
    header, rows = _rows(os.path.join(out, "loss_log.csv"))
    assert header == REF_CSV_HEADER and rows == []


@pytest.mark.gpu
def test_trainer_guard_skips_update_and_rolls_back():
    """Trainer-level view of the same guard: parameters after a diverged
    launch equal the parameters before it."""
    from paper_2206_14735_b200 import optimizer
    ds, cfg = small_setup(divergence_threshold=-1.0)
    model = optimizer.build_model(ds, cfg, skip_init=True)
    opt = optimizer.make_optimizer(model, cfg)
    before = [p.numpy().copy() for p in model.parameters()]
    T = optimizer.Trainer(model, ds, cfg, opt)
    T.launch(0, slot=0)
    T.launch(1, slot=1)
    T.parts(1)
    for a, b in zip(before, model.parameters()):
        np.testing.assert_array_equal(a, b.numpy())
    assert int(opt.status[5].item()) == 1  # GSB_ST_DIVERGED


@pytest.mark.gpu
def test_trainer_overlapped_adam_is_bit_identical():
    """The side-stream colour-grid Adam (optimizer.AdamOverlap, under the
    next step's sampling phase) gives the fused launch's parameters and
    moments bit for bit (deterministic scatter mode on both, so the
    gradients themselves are run-to-run identical)."""
    from paper_2206_14735_b200 import optimizer
    from paper_2206_14735_b200.renderer import engine_for
    ds, cfg = small_setup()
    out = []
    for overlap in (False, True):
        model = optimizer.build_model(ds, cfg, skip_init=True)
        opt = optimizer.make_optimizer(model, cfg)
        T = optimizer.Trainer(model, ds, cfg, opt, overlap_adam=overlap)
        T.engine.deterministic = True
        assert engine_for(model, T.dataset) is T.engine
        for it in range(4):
            T.launch(it, slot=it % 2)
            T.parts(it % 2)
        T.drain()
        out.append(([p.numpy() for p in model.parameters()],
                    opt.m_arena.cpu().numpy(), opt.v_arena.cpu().numpy()))
    (p0, m0, v0), (p1, m1, v1) = out
    for a, b in zip(p0, p1):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(m0, m1)
    np.testing.assert_array_equal(v0, v1)
