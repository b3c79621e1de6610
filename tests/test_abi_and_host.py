"""CPU tests: the C-ABI library loads and exports what include/gsb.h
declares; host-side logic (init streams, batch ids, smoothness draws,
checkpoints, learning-rate segments) matches the reference/golden."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from _golden import ROOT, load, rel_maxnorm
from oracle import gridsurf_oracle as O

HEADER = os.path.join(ROOT, "include", "gsb.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|uint64_t)\s+(gsb_\w+)\s*\(", src)))


def test_header_declarations_match_binding():
    from paper_2206_14735_b200 import _lib
    assert declared_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_2206_14735_b200 import _lib
    L = _lib.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert L.gsb_version() == 1


def test_struct_sizes_are_stable():
    from paper_2206_14735_b200 import _lib
    # layout of the ABI structs as compiled (x86-64): guards accidental drift
    assert C.sizeof(_lib.Level) == 56
    assert C.sizeof(_lib.Pcg64) == 32
    assert C.sizeof(_lib.Model) == 8 + 56 * _lib.MAX_LEVELS + 56 + 24 + 48 + 16


def _cpu_model(G):
    from paper_2206_14735_b200 import optimizer
    cfg = optimizer.TrainConfig(precision=G.cfg.precision, **{
        k: v for k, v in G.meta["cfg"].items() if k not in ("bounds", "voxel_sizes")},
        voxel_sizes=G.cfg.voxel_sizes, bounds=G.cfg.bounds)
    cfg.weights.smooth_count = G.meta["smooth_count"]
    from paper_2206_14735_b200 import data
    ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"], G.ds.intrinsics)
    model = optimizer.build_model(ds, cfg, skip_init=True, device="cpu")
    return model, ds, cfg


@pytest.mark.parametrize("case", ["tiny", "small"])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_build_model_init_matches_reference(case, precision):
    G = load(case, precision)
    model, ds, cfg = _cpu_model(G)
    np.testing.assert_allclose(model.grid.lo, G.meta["lo"], rtol=0, atol=0)
    for n, p in zip(model.param_names(), model.parameters()):
        ref = G.a[f"init_{n}"]
        got = p.numpy()
        assert got.shape == ref.shape, n
        np.testing.assert_array_equal(got, ref, err_msg=n)


@pytest.mark.parametrize("case", ["tiny", "small"])
def test_host_draws_match_reference(case):
    from paper_2206_14735_b200 import engine, sampler, seeds
    G = load(case, "double")
    model, ds, cfg = _cpu_model(G)
    it = G.meta["iteration"]
    b = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, it), cfg.batch_rays,
                               near=cfg.near, far=cfg.max_depth)
    for k in ("frame_ids", "pixels", "color", "depth_ray", "valid", "dir_cam"):
        np.testing.assert_array_equal(getattr(b, k), G.a[f"batch_{k}"], err_msg=k)
    # smoothness set through the prefix-count valid-pixel index
    P = O.create_params(G.meta["lo"], G.meta["hi"], G.ds.poses, seed=cfg.seed,
                        voxel_sizes=cfg.voxel_sizes, geom_width=cfg.geom_feat_dim,
                        color_width=cfg.color_feat_dim)
    ref = O.draw_smooth_points(P, G.ds, 64, 0.16, 0.004, O.substream(cfg.seed, O.SMOOTH, it))
    got = engine.draw_smooth_points(model, ds, 64, 0.16, 0.004,
                                    seeds.substream(cfg.seed, seeds.SMOOTH, it))
    np.testing.assert_array_equal(got[0], ref[0])
    np.testing.assert_array_equal(got[1], ref[1])


def test_valid_pixel_index_matches_nonzero():
    from paper_2206_14735_b200 import data
    rng = np.random.default_rng(0)
    dep = (rng.uniform(size=(3, 7, 11)) > 0.4).astype(np.uint16) * 1234
    col = np.zeros((3, 7, 11, 3), np.uint8)
    from paper_2206_14735_b200.camera import Intrinsics
    ds = data.Dataset(col, dep, np.tile(np.eye(4), (3, 1, 1)), Intrinsics(5, 5, 5, 3, 11, 7))
    f, v, u = np.nonzero(dep > 0)
    k = np.arange(f.size)
    gf, gv, gu = ds.valid_pixel(k)
    np.testing.assert_array_equal(gf, f)
    np.testing.assert_array_equal(gv, v)
    np.testing.assert_array_equal(gu, u)


def test_pcg64_state_export():
    from paper_2206_14735_b200 import _lib, seeds
    g = seeds.substream(3, seeds.STRATIFY, 7)
    st = _lib.Pcg64.from_generator(g)
    s, inc = seeds.pcg64_state(3, seeds.STRATIFY, 7)
    assert (st.state_hi << 64) | st.state_lo == s
    assert (st.inc_hi << 64) | st.inc_lo == inc


def test_checkpoint_round_trip_cpu(tmp_path):
    from paper_2206_14735_b200 import optimizer
    G = load("tiny", "single")
    model, ds, cfg = _cpu_model(G)
    path = str(tmp_path / "m.gsck")
    optimizer.save_model(path, model, cfg, 7)
    m2, cfg2, it, opt = optimizer.load_model(path, device="cpu")
    assert it == 7 and opt is None
    for a, b in zip(model.parameters(), m2.parameters()):
        np.testing.assert_array_equal(a.numpy(), b.numpy())
    assert cfg2.voxel_sizes == cfg.voxel_sizes


def test_checkpoint_readable_by_reference_layout(tmp_path):
    """Header/array names follow gs/optimizer.py:243-280."""
    from paper_2206_14735_b200 import checkpoint, optimizer
    G = load("small", "double")
    model, ds, cfg = _cpu_model(G)
    path = str(tmp_path / "m.gsck")
    optimizer.save_model(path, model, cfg, 3)
    header, arrays = checkpoint.read_container(path)
    assert header["kind"] == "gridsurf-model"
    assert header["array_order"][:len(G.meta["names"])] == G.meta["names"]
    assert [l["dims"] for l in header["grid"]["levels"]][0] == list(model.grid.levels[0].geom.dims)
    # np.ascontiguousarray (gs/checkpoint.py:27) stores the 0-d log_s as shape (1,)
    assert arrays["log_s"].shape == (1,)


def test_adam_segments():
    from paper_2206_14735_b200 import optimizer
    G = load("small", "single")
    model, ds, cfg = _cpu_model(G)
    opt = optimizer.make_optimizer(model, cfg)
    b, l = opt._segments()
    assert b[0] == 0 and l[0] == cfg.lr_grids
    assert b[1] == model.arena["geom_w0"].offset and l[1] == cfg.lr_decoders
    assert l[2:] in ([], [0.0])  # the arena's alignment tail (no parameter) has lr 0
    # geometric-init style subset: grids + geometry net only
    params = [lv.features for lv in model.grid.levels] + model.geom_net.parameters()
    opt2 = optimizer.Adam(params, [1e-2] * len(model.grid.levels) + [1e-3] * 6)
    b2, l2 = opt2._segments()
    assert l2[:4] == [1e-2, 0.0, 1e-3, 0.0] and l2[4:] in ([], [0.0])
    assert b2[1] == model.grid.color.features.offset
    assert b2[3] == model.arena["color_w0"].offset
    for x in b2:
        assert x % 4 == 0


def test_oracle_matches_reference_objective_double_small():
    """Re-run of the golden check through the test helper (cheap smoke)."""
    G = load("small", "double")
    from _golden import oracle_params
    P = oracle_params(G)
    it = G.meta["iteration"]
    batch = O.draw_ray_batch(G.ds, O.substream(G.cfg.seed, O.RAYS, it), G.cfg.batch_rays)
    R = O.train_objective(P, G.ds, batch, it, G.cfg)
    assert R["parts"]["total"] == G.meta["parts"]["total"]
    assert rel_maxnorm(R["grads"]["level3"], G.a["grad_level3"]) < 1e-12


def test_draw_prefetcher_order_and_errors():
    from paper_2206_14735_b200.optimizer import DrawPrefetcher

    def fn(it):
        if it == 8:
            raise ValueError("boom")
        return it * 2

    p = DrawPrefetcher(fn, 5)
    assert [p.get(i) for i in (5, 6, 7)] == [10, 12, 14]
    import pytest
    with pytest.raises(ValueError):
        p.get(8)
    p.close()
    q = DrawPrefetcher(lambda it: it, 0)
    q.get(0)
    with pytest.raises(RuntimeError):
        q.get(5)  # out of order is an error, not a silent mismatch
    q.close()


def test_product_path_fails_loudly_without_extension(monkeypatch, tmp_path):
    """No CPU fallback: with the CUDA extension absent the library loader and
    a model build raise instead of computing anything on the host."""
    from paper_2206_14735_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing_gsb.so"))
    with pytest.raises(_lib.GsbError):
        _lib.lib()


def test_build_model_refuses_cpu_device():
    """The step has no host implementation: build_model needs CUDA."""
    import torch
    from paper_2206_14735_b200 import optimizer
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    G = load("tiny", "single")
    cfg = optimizer.TrainConfig(precision="single", batch_rays=8)
    from paper_2206_14735_b200 import data
    ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"], G.ds.intrinsics)
    with pytest.raises(RuntimeError, match="CUDA"):
        optimizer.build_model(ds, cfg, skip_init=True)


def test_foreign_batch_checks():
    """A reference-shaped batch (per-ray arrays) is accepted only when its
    bounds are uniform and its targets are the dataset's (renderer.py)."""
    from types import SimpleNamespace
    from _golden import load
    from paper_2206_14735_b200 import camera, data, sampler
    from paper_2206_14735_b200.renderer import _check_foreign_batch
    G = load("tiny", "double")
    i = G.ds.intrinsics
    ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"],
                      camera.Intrinsics(i.fx, i.fy, i.cx, i.cy, i.width, i.height))
    b = sampler.draw_ray_batch(ds, np.random.default_rng(0), 16, near=0.01, far=8.0)
    ref = SimpleNamespace(**{k: getattr(b, k) for k in ("frame_ids", "pixels", "color", "depth_ray",
                                                        "valid", "dir_cam", "near", "far")})
    assert _check_foreign_batch(ref, ds) == (0.01, 8.0)
    bad = SimpleNamespace(**vars(ref))
    bad.far = ref.far.copy()
    bad.far[3] = 5.0
    with pytest.raises(ValueError, match="near/far"):
        _check_foreign_batch(bad, ds)
    bad = SimpleNamespace(**vars(ref))
    bad.color = ref.color + 0.01
    with pytest.raises(ValueError, match="color"):
        _check_foreign_batch(bad, ds)
