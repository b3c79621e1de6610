"""Mesh extraction and metrics (gs/mesher.py) against golden vectors produced
by running the reference's own mesher (tests/golden/make_golden_mesh.py; its
marching cubes is the oracle's, see there), plus table / watertightness
checks of the generated marching-cubes table."""

import json
import os
import sys
from collections import Counter
from types import SimpleNamespace

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from _golden import load  # noqa: E402


def golden():
    z = np.load(os.path.join(HERE, "golden", "mesh_small.npz"))
    a = {k: z[k] for k in z.files}
    meta = json.loads(a.pop("meta_json").tobytes().decode())
    metrics = json.loads(a.pop("metrics_json").tobytes().decode())
    return a, meta, metrics


def _mesh(v, f):
    from paper_2206_14735_b200.mesher import TriangleMesh
    return TriangleMesh(v, f)


def test_mc_table_is_watertight_on_random_volumes():
    from oracle import gridsurf_oracle as O
    rng = np.random.default_rng(3)
    for _ in range(4):
        vol = rng.normal(size=(8, 7, 6)).astype(np.float32)
        vol[[0, -1], :, :] = 1
        vol[:, [0, -1], :] = 1
        vol[:, :, [0, -1]] = 1
        v, f = O.marching_cubes(vol)
        key = {tuple(np.round(x, 12)) for x in v}
        vid = {k: i for i, k in enumerate(sorted(key))}
        fi = np.array([[vid[tuple(np.round(v[j], 12))] for j in t] for t in f])
        und = Counter(frozenset((a, b)) for t in fi for a, b in ((t[0], t[1]), (t[1], t[2]), (t[2], t[0])))
        dire = Counter((a, b) for t in fi for a, b in ((t[0], t[1]), (t[1], t[2]), (t[2], t[0])))
        assert set(und.values()) == {2} and set(dire.values()) == {1}


def test_subdivide_matches_reference_exactly():
    from paper_2206_14735_b200.mesher import subdivide_to_edge_length
    a, _, _ = golden()
    sub = subdivide_to_edge_length(_mesh(a["mesh_v"], a["mesh_f"]), 0.06)
    np.testing.assert_array_equal(sub.faces, a["sub_f"])
    np.testing.assert_array_equal(sub.vertices, a["sub_v"])


def test_sample_surface_matches_reference_stream():
    from paper_2206_14735_b200.mesher import sample_surface
    a, meta, _ = golden()
    pts, _ = sample_surface(_mesh(a["mesh_v"], a["mesh_f"]), meta["density"])
    np.testing.assert_array_equal(pts, a["nn_q"])


def test_mesh_io_roundtrip(tmp_path):
    from paper_2206_14735_b200.mesher import load_mesh, save_mesh
    a, _, _ = golden()
    m = _mesh(a["mesh_v"][:300], a["mesh_f"][:100])
    for name, binary in (("m.ply", True), ("a.ply", False), ("m.obj", False)):
        p = str(tmp_path / name)
        save_mesh(p, m, binary=binary)
        r = load_mesh(p)
        np.testing.assert_array_equal(r.faces, m.faces)
        tol = 1e-6 if name == "m.ply" else 1e-8
        np.testing.assert_allclose(r.vertices, m.vertices, atol=tol)


# ---------------------------------------------------------------------------- device


def _gpu_model(prefix, precision):
    import torch
    from paper_2206_14735_b200 import data, optimizer
    G = load("small", precision)
    cfg = optimizer.TrainConfig(precision=precision, **{
        k: v for k, v in G.meta["cfg"].items() if k not in ("bounds", "voxel_sizes")},
        voxel_sizes=G.cfg.voxel_sizes, bounds=G.cfg.bounds)
    ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"], G.ds.intrinsics)
    model = optimizer.build_model(ds, cfg, skip_init=True, device=torch.device("cuda", 0))
    a, _, _ = golden()
    for i, l in enumerate(model.grid.levels):
        l.features.set(a[f"{prefix}level{i}"])
    for i, (W, b) in enumerate(model.geom_net.layers):
        W.set(a[f"{prefix}geom_w{i}"])
        b.set(a[f"{prefix}geom_b{i}"])
    return model, ds


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["double", "single"])
def test_sdf_volume_matches_reference(precision):
    from paper_2206_14735_b200.mesher import sdf_volume
    a, meta, _ = golden()
    pre = "d_" if precision == "double" else "s_"
    model, _ = _gpu_model(pre, precision)
    vol, lo, res = sdf_volume(model, meta["res"])
    np.testing.assert_array_equal(lo, a[f"{pre}vol_lo"])
    assert vol.shape == a[f"{pre}vol"].shape
    ref = a[f"{pre}vol"]
    err = np.abs(vol.astype(np.float64) - ref).max() / np.abs(ref).max()
    # double: the volume is float32 storage of a ~1e-12-close phi; single: fp32 MLP order
    assert err <= (1e-7 if precision == "double" else 2e-5), err


@pytest.mark.gpu
def test_marching_cubes_device_equals_oracle_table():
    from paper_2206_14735_b200.mesher import mesh_from_sdf
    a, meta, _ = golden()
    mesh = mesh_from_sdf(a["d_vol"], a["d_vol_lo"], meta["res"])
    np.testing.assert_array_equal(mesh.faces, a["mesh_f"])
    np.testing.assert_array_equal(mesh.vertices, a["mesh_v"])


@pytest.mark.gpu
def test_empty_level_set_raises():
    from paper_2206_14735_b200.mesher import EmptyLevelSetError, mesh_from_sdf
    with pytest.raises(EmptyLevelSetError):
        mesh_from_sdf(np.ones((4, 4, 4), np.float32), np.zeros(3), 0.1)


@pytest.mark.gpu
def test_nearest_neighbors_bit_exact():
    from paper_2206_14735_b200.mesher import nearest_neighbors
    a, _, _ = golden()
    d, i = nearest_neighbors(a["nn_q"], a["nn_ref"], 0.05)
    np.testing.assert_array_equal(d, a["nn_d"])
    np.testing.assert_array_equal(i, a["nn_i"])


@pytest.mark.gpu
def test_evaluate_matches_reference_metrics():
    from paper_2206_14735_b200.mesher import evaluate
    a, meta, metrics = golden()
    rep = evaluate(_mesh(a["mesh_v"], a["mesh_f"]), _mesh(a["gt_v"], a["gt_f"]), threshold=0.05,
                   density=meta["density"])
    for k, v in metrics.items():
        assert getattr(rep, k) == v, (k, getattr(rep, k), v)


@pytest.mark.gpu
def test_cull_mesh_matches_reference():
    from paper_2206_14735_b200 import data
    from paper_2206_14735_b200.mesher import cull_mesh
    a, _, _ = golden()
    G = load("small", "double")
    ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"], G.ds.intrinsics)
    culled = cull_mesh(_mesh(a["mesh_v"], a["mesh_f"]), ds, max_edge=0.12)
    np.testing.assert_array_equal(culled.faces, a["cull_f"])
    np.testing.assert_array_equal(culled.vertices, a["cull_v"])


@pytest.mark.gpu
def test_extract_mesh_end_to_end_reaches_reference_quality():
    """Device extraction of the pre-fit model vs the analytic sphere: the
    reference pipeline's Chamfer / F-score (golden) within 1e-6."""
    from paper_2206_14735_b200.mesher import evaluate, extract_mesh
    a, meta, metrics = golden()
    model, _ = _gpu_model("d_", "double")
    mesh = extract_mesh(model, resolution=meta["res"])
    rep = evaluate(mesh, _mesh(a["gt_v"], a["gt_f"]), threshold=0.05, density=meta["density"])
    assert abs(rep.chamfer_l1 - metrics["chamfer_l1"]) <= 1e-6
    assert abs(rep.f_score - metrics["f_score"]) <= 1e-6
