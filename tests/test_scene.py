"""Data path: synthetic RGB-D frames against the
reference renderer's own output (gs/scenegen.py:290-368; fixtures from
tests/golden/make_golden_scene.py, make_golden_c1.py, make_golden.py).

* CPU: the oracle's numpy renderer (oracle/scene_host.py, the device's
  postfix program evaluated with numpy) reproduces every pixel.
* GPU: gsb_render_frames (one thread per pixel, the CSG tree as a postfix
  program) reproduces every pixel -- clean frames at c1 (20 x 160x120) and
  the small case, depth noise + all three dropouts, the thin slab."""

import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def cases():
    from paper_2206_14735_b200 import camera
    z = np.load(os.path.join(HERE, "golden", "scene_frames.npz"))
    meta = json.loads(z["meta_json"].tobytes().decode())
    out = []
    for name, m in meta.items():
        fx, fy, cx, cy, w, h = m["intr"]
        kw = dict(m["kw"])
        if "dropout_rect" in kw:
            kw["dropout_rect"] = tuple(kw["dropout_rect"])
        out.append((name, m["scene"], camera.Intrinsics(fx, fy, cx, cy, int(w), int(h)), z[f"{name}_poses"],
                    kw, z[f"{name}_colors_u8"], z[f"{name}_depths_u16"]))
    for gname, frames, w, h in (("c1_double", 20, 160, 120), ("small_double", 6, 32, 24)):
        g = np.load(os.path.join(HERE, "golden", f"{gname}.npz"))
        f = 0.5 * w / np.tan(np.radians(35.0))
        out.append((gname, "sphere_in_box", camera.Intrinsics(f, f, w / 2.0, h / 2.0, w, h), g["poses"], {},
                    g["colors_u8"], g["depths_u16"]))
    return out


def _check(name, cols, deps, ref_c, ref_d):
    assert cols.shape == ref_c.shape and deps.shape == ref_d.shape
    bad_c = int((cols != ref_c).sum())
    bad_d = int((deps != ref_d).sum())
    assert bad_c == 0 and bad_d == 0, (name, bad_c, bad_d, np.abs(deps.astype(int) - ref_d).max())


@pytest.mark.parametrize("which", ["corrupt", "slab", "small_double", "c1_double"])
def test_host_render_matches_reference(which):
    from oracle import scene_host
    from paper_2206_14735_b200 import scenes
    for name, scene, intr, poses, kw, ref_c, ref_d in cases():
        if name != which:
            continue
        cols, deps = scene_host.render_sequence(getattr(scenes, scene)(), poses, intr, max_t=8.0, **kw)
        _check(name, cols, deps, ref_c, ref_d)


@pytest.mark.gpu
def test_device_render_matches_reference():
    from paper_2206_14735_b200 import scenes
    for name, scene, intr, poses, kw, ref_c, ref_d in cases():
        cols, deps = scenes.render_frames_device(getattr(scenes, scene)(), poses, intr, max_t=8.0, **kw)
        _check(name, cols.cpu().numpy(), deps.cpu().numpy().view(np.uint16), ref_c, ref_d)


@pytest.mark.gpu
def test_device_render_dataset_is_a_dataset():
    from oracle import scene_host
    from paper_2206_14735_b200 import scenes
    ds = scenes.render_dataset(scenes.sphere_in_box(), scenes.orbit_trajectory(3),
                               scenes.fov_intrinsics(40, 30))
    cols, deps = scene_host.render_sequence(scenes.sphere_in_box(), scenes.orbit_trajectory(3),
                                            scenes.fov_intrinsics(40, 30))
    np.testing.assert_array_equal(ds.colors_u8, cols)
    np.testing.assert_array_equal(ds.depths_mm, deps)
    assert ds.n_valid == int((deps > 0).sum())


def test_scene_program_flattening_and_validation():
    """The CSG tree becomes a postfix program (Complement -> NEG, Union -> MIN
    over its children in order); the library rejects malformed programs
    before launching anything (no GPU needed)."""
    import ctypes as C
    from paper_2206_14735_b200 import _lib, scenes
    S = scenes.scene_program(scenes.sphere_in_box())
    ops = [(S.op[i][0], S.op[i][1]) for i in range(S.n_ops)]
    assert ops == [(0, 0), (1, 0), (0, 1), (2, 2)]
    assert S.prim[0][0] == 1.0 and S.prim[1][0] == 0.0  # room box, then the ball
    assert S.prim[0][13] == 0.25  # checker size of the room
    L = _lib.lib()
    O = _lib.RenderOpts()
    dummy = C.c_void_p(16)
    bad = scenes.scene_program(scenes.scannet_room())
    bad.op[bad.n_ops - 1][1] = 9  # MIN over more entries than the stack holds
    rc = L.gsb_render_frames(C.byref(bad), dummy, 1, 4, 4, 1.0, 1.0, 2.0, 2.0, 8.0, None, 0.0, C.byref(O),
                             dummy, dummy, None)
    assert rc == -1  # GSB_E_ARG
    S.n_ops = 3  # leaves two entries on the stack
    rc = L.gsb_render_frames(C.byref(S), dummy, 1, 4, 4, 1.0, 1.0, 2.0, 2.0, 8.0, None, 0.0, C.byref(O),
                             dummy, dummy, None)
    assert rc == -1
