"""Host (numpy) renderer of the synthetic RGB-D scenes -- TEST INFRASTRUCTURE ONLY.

The product renders frames on the device only (``gsb_render_frames``,
``paper_2206_14735_b200/scenes.py``).  This module is the CPU checker for
that kernel and the dataset source of ``bench.py``'s port fallback (a CPU
leg that must not load the repository's ``.so``).  Only ``tests/`` and
``bench.py``'s CPU legs import it.

It evaluates the same postfix program the device kernel runs (the CSG tree
flattened: PRIM pushes (value, primitive, sign), NEG flips value and sign,
MIN(k) keeps the first minimum of the top k entries), vectorised over all
pixels of a frame.  The per-primitive formulas and the frame pipeline follow
the reference renderer (``gs/scenegen.py``):

    primitive SDFs / normals / albedo   gs/scenegen.py:41-137
    shading                             gs/scenegen.py:151-155
    sphere tracing                      gs/scenegen.py:223-252
    one frame (noise, dropouts, u8/u16) gs/scenegen.py:290-325
    a sequence                          gs/scenegen.py:328-368

with numpy's own operations for each formula, so frames are pixel-identical
to the reference's (``tests/test_scene.py`` against the reference's output).
"""

from __future__ import annotations

import os
import sys
from concurrent.futures import ThreadPoolExecutor
from types import SimpleNamespace

import numpy as np

from .gridsurf_oracle import pixel_rays, ray_to_z_scale, substream

DEPTH_NOISE = 5  # gs/seeds.py:18, the per-frame depth-noise stream tag
_PRIM, _NEG, _MIN = 0, 1, 2


def flatten(root):
    """Scene tree (``paper_2206_14735_b200.scenes`` nodes) -> (prims, ops)."""
    prims, ops = [], []
    stack = [(root, False)]
    # iterative post-order walk: children first, then the node's operator
    while stack:
        node, done = stack.pop()
        kind = type(node).__name__
        if kind in ("Sphere", "Box"):
            prims.append(node)
            ops.append((_PRIM, len(prims) - 1))
        elif done:
            ops.append((_NEG, 0) if kind == "Complement" else (_MIN, len(node.children)))
        elif kind == "Complement":
            stack += [(node, True), (node.child, False)]
        elif kind == "Union":
            stack.append((node, True))
            stack += [(c, False) for c in reversed(node.children)]
        else:
            raise TypeError(f"unsupported scene node {kind}")
    return prims, ops


def _prim_value(p, x):
    c = np.asarray(p.center, dtype=np.float64)
    if type(p).__name__ == "Sphere":
        return np.linalg.norm(x - c, axis=-1) - float(p.radius)
    q = np.abs(x - c) - np.asarray(p.half, dtype=np.float64)
    return np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(q.max(axis=-1), 0.0)


def _prim_normal(p, x):
    c = np.asarray(p.center, dtype=np.float64)
    d = x - c
    if type(p).__name__ == "Sphere":
        return d / np.maximum(np.linalg.norm(d, axis=-1, keepdims=True), 1e-300)
    q = np.abs(d) - np.asarray(p.half, dtype=np.float64)
    sgn = np.sign(d)
    sgn[sgn == 0] = 1.0
    pos = np.maximum(q, 0.0)
    outward = sgn * pos / np.maximum(np.linalg.norm(pos, axis=-1, keepdims=True), 1e-300)
    face = np.zeros_like(x)
    np.put_along_axis(face, np.argmax(q, axis=-1)[..., None], 1.0, axis=-1)
    return np.where((q < 0).all(axis=-1)[..., None], face * sgn, outward)


def _prim_albedo(p, x):
    out = np.broadcast_to(np.asarray(p.albedo, dtype=np.float64), x.shape).copy()
    chk = float(getattr(p, "checker", 0.0))
    if type(p).__name__ == "Box" and chk > 0:
        parity = np.floor(x / chk).sum(axis=-1).astype(np.int64) % 2
        out[parity.astype(bool)] = np.asarray(p.albedo2, dtype=np.float64)
    return out


def evaluate(program, x, need_select=False):
    """Run the postfix program at points x (n, 3): SDF value, and optionally
    the (primitive, sign) each point's value came from."""
    prims, ops = program
    vals, sel, sgn = [], [], []
    for op, arg in ops:
        if op == _PRIM:
            vals.append(_prim_value(prims[arg], x))
            sel.append(np.full(x.shape[0], arg, dtype=np.int64))
            sgn.append(np.ones(x.shape[0]))
        elif op == _NEG:
            vals[-1], sgn[-1] = -vals[-1], -sgn[-1]
        else:
            v, s, g = np.stack(vals[-arg:]), np.stack(sel[-arg:]), np.stack(sgn[-arg:])
            del vals[-arg:], sel[-arg:], sgn[-arg:]
            k = v.argmin(axis=0)[None]
            vals.append(v.min(axis=0))
            sel.append(np.take_along_axis(s, k, axis=0)[0])
            sgn.append(np.take_along_axis(g, k, axis=0)[0])
    if len(vals) != 1:
        raise ValueError("malformed scene program")
    return (vals[0], sel[0], sgn[0]) if need_select else vals[0]


def shade(program, scene, x):
    prims, _ = program
    _, which, sign = evaluate(program, x, need_select=True)
    n = np.zeros_like(x)
    alb = np.zeros_like(x)
    for i, p in enumerate(prims):
        m = which == i
        if m.any():
            n[m] = _prim_normal(p, x[m])
            alb[m] = _prim_albedo(p, x[m])
    n = n * sign[:, None]
    lam = np.maximum(-(n @ np.asarray(scene.light_dir, dtype=np.float64)), 0.0)
    return np.clip(alb * (0.35 + 0.65 * lam[..., None]), 0.0, 1.0)


def trace(program, origins, dirs, max_t, tol=1e-6, max_steps=256):
    """Sphere tracing: march t by the SDF until |sdf| < tol or t > max_t."""
    t = np.zeros(origins.shape[0])
    hit = np.zeros(origins.shape[0], dtype=bool)
    live = np.arange(origins.shape[0])
    for _ in range(max_steps):
        if live.size == 0:
            break
        s = evaluate(program, origins[live] + t[live, None] * dirs[live])
        done = np.abs(s) < tol
        hit[live[done]] = True
        t[live[~done]] += s[~done]
        live = live[~done]
        live = live[~(t[live] > max_t)]
    return t, hit


def render_frame(scene, pose, intr, max_t=8.0, noise_sigma0=0.0, dropout_rect=None,
                 dropout_world=None, dropout_box=None, rng_noise=None, program=None):
    program = program or flatten(scene.root)
    h, w = intr.height, intr.width
    uu, vv = np.meshgrid(np.arange(w), np.arange(h))
    pix = np.stack([uu.ravel(), vv.ravel()], axis=1).astype(np.float64)
    dirs = pixel_rays(intr, pix) @ pose[:3, :3].T
    org = np.broadcast_to(pose[:3, 3], dirs.shape)
    t, hit = trace(program, org, dirs, max_t)
    xs = org + t[:, None] * dirs
    rgb = np.broadcast_to(np.asarray(scene.background, dtype=np.float64), (h * w, 3)).copy()
    if hit.any():
        rgb[hit] = shade(program, scene, xs[hit])
    z = np.where(hit, t / ray_to_z_scale(intr, pix), 0.0)
    if noise_sigma0 > 0:
        e = rng_noise.normal(0.0, 1.0, size=z.shape)
        z = np.maximum(np.where(hit, z + e * noise_sigma0 * z ** 2, 0.0), 0.0)
    if dropout_world is not None:
        ctr = np.asarray(dropout_world[0], dtype=np.float64)
        z[hit & (np.linalg.norm(xs - ctr, axis=1) < float(dropout_world[1]))] = 0.0
    if dropout_box is not None:
        lo, hi = (np.asarray(b, dtype=np.float64) for b in dropout_box)
        z[hit & np.all((xs >= lo) & (xs <= hi), axis=1)] = 0.0
    dmm = np.round(z * 1000.0).astype(np.uint16).reshape(h, w)
    if dropout_rect is not None:
        x0, y0, x1, y1 = dropout_rect
        dmm[y0:y1, x0:x1] = 0
    return np.round(rgb * 255.0).astype(np.uint8).reshape(h, w, 3), dmm


def render_sequence(scene, trajectory, intr, max_t=8.0, threads=1, seed=0, **kw):
    """(colors u8 (F,H,W,3), depths u16 (F,H,W)) for a trajectory."""
    traj = np.asarray(trajectory, dtype=np.float64)
    program = flatten(scene.root)

    def one(f):
        return render_frame(scene, traj[f], intr, max_t, rng_noise=substream(seed, DEPTH_NOISE, f),
                            program=program, **kw)

    if threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            frames = list(ex.map(one, range(traj.shape[0])))
    else:
        frames = [one(f) for f in range(traj.shape[0])]
    return np.stack([c for c, _ in frames]), np.stack([d for _, d in frames])


# ---------------------------------------------------------------------------
# the bench configurations as oracle datasets (bench.py's port fallback)

CONFIG2_BOUNDS = ((-3.5, -3.5, -0.5), (3.5, 3.5, 2.75))


def config_dataset(config, frames, threads=1):
    """Config 1 (sphere-in-box, 160x120) or 2 (ScanNet-shaped room, 640x480)
    as an oracle dataset (f64 colours/depths).  Scene descriptions come from
    the package's data-only scene module (no device code is loaded)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    from paper_2206_14735_b200 import scenes
    if config == 1:
        w, h = 160, 120
        f = 0.5 * w / np.tan(np.radians(35.0))
        intr = SimpleNamespace(fx=f, fy=f, cx=w / 2.0, cy=h / 2.0, width=w, height=h)
        scene, traj = scenes.sphere_in_box(), scenes.orbit_trajectory(frames)
    else:
        intr = SimpleNamespace(fx=577.87, fy=577.87, cx=319.5, cy=239.5, width=640, height=480)
        scene = scenes.scannet_room()
        traj = scenes.orbit_trajectory(frames, target=(0.0, 0.0, 0.8), radius=1.8, height=1.5,
                                       height_amp=0.3)
    cols, deps = render_sequence(scene, traj, intr, threads=threads)
    sys.path.insert(0, os.path.join(root, "tests"))
    from _golden import OracleDataset
    return OracleDataset(cols, deps, traj, intr)
