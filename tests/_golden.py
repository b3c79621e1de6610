"""Load the committed golden fixtures (tests/golden/*.npz, produced by
tests/golden/make_golden.py from the reference package itself)."""

from __future__ import annotations

import json
import os
import sys
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


class OracleDataset:
    """Dataset restated (gs/scenegen.py:267-287): f64 colours/depths."""

    def __init__(self, colors_u8, depths_u16, poses, intr):
        self.colors_u8, self.depths_u16 = colors_u8, depths_u16
        self.colors = colors_u8.astype(np.float64) / 255.0
        self.depths = depths_u16.astype(np.float64) / 1000.0
        self.poses = poses
        self.intrinsics = intr
        self._vp = None

    def __len__(self):
        return self.colors.shape[0]

    @property
    def valid_pixels(self):
        if self._vp is None:
            f, v, u = np.nonzero(self.depths > 0)
            self._vp = (f.astype(np.int64), v.astype(np.int64), u.astype(np.int64))
        return self._vp


def weights_ns(**kw):
    d = dict(rgb=10.0, depth=1.0, sdf=10.0, fs=1.0, eik=1.0, smooth=1.0, truncation=0.16,
             freespace_alpha=5.0, smooth_delta=0.004, smooth_count=1024)
    d.update(kw)
    return SimpleNamespace(**d)


def cfg_ns(**kw):
    """TrainConfig defaults, gs/optimizer.py:94-125."""
    d = dict(iterations=10000, batch_rays=6144, coarse_samples=96, importance_rounds=3,
             importance_add=12, seed=0, precision="double", near=0.01, max_depth=8.0,
             bounds=None, bounds_padding=0.5, voxel_sizes=(0.96, 0.24, 0.06, 0.03),
             color_voxel=None, geom_feat_dim=4, color_feat_dim=6, fixed_far=None,
             lr_grids=1e-2, lr_decoders=1e-3, lr_poses=5e-4, refine_poses=False,
             freeze_first_pose=True, pose_refresh_every=100)
    d.update(kw)
    d.setdefault("weights", weights_ns())
    return SimpleNamespace(**d)


def load(name, precision):
    z = np.load(os.path.join(GOLDEN, f"{name}_{precision}.npz"))
    arrays = {k: z[k] for k in z.files}
    meta = json.loads(arrays.pop("meta_json").tobytes().decode())
    fx, fy, cx, cy, w, h = meta["intr"]
    intr = SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))
    ds = OracleDataset(arrays["colors_u8"], arrays["depths_u16"], arrays["poses"], intr)
    c = dict(meta["cfg"])
    if "voxel_sizes" in c:
        c["voxel_sizes"] = tuple(c["voxel_sizes"])
    if "bounds" in c:
        c["bounds"] = tuple(map(tuple, c["bounds"]))
    cfg = cfg_ns(precision=precision, **c)
    cfg.weights.smooth_count = meta["smooth_count"]
    return SimpleNamespace(ds=ds, cfg=cfg, meta=meta, a=arrays,
                           dtype=np.float64 if precision == "double" else np.float32)


def oracle_params(G):
    """Oracle parameters built the way gs/optimizer.py:181-205 builds them."""
    from oracle import gridsurf_oracle as O
    cfg = G.cfg
    return O.create_params(G.meta["lo"], G.meta["hi"], G.ds.poses, seed=cfg.seed,
                           voxel_sizes=cfg.voxel_sizes, geom_width=cfg.geom_feat_dim,
                           color_voxel=cfg.color_voxel, color_width=cfg.color_feat_dim,
                           dtype=G.dtype, truncation=cfg.weights.truncation)


def rel_maxnorm(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = max(np.abs(b).max(), 1e-300)
    return float(np.abs(a - b).max() / den)
