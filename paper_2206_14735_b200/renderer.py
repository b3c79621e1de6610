"""Training objective on the device (gs/renderer.py).

``train_objective`` keeps the reference signature and return values but
runs the whole forward AND backward as one device step: the returned
``total`` is an :class:`Objective` whose gradients already sit in the
parameter arena, and :func:`grad` hands out views of them.  Host
synchronisation happens once, to read the loss parts and status words.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import StepEngine, draw_smooth_points, host_draws
from .model import ModelState  # noqa: F401  (gs/renderer.py:69-105)
from .sampler import batch_ray_ids

__all__ = ["LossWeights", "train_objective", "grad", "Objective", "draw_smooth_points",
           "GridBoundsError", "SIGMA_FLOOR", "TRANS_FLOOR"]

SIGMA_FLOOR = 1e-12  # gs/renderer.py:42-43
TRANS_FLOOR = 1e-15


class GridBoundsError(ValueError):
    """A sample position fell outside the grid's world box (gs/diffcore.py:46)."""


@dataclass
class LossWeights:
    """Objective term weights and constants (gs/renderer.py:46-66)."""

    rgb: float = 10.0
    depth: float = 1.0
    sdf: float = 10.0
    fs: float = 1.0
    eik: float = 1.0
    smooth: float = 1.0
    truncation: float = 0.16
    freespace_alpha: float = 5.0
    smooth_delta: float = 0.004
    smooth_count: int = 1024

    def __post_init__(self):
        if self.truncation <= 0:
            raise ValueError("truncation must be positive")
        for name in ("rgb", "depth", "sdf", "fs", "eik", "smooth"):
            if getattr(self, name) < 0:
                raise ValueError(f"loss weight {name} must be non-negative")


class Objective:
    """The scalar objective of one step; its gradients live in the arena."""

    def __init__(self, value, model, generation):
        self.data = np.asarray(value)
        self.model = model
        self.generation = generation
        self.requires_grad = True

    @property
    def shape(self):
        return ()

    def item(self):
        return float(self.data)

    def __float__(self):
        return float(self.data)


def grad(output, wrt, grad_output=None, create_graph=False):
    """Gradients of an Objective w.r.t. model parameters (gs/diffcore.py:1035).

    Returns device tensors (views of the gradient arena).  Higher-order
    graphs are not materialised on this path (create_graph is refused)."""
    if create_graph:
        raise NotImplementedError("create_graph is not supported on the fused device step")
    if not isinstance(output, Objective):
        raise TypeError("grad() expects the Objective returned by train_objective")
    arena = output.model.arena
    if arena.generation != output.generation:
        raise RuntimeError("gradients of this objective were already consumed or overwritten")
    if grad_output is not None and float(np.asarray(grad_output)) != 1.0:
        scale = float(np.asarray(grad_output))
        arena.grads.mul_(scale)
    single = not isinstance(wrt, (list, tuple))
    lst = [wrt] if single else list(wrt)
    out = []
    for p in lst:
        if getattr(p, "arena", None) is not arena:
            raise ValueError("parameter does not belong to this model")
        out.append(p.grad)
    return out[0] if single else out


class _Extras(dict):
    """extras dict with lazily fetched depths / weights (device -> host)."""

    def __init__(self, base, fetch):
        super().__init__(base)
        self._fetch = fetch

    def __missing__(self, key):
        if key in ("depths", "weights"):
            v = self._fetch(key)
            self[key] = v
            return v
        raise KeyError(key)

    def __contains__(self, key):
        return key in ("depths", "weights") or dict.__contains__(self, key)


def engine_for(model, dataset):
    cache = model.__dict__.setdefault("_engines", {})
    key = id(dataset)
    if key not in cache:
        cache[key] = StepEngine(model, dataset)
    return cache[key]


def check_status(status, precision="single"):
    """Raise the reference's exception for a step's device status words
    (a device tensor or the host copy of one)."""
    st = status.cpu().numpy() if hasattr(status, "cpu") else np.asarray(status)
    if st[_lib.ST_BOUNDS]:
        raise GridBoundsError("sample point(s) outside grid box")
    if st[_lib.ST_VIEWDIR]:
        raise ValueError("view directions must be unit length")
    if st[_lib.ST_OVERFLOW]:
        raise RuntimeError("importance evaluation list overflow")


def parts_from(ws):
    p = ws["parts"].cpu().numpy()
    return {k: float(p[i]) for i, k in enumerate(_lib.PART_NAMES)}


def train_objective(model, dataset, batch, iteration, cfg, smooth_override=None, deterministic=None):
    """Evaluate the objective for one ray batch and its full gradient
    (gs/renderer.py:279-468 + gs/diffcore.py:1035).

    ``deterministic`` (not in the reference): True switches the grid-gradient
    scatters to the sorted, sample-ordered reduction (bit-reproducible run to
    run, for validation); None keeps the engine's current mode.

    Returns (total Objective, parts dict of floats, extras dict)."""
    from .data import Dataset
    dataset = dataset if isinstance(dataset, Dataset) else Dataset.wrap(dataset)
    if hasattr(batch, "near_value"):
        near, far = batch.near_value, batch.far_value
    else:
        near, far = _check_foreign_batch(batch, dataset)
    if near != cfg.near or far != cfg.max_depth:
        cfg = _with(cfg, near=near, max_depth=far)
    eng = engine_for(model, dataset)
    if deterministic is not None:
        eng.deterministic = bool(deterministic)
    draws = host_draws(model, dataset, cfg, iteration, ray_ids=batch_ray_ids(batch, dataset),
                       smooth_override=smooth_override)
    ids, sm = eng.upload(draws)
    ws = eng.launch(cfg, draws, ids, sm)
    arena = model.arena
    arena.generation = getattr(arena, "generation", 0) + 1
    parts = parts_from(ws)
    check_status(ws["status"])
    if cfg.precision == "double" and not np.isfinite(parts["total"]):
        raise FloatingPointError("non-finite values in total loss")
    counts = ws["counts"].cpu().numpy()
    n = cfg.coarse_samples + cfg.importance_rounds * cfg.importance_add
    extras = {
        "samples_per_ray": n,
        "n_valid_rays": int(counts[_lib.C_VALID]),
        "n_tr": int(counts[_lib.C_TR]),
        "n_fs": int(counts[_lib.C_FS]),
        "n_eik": int(counts[_lib.C_EIK]),
        "n_smooth": draws.n_smooth,
        "empty_tr": bool(counts[_lib.C_TR] == 0),
        "empty_fs": bool(counts[_lib.C_FS] == 0),
    }

    def fetch(key):
        if key == "depths":
            return ws["depths"][:, :n].cpu().numpy().copy()
        return ws["weights"].cpu().numpy().copy()

    total = Objective(parts["total"], model, arena.generation)
    return total, parts, _Extras(extras, fetch)


def _check_foreign_batch(batch, dataset):
    """A reference-shaped RayBatch (gs/sampler.py:35-55) carries per-ray
    bounds and targets; the device step derives the targets from the ray ids
    and takes one near / far for the batch (what draw_ray_batch produces).
    Anything else would be trained on different inputs: refuse it."""
    from .sampler import RayBatch
    nr, fr = np.asarray(batch.near, dtype=np.float64), np.asarray(batch.far, dtype=np.float64)
    if nr.size == 0:
        raise ValueError("empty ray batch")
    if np.any(nr != nr[0]) or np.any(fr != fr[0]):
        raise ValueError("per-ray near/far bounds are not supported: the batch must share one near and far")
    mine = RayBatch(dataset, batch_ray_ids(batch, dataset), nr[0], fr[0])
    for k in ("color", "depth_ray", "valid", "dir_cam"):
        if hasattr(batch, k) and not np.array_equal(np.asarray(getattr(batch, k)), getattr(mine, k)):
            raise ValueError(f"batch.{k} differs from the dataset's values at the batch's pixels")
    return float(nr[0]), float(fr[0])


def _with(cfg, **kw):
    import copy
    c = copy.copy(cfg)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def realized_pose_arrays(model, frames):
    """gs/renderer.py:218-225: rows R (U, 9) and t (U, 3) of the given frames,
    in the model dtype, as the step realises them (R0 exp_so3(nu), t)."""
    frames = np.asarray(frames, dtype=np.int64).reshape(-1)
    dt = model.dtype
    R = np.stack([(model.poses[f].R0.astype(dt) @ _exp_dt(model.poses[f].nu_data(), dt)).reshape(9)
                  for f in frames]) if len(frames) else np.zeros((0, 9), dt)
    T = np.stack([np.asarray(model.poses[f].t_data(), dtype=dt) for f in frames]) if len(frames) \
        else np.zeros((0, 3), dt)
    return R.astype(dt), T.astype(dt)


def _exp_dt(nu, dt):
    from .camera import exp_so3_data
    return exp_so3_data(np.asarray(nu, dtype=np.float64)).astype(dt)
