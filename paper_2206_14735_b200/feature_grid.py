"""Feature-grid API mirror (gs/feature_grid.py): the grid containers live in
model.py (one parameter arena); trilinear lookups run on the device through
gsb_grid_sample (the exact twin of diffcore.grid_sample's forward:
fp64 locate, numba's per-corner rounding)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .model import GridLevel, MultiGrid, world_box_from_frusta  # noqa: F401

__all__ = ["GridLevel", "MultiGrid", "sample", "sample_multi", "world_box_from_frusta"]


def _level_struct(level):
    g = level.geom
    nx, ny, nz = g.dims
    return _lib.Level(nx, ny, nz, int(level.width), float(g.origin[0]), float(g.origin[1]), float(g.origin[2]),
                      float(g.voxel_size), 0)


def sample(level, x):
    """Interpolate one level's features at world points (gs/feature_grid.py:120-132):
    (N, 3) points inside the level's box -> (N, width) array in the model dtype.
    Raises GridBoundsError for points outside the lattice."""
    import torch

    from .renderer import GridBoundsError
    feat = level.features.data
    dt = np.float32 if feat.dtype == torch.float32 else np.float64
    pts = torch.from_numpy(np.array(np.atleast_2d(x), dtype=dt)).to(feat.device)
    n = pts.shape[0]
    out = torch.empty((n, level.width), dtype=feat.dtype, device=feat.device)
    status = torch.zeros(_lib.N_STATUS, dtype=torch.int32, device=feat.device)
    L = _level_struct(level)
    if n:
        _lib.check(_lib.lib().gsb_grid_sample(0 if dt == np.float32 else 1, C.byref(L), feat.data_ptr(),
                                              pts.data_ptr(), n, out.data_ptr(), status.data_ptr(),
                                              _lib.stream_handle()), "gsb_grid_sample")
    if int(status[_lib.ST_BOUNDS].item()):
        raise GridBoundsError("points outside the grid box")
    return out.cpu().numpy()


def sample_multi(grid, x):
    """Per-level geometry features concatenated coarse to fine (gs/feature_grid.py:135-139)."""
    return np.concatenate([sample(lev, x) for lev in grid.levels], axis=1)
