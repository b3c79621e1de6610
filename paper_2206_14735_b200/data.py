"""RGB-D datasets: host handle (reference-compatible) and device residency.

The reference keeps colours/depths as float64 arrays (gs/scenegen.py:267-287)
that are exactly u8/255 and u16/1000 (every reference dataset comes from
8-bit PNGs and millimetre depth, gs/scenegen.py:319-392).  Here the
quantised arrays are the storage: 5 bytes per pixel on the host and in HBM
instead of 32, and the float64 views are produced on demand with the same
arithmetic.  The valid-pixel list (gs/scenegen.py:281-287, 24 B per pixel)
is replaced by a per-row prefix count that yields the same k-th valid pixel.
"""

from __future__ import annotations

import os

import numpy as np

from . import camera


class Dataset:
    """Posed RGB-D sequence (gs/scenegen.py:267-287)."""

    def __init__(self, colors_u8, depths_mm, poses, intrinsics, root=None):
        colors_u8 = np.ascontiguousarray(colors_u8, dtype=np.uint8)
        depths_mm = np.ascontiguousarray(depths_mm, dtype=np.uint16)
        if colors_u8.ndim != 4 or colors_u8.shape[3] != 3:
            raise ValueError("colors must be (F, H, W, 3)")
        if depths_mm.shape != colors_u8.shape[:3]:
            raise ValueError("depths must be (F, H, W)")
        if (colors_u8.shape[1], colors_u8.shape[2]) != (intrinsics.height, intrinsics.width):
            raise ValueError("frame dimensions do not match intrinsics")
        self.colors_u8 = colors_u8
        self.depths_mm = depths_mm
        self.poses = np.asarray(poses, dtype=np.float64)
        if self.poses.shape != (colors_u8.shape[0], 4, 4):
            raise ValueError("poses must be (F, 4, 4)")
        self.intrinsics = intrinsics
        self.root = root
        self._row_cum = None
        self._device = {}

    @classmethod
    def from_float(cls, colors, depths, poses, intrinsics, root=None):
        """Accept reference-style float64 arrays; they must be exactly u8/255
        and u16/1000 (as every reference dataset is)."""
        c8 = np.round(np.asarray(colors) * 255.0).astype(np.uint8)
        d16 = np.round(np.asarray(depths) * 1000.0).astype(np.uint16)
        if not np.array_equal(c8.astype(np.float64) / 255.0, colors):
            raise ValueError("colours are not 8-bit quantised (u8/255)")
        if not np.array_equal(d16.astype(np.float64) / 1000.0, depths):
            raise ValueError("depths are not millimetre quantised (u16/1000)")
        return cls(c8, d16, poses, intrinsics, root=root)

    @classmethod
    def wrap(cls, ds):
        """Convert any reference-like dataset handle."""
        if isinstance(ds, Dataset):
            return ds
        if hasattr(ds, "colors_u8") and hasattr(ds, "depths_u16"):
            return cls(ds.colors_u8, ds.depths_u16, ds.poses, ds.intrinsics)
        return cls.from_float(ds.colors, ds.depths, ds.poses, ds.intrinsics,
                              root=getattr(ds, "root", None))

    def __len__(self):
        return self.colors_u8.shape[0]

    @property
    def colors(self):
        """(F, H, W, 3) float64 in [0, 1] (materialised on demand)."""
        return self.colors_u8.astype(np.float64) / 255.0

    @property
    def depths(self):
        """(F, H, W) float64 z-metres, 0 = missing (materialised on demand)."""
        return self.depths_mm.astype(np.float64) / 1000.0

    def depth_at(self, f, v, u):
        return self.depths_mm[f, v, u].astype(np.float64) / 1000.0

    # ---- valid pixels (gs/scenegen.py:281-287) without the 24 B/pixel list
    def _rows(self):
        if self._row_cum is None:
            cnt = (self.depths_mm > 0).sum(axis=2).reshape(-1).astype(np.int64)
            self._row_cum = np.cumsum(cnt)
        return self._row_cum

    @property
    def n_valid(self):
        cum = self._rows()
        return int(cum[-1]) if cum.size else 0

    def valid_pixel(self, k):
        """(frames, vs, us) of the k-th valid pixels in np.nonzero order."""
        k = np.asarray(k, dtype=np.int64)
        cum = self._rows()
        row = np.searchsorted(cum, k, side="right")
        before = np.where(row > 0, cum[np.maximum(row - 1, 0)], 0)
        r = k - before
        h, wd = self.intrinsics.height, self.intrinsics.width
        f, v = row // h, row % h
        # rows without missing depth: the r-th valid pixel is u = r; only
        # partial rows need the in-row prefix scan
        cnt = cum[row] - before
        u = r.copy()
        part = np.flatnonzero(cnt < wd)
        if part.size:
            mask = self.depths_mm[f[part], v[part]] > 0  # (n_part, W)
            csum = np.cumsum(mask, axis=1, dtype=np.int32)
            u[part] = np.argmax(csum > r[part, None], axis=1)
        return f.astype(np.int64), v.astype(np.int64), u.astype(np.int64)

    @property
    def valid_pixels(self):
        """Reference API (full index arrays; prefer n_valid/valid_pixel)."""
        f, v, u = np.nonzero(self.depths_mm > 0)
        return f.astype(np.int64), v.astype(np.int64), u.astype(np.int64)

    # ---- device residency
    def device_tensors(self, device, dtype):
        """u8 colours, u16 depths and (F, 12) dtype-rounded poses in HBM."""
        import torch
        key = (str(device), np.dtype(dtype).str)
        if key not in self._device:
            col = torch.from_numpy(self.colors_u8).to(device)
            dep = torch.from_numpy(self.depths_mm.view(np.int16)).to(device)
            P = np.zeros((len(self), 12), dtype=np.float64)
            # PoseParam stores R0 (f64) and t in the model dtype; the realised
            # rotation is R0.astype(dtype) @ exp(0) = R0.astype(dtype)
            # (gs/camera.py:68-70, gs/renderer.py:218-225)
            P[:, :9] = self.poses[:, :3, :3].reshape(-1, 9).astype(dtype).astype(np.float64)
            P[:, 9:] = self.poses[:, :3, 3].astype(dtype).astype(np.float64)
            self._device[key] = (col, dep, torch.from_numpy(P).to(device))
        return self._device[key]


def load_dataset(root):
    """gs/scenegen.py:371-392: color/%06d.png, depth/%06d.png, poses.txt, intrinsics.txt."""
    from PIL import Image
    intr = camera.load_intrinsics(os.path.join(root, "intrinsics.txt"))
    poses = camera.load_poses(os.path.join(root, "poses.txt"))
    cdir, ddir = os.path.join(root, "color"), os.path.join(root, "depth")
    if not os.path.isdir(cdir) or not os.path.isdir(ddir):
        raise FileNotFoundError(f"{root}: expected color/ and depth/ subdirectories")
    cfiles = sorted(f for f in os.listdir(cdir) if f.endswith(".png"))
    dfiles = sorted(f for f in os.listdir(ddir) if f.endswith(".png"))
    if len(cfiles) != len(dfiles):
        raise ValueError(f"{root}: {len(cfiles)} color frames but {len(dfiles)} depth frames")
    if len(cfiles) != poses.shape[0]:
        raise ValueError(f"{root}: {len(cfiles)} frames but {poses.shape[0]} poses")
    cols, deps = [], []
    for cf, df in zip(cfiles, dfiles):
        img = np.asarray(Image.open(os.path.join(cdir, cf)))
        dep = np.asarray(Image.open(os.path.join(ddir, df)))
        if img.shape[:2] != (intr.height, intr.width) or dep.shape != (intr.height, intr.width):
            raise ValueError(f"{root}: frame {cf} dimensions do not match intrinsics")
        cols.append(img.astype(np.uint8))
        deps.append(dep.astype(np.uint16))
    return Dataset(np.stack(cols), np.stack(deps), poses, intr, root=root)
