"""Ray batches (gs/sampler.py).

On the B200 path a batch is just the drawn flat pixel ids; the per-ray
fields (pixel, colour, along-ray depth, validity, camera direction) are
computed on the device by the step kernel.  The reference RayBatch fields
remain available on the host, computed with the reference's formulas
(gs/sampler.py:70-88), for API compatibility and tests.
"""

from __future__ import annotations

import numpy as np

from .camera import pixel_rays, ray_to_z_scale

N_COARSE = 96  # gs/sampler.py:29-32
N_IMPORTANCE_ROUNDS = 3
N_IMPORTANCE_ADD = 12
MIN_SEPARATION = 1e-9


class RayBatch:
    """One optimisation batch of rays (gs/sampler.py:35-55)."""

    def __init__(self, dataset, ray_ids, near=0.01, far=8.0):
        self.dataset = dataset
        self.ray_ids = np.asarray(ray_ids, dtype=np.int64)
        self.near_value = float(near)
        self.far_value = float(far)
        self._f = None

    def __len__(self):
        return self.ray_ids.shape[0]

    def _fields(self):
        if self._f is None:
            ds = self.dataset
            intr = ds.intrinsics
            h, w = intr.height, intr.width
            flat = self.ray_ids
            frame = flat // (h * w)
            rem = flat % (h * w)
            v, u = rem // w, rem % w
            pixels = np.stack([u, v], axis=1).astype(np.float64)
            color = ds.colors_u8[frame, v, u].astype(np.float64) / 255.0
            depth_z = ds.depths_mm[frame, v, u].astype(np.float64) / 1000.0
            scale = ray_to_z_scale(intr, pixels)
            self._f = dict(frame_ids=frame.astype(np.int64), pixels=pixels, color=color,
                           depth_ray=depth_z * scale, valid=depth_z > 0,
                           dir_cam=pixel_rays(intr, pixels))
        return self._f

    frame_ids = property(lambda self: self._fields()["frame_ids"])
    pixels = property(lambda self: self._fields()["pixels"])
    color = property(lambda self: self._fields()["color"])
    depth_ray = property(lambda self: self._fields()["depth_ray"])
    valid = property(lambda self: self._fields()["valid"])
    dir_cam = property(lambda self: self._fields()["dir_cam"])
    near = property(lambda self: np.full(len(self), self.near_value))
    far = property(lambda self: np.full(len(self), self.far_value))


def draw_ray_batch(dataset, rng, m, near=0.01, far=8.0):
    """Sample M rays uniformly over every (frame, pixel) pair (gs/sampler.py:58-88)."""
    intr = dataset.intrinsics
    f = len(dataset)
    flat = rng.integers(0, f * intr.height * intr.width, size=m)
    return RayBatch(dataset, flat, near, far)


def batch_ray_ids(batch, dataset):
    """Flat ids of a RayBatch-like object (ours or the reference's)."""
    if isinstance(batch, RayBatch):
        return batch.ray_ids
    intr = dataset.intrinsics
    px = np.asarray(batch.pixels)
    u = px[:, 0].astype(np.int64)
    v = px[:, 1].astype(np.int64)
    return (np.asarray(batch.frame_ids, dtype=np.int64) * intr.height + v) * intr.width + u


def stratified_coarse(near, far, n, uniforms):
    """gs/sampler.py:91-107 (host form, used by tests and tools)."""
    near = np.asarray(near)
    far = np.asarray(far)
    if np.any(far <= near):
        raise ValueError("degenerate ray bounds")
    steps = (np.arange(n) + uniforms) / n
    return near[:, None] + (far - near)[:, None] * steps


def importance_refine_with_sources(depths, weights, near, far, uniforms):
    """gs/sampler.py:128-169 on the device (gsb_importance_refine): invert the
    piecewise-constant weight CDF, merge stably, enforce the 1e-9 separation.
    Returns ((M, K + A) depths, (M, K + A) int64 provenance, -1 = new/moved)."""
    import torch

    from . import _lib
    d = np.ascontiguousarray(depths, dtype=np.float64)
    M, K = d.shape
    A = np.asarray(uniforms).shape[1]
    if K + A > _lib.KMAX or A > _lib.AMAX:
        raise ValueError("too many samples per ray for the device kernel")
    dev = torch.device("cuda", torch.cuda.current_device())
    ld = K + A
    T = lambda a: torch.from_numpy(np.array(a, dtype=np.float64)).to(dev)  # a writable copy
    dd = torch.zeros((M, ld), dtype=torch.float64, device=dev)
    dd[:, :K] = T(d)
    ww = torch.zeros((M, ld), dtype=torch.float64, device=dev)
    ww[:, :K] = T(weights)
    nt, ft, ut = T(np.broadcast_to(near, (M,))), T(np.broadcast_to(far, (M,))), T(uniforms)
    out = torch.zeros((M, ld), dtype=torch.float64, device=dev)
    src = torch.zeros((M, ld), dtype=torch.int32, device=dev)
    if M:
        _lib.check(_lib.lib().gsb_importance_refine(M, K, A, ld, dd.data_ptr(), ww.data_ptr(), nt.data_ptr(),
                                                    ft.data_ptr(), ut.data_ptr(), out.data_ptr(),
                                                    src.data_ptr(), _lib.stream_handle()),
                   "gsb_importance_refine")
    return out.cpu().numpy(), src.cpu().numpy().astype(np.int64)


def importance_refine(depths, weights, near, far, uniforms):
    """gs/sampler.py:110-125."""
    return importance_refine_with_sources(depths, weights, near, far, uniforms)[0]
