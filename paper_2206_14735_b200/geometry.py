"""Geometry on point lists: dense SDF queries and the sphere pre-fit
(decoders.geometric_init, gs/decoders.py:102-177), on the device.

The pre-fit keeps the reference's loop on the host: uniform batch draws from
substream(seed, SPHERE_INIT, step), the 13 anchors, the held-out RMSE checks
every 50 steps from step 100, and the final 10k-point check that raises
InitError.  Each step is one `gsb_sdf_fit_step` (phi at batch + anchors, the
MSE seeds, phi-only backward into the geometry levels and geometry decoder)
plus Adam over those tensors only (their own moments, per-tensor step counts
as in gs/optimizer.py:58-91)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, seeds


from .model import HIDDEN_WIDTH, DecoderNet  # noqa: E402,F401  (gs/decoders.py:22-76)

N_HIDDEN = 2  # hidden ReLU layers of each decoder (gs/decoders.py:23)


class InitError(RuntimeError):
    """Geometric initialization failed to reach tolerance in budget."""


class SdfQuery:
    """phi at arbitrary points (model dtype) through gsb_sdf_points."""

    def __init__(self, model, capacity=1 << 16):
        import torch
        from .engine import model_struct
        self.torch = torch
        self.model = model
        self.ms = model_struct(model)
        self.lib = _lib.lib()
        self.capacity = 0
        self.ws = None
        self._reserve(capacity)

    def _reserve(self, n):
        if n <= self.capacity:
            return
        nb = C.c_size_t(0)
        _lib.check(self.lib.gsb_sdf_workspace_size(C.byref(self.ms), int(n), C.byref(nb)),
                   "gsb_sdf_workspace_size")
        self.ws = self.torch.empty(nb.value, dtype=self.torch.uint8, device=self.model.arena.device)
        self.capacity = int(n)

    def device(self, pts):
        """(n, 3) host points -> (n,) device phi (model dtype)."""
        torch = self.torch
        a = self.model.arena
        p = torch.from_numpy(np.ascontiguousarray(pts, dtype=a.dtype)).to(a.device)
        n = p.shape[0]
        self._reserve(n)
        phi = torch.empty(n, dtype=p.dtype, device=a.device)
        _lib.check(self.lib.gsb_sdf_points(C.byref(self.ms), p.data_ptr(), n, phi.data_ptr(),
                                           self.ws.data_ptr(), self.ws.numel(),
                                           _lib.stream_handle()), "gsb_sdf_points")
        return phi

    def __call__(self, pts, chunk=1 << 22):
        out = []
        for i in range(0, len(pts), chunk):
            out.append(self.device(pts[i:i + chunk]).cpu().numpy())
        return np.concatenate(out) if out else np.zeros(0, dtype=self.model.arena.dtype)


class _RangeAdam:
    """Adam (gs/optimizer.py:38-91) over contiguous arena ranges, each with its
    own learning rate and zero-initialised moments; one shared step count
    (all tensors step together, as in geometric_init)."""

    def __init__(self, arena, ranges, beta1=0.9, beta2=0.999, eps=1e-8):
        import torch
        self.arena, self.ranges = arena, ranges
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        dev, tdt = arena.device, arena.params.dtype
        self.m = [torch.zeros(e - b, dtype=tdt, device=dev) for b, e, _ in ranges]
        self.v = [torch.zeros(e - b, dtype=tdt, device=dev) for b, e, _ in ranges]
        self.status = torch.zeros(_lib.N_STATUS, dtype=torch.int32, device=dev)
        self.t = 0

    def step(self):
        self.t += 1
        t = float(self.t)
        c1 = 1.0 - self.beta1 ** t  # host pow == numba's libm pow
        c2 = 1.0 - self.beta2 ** t
        a = self.arena
        esz = a.params.element_size()
        L = _lib.lib()
        for (b, e, lr), m, v in zip(self.ranges, self.m, self.v):
            B = (C.c_int64 * 1)(0)
            Lr = (C.c_double * 1)(lr)
            _lib.check(L.gsb_adam_step(
                0 if a.dtype == np.float32 else 1, a.params.data_ptr() + b * esz,
                a.grads.data_ptr() + b * esz, m.data_ptr(), v.data_ptr(), e - b, B, Lr, 1,
                self.beta1, self.beta2, self.eps, c1, c2, None, 0.0, None, self.status.data_ptr(),
                _lib.stream_handle()), "gsb_adam_step")
        a.grads_clean = True  # the kernel zeroes the gradients it consumed


def _ranges(model, lr_grid, lr_net):
    levels = [l.features for l in model.grid.levels]
    net = model.geom_net.parameters()
    # levels are adjacent in the arena (grid group, in order); so is the net
    lv = (levels[0].offset, levels[-1].offset + levels[-1].size, lr_grid)
    nt = (net[0].offset, net[-1].offset + net[-1].size, lr_net)
    return [lv, nt]


def geometric_init(model, center, radius, seed=0, max_steps=2000, tol=0.01, batch=4096,
                   lr_grid=1e-2, lr_net=1e-3, info=None):
    """Fit grid + geometry decoder to the SDF of a sphere (gs/decoders.py:102-177).

    Runs Adam on batches of uniform in-box points against ||x - c|| - r until
    the RMSE on a held-out probe set drops below ``tol`` (with the anchors also
    below it), then verifies on 10k fresh points.  Returns that RMSE.

    ``info`` (optional dict) receives the number of Adam steps taken.

    Raises:
        InitError: tolerance not reached within ``max_steps``.
    """
    import torch
    from .engine import model_struct
    a = model.arena
    dt = a.dtype
    grid = model.grid
    center = np.asarray(center, dtype=np.float64)
    lo = grid.lo + 0.5 * grid.finest_voxel
    hi = grid.hi - 0.5 * grid.finest_voxel
    if np.any(center - radius < grid.lo) or np.any(center + radius > grid.hi):
        raise ValueError("sphere must fit inside the grid box")

    def sphere_sdf(x):
        return np.linalg.norm(x - center, axis=1, keepdims=True) - radius

    axes = np.concatenate([np.eye(3), -np.eye(3)], axis=0)
    anchors = np.clip(np.concatenate([center[None, :], center + radius * axes,
                                      center + 2.0 * radius * axes]), lo, hi)
    anchor_target = sphere_sdf(anchors).astype(dt)
    n_anchor = anchors.shape[0]

    lib = _lib.lib()
    ms = model_struct(model)
    nbytes = C.c_size_t(0)
    _lib.check(lib.gsb_sdf_workspace_size(C.byref(ms), batch + n_anchor, C.byref(nbytes)),
               "gsb_sdf_workspace_size")
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=a.device)
    query = SdfQuery(model, capacity=10_000)
    opt = _RangeAdam(a, _ranges(model, lr_grid, lr_net))
    pts_h = torch.empty((batch + n_anchor, 3), dtype=a.params.dtype).pin_memory()
    tgt_h = torch.empty(batch + n_anchor, dtype=a.params.dtype).pin_memory()
    pts_h.numpy()[batch:] = anchors.astype(dt)
    tgt_h.numpy()[batch:] = anchor_target[:, 0]
    pts_d = torch.empty_like(pts_h, device=a.device)
    tgt_d = torch.empty_like(tgt_h, device=a.device)

    def rmse(n_pts, stream_idx):
        r = seeds.substream(seed, seeds.SPHERE_INIT, 10_000 + stream_idx)
        pts = r.uniform(lo, hi, size=(n_pts, 3))
        phi = query(pts.astype(dt)).reshape(-1, 1)
        return float(np.sqrt(np.mean((phi - sphere_sdf(pts)) ** 2)))

    def anchor_err():
        phi = query(anchors.astype(dt)).reshape(-1, 1)
        return float(np.max(np.abs(phi - sphere_sdf(anchors))))

    steps = 0
    for step in range(max_steps):
        rng = seeds.substream(seed, seeds.SPHERE_INIT, step)
        pts = rng.uniform(lo, hi, size=(batch, 3))
        torch.cuda.current_stream().synchronize()  # pinned staging buffers are reused
        pts_h.numpy()[:batch] = pts.astype(dt)
        tgt_h.numpy()[:batch] = sphere_sdf(pts).astype(dt)[:, 0]
        pts_d.copy_(pts_h, non_blocking=True)
        tgt_d.copy_(tgt_h, non_blocking=True)
        a.zero_grads()
        _lib.check(lib.gsb_sdf_fit_step(C.byref(ms), pts_d.data_ptr(), tgt_d.data_ptr(), batch,
                                        n_anchor, ws.data_ptr(), ws.numel(), None,
                                        _lib.stream_handle()), "gsb_sdf_fit_step")
        a.grads_clean = False
        opt.step()
        steps += 1
        if (step >= 100 and step % 50 == 0
                and rmse(2048, step) < 0.8 * tol and anchor_err() < 0.8 * tol):
            break

    final = rmse(10_000, -1)
    if info is not None:
        info["steps"] = steps
    if final >= tol:
        raise InitError(f"sphere pre-fit RMSE {final:.4f} m did not reach {tol} m "
                        f"within {max_steps} steps")
    return final
