"""Model state over one parameter arena in HBM.

Mirrors the reference containers (gs/feature_grid.py GridLevel/MultiGrid,
gs/decoders.py DecoderNet, gs/renderer.py ModelState) but every parameter is
a view into ONE contiguous device buffer (the "arena"), with gradient, Adam
m and v arenas of identical layout, so the dense Adam update and a
data-parallel gradient all-reduce are each a single call.

Arena layout (elements of the model dtype):
    level0 (V0, C) | level1 | ... | colour grid (Vc, Cc)      each 16-byte aligned
    MLP block: geom W0 b0 W1 b1 W2 b2 | pad to 4 | colour W0 b0 W1 b1 W2 b2
               (this exact layout is copied into __constant__ memory per step)
    log_s | pose nu0 t0 nu1 t1 ... (trainable frames only)
"""

from __future__ import annotations

import numpy as np

from . import seeds
from .camera import PoseParam

DEFAULT_GEOM_VOXELS = (0.96, 0.24, 0.06, 0.03)  # gs/feature_grid.py:33
GEOM_FEATURE_WIDTH = 4
COLOR_FEATURE_WIDTH = 6
FEATURE_INIT_SCALE = 1e-4
HIDDEN_WIDTH = 32  # gs/decoders.py:22


def _torch_dtype(dtype):
    import torch
    return torch.float32 if np.dtype(dtype) == np.float32 else torch.float64


class GridGeom:
    """World geometry of a dense vertex lattice (gs/diffcore.py:704-728)."""

    __slots__ = ("origin", "voxel_size", "dims")

    def __init__(self, origin, voxel_size, dims):
        self.origin = np.asarray(origin, dtype=np.float64)
        self.voxel_size = float(voxel_size)
        self.dims = tuple(int(d) for d in dims)
        if any(d < 2 for d in self.dims):
            raise ValueError("grid needs at least 2 vertices per axis")

    @property
    def n_vertices(self):
        nx, ny, nz = self.dims
        return nx * ny * nz

    def world_max(self):
        return self.origin + self.voxel_size * (np.array(self.dims) - 1)


class Param:
    """One parameter tensor: a view of the arena (the reference's dc.leaf)."""

    def __init__(self, arena, name, offset, shape):
        self.arena, self.name, self.offset = arena, name, int(offset)
        self.shape = tuple(int(s) for s in shape)
        self.size = int(np.prod(self.shape)) if self.shape else 1
        self.requires_grad = True

    @property
    def dtype(self):
        return self.arena.dtype

    @property
    def data(self):
        """Device view (torch) of the parameter values."""
        return self.arena.params[self.offset:self.offset + self.size].view(self.shape)

    @property
    def grad(self):
        return self.arena.grads[self.offset:self.offset + self.size].view(self.shape)

    def numpy(self):
        d = self.data
        if d.is_cuda:  # every stream (the Trainer updates the colour grid on a side stream)
            import torch
            torch.cuda.synchronize(d.device)
        return d.detach().cpu().numpy().copy()

    def set(self, values):
        import torch
        v = torch.as_tensor(np.asarray(values, dtype=self.dtype).reshape(self.shape))
        self.data.copy_(v.to(self.data.device))

    def __repr__(self):
        return f"Param({self.name}, shape={self.shape}, dtype={np.dtype(self.dtype).name})"


class ParamArena:
    """Parameters / gradients as single device buffers with named views."""

    ALIGN = 4  # elements; 16 B for float32 rows and vector Adam
    TOTAL_ALIGN = 256

    def __init__(self, specs, dtype, device):
        """specs: list of (name, shape, group) with group in {"grid", "mlp", "log_s"}."""
        import torch
        self.dtype = np.dtype(dtype)
        self.device = device
        self.params_by_name = {}
        self.order = []
        off = 0
        prev_group = None
        self.group_begin = {}
        for name, shape, group in specs:
            n = int(np.prod(shape)) if shape else 1
            if group == "grid" or group != prev_group or group == "log_s":
                off = (off + self.ALIGN - 1) // self.ALIGN * self.ALIGN
            if group not in self.group_begin:
                self.group_begin[group] = off
            self.params_by_name[name] = Param(self, name, off, shape)
            self.order.append(name)
            off += n
            prev_group = group
        # padded to a multiple of TOTAL_ALIGN so a data-parallel world of up
        # to 64 ranks splits the arena into equal 16-byte-aligned shards
        # (reduce-scatter / sharded Adam / all-gather, parallel.py)
        self.n = (off + self.TOTAL_ALIGN - 1) // self.TOTAL_ALIGN * self.TOTAL_ALIGN
        tdt = _torch_dtype(dtype)
        self.params = torch.zeros(self.n, dtype=tdt, device=device)
        self.grads = torch.zeros(self.n, dtype=tdt, device=device)
        self.grads_clean = True  # grads known to be all-zero
        self.generation = 0      # bumps whenever the gradient arena changes meaning

    def __getitem__(self, name):
        return self.params_by_name[name]

    def params_list(self):
        return [self.params_by_name[n] for n in self.order]

    def zero_grads(self):
        if not self.grads_clean:
            self.grads.zero_()
            self.grads_clean = True


class GridLevel:
    """One dense grid of per-vertex features (gs/feature_grid.py:39-64)."""

    def __init__(self, geom, features):
        self.geom = geom
        self.features = features

    @property
    def width(self):
        return self.features.shape[1]


class MultiGrid:
    """Geometry levels (coarse->fine) + colour level (gs/feature_grid.py:67-117)."""

    def __init__(self, levels, color, lo, hi):
        self.levels = list(levels)
        self.color = color
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)

    @property
    def geom_width(self):
        return sum(l.width for l in self.levels)

    @property
    def finest_voxel(self):
        return min(l.geom.voxel_size for l in self.levels)

    def clamp_points(self, x):
        """gs/feature_grid.py:101-109."""
        margin = 0.5 * self.finest_voxel
        return np.clip(x, self.lo + margin, self.hi - margin)

    def clamp_box(self):
        margin = 0.5 * self.finest_voxel
        return self.lo + margin, self.hi - margin

    def parameters(self):
        return [l.features for l in self.levels] + [self.color.features]


class DecoderNet:
    """ReLU MLP, hidden 32, linear output (gs/decoders.py:30-76)."""

    def __init__(self, layers):
        self.layers = layers  # [(W Param (in, out), b Param (out,))]

    @property
    def in_width(self):
        return self.layers[0][0].shape[0]

    def parameters(self):
        out = []
        for W, b in self.layers:
            out.extend([W, b])
        return out


class ModelState:
    """Everything the objective optimises (gs/renderer.py:69-105)."""

    def __init__(self, grid, geom_net, color_net, log_s, poses, arena):
        self.grid = grid
        self.geom_net = geom_net
        self.color_net = color_net
        self.log_s = log_s
        self.poses = poses
        self.arena = arena

    @property
    def dtype(self):
        return self.arena.dtype

    @property
    def device(self):
        return self.arena.device

    def s_value(self):
        return float(np.exp(self.log_s.numpy()))

    def grid_params(self):
        return [l.features for l in self.grid.levels] + [self.grid.color.features]

    def decoder_params(self):
        return self.geom_net.parameters() + self.color_net.parameters() + [self.log_s]

    def pose_params(self):
        out = []
        for p in self.poses:
            out.extend(p.parameters())
        return out

    @property
    def refine_poses(self):
        return any(p.trainable for p in self.poses)

    def parameters(self):
        return self.grid_params() + self.decoder_params() + self.pose_params()

    def pose_matrices(self):
        return np.stack([p.matrix() for p in self.poses], axis=0)

    def param_names(self):
        """gs/optimizer.py:217-226."""
        names = [f"level{i}" for i in range(len(self.grid.levels))] + ["colorgrid"]
        for tag, net in (("geom", self.geom_net), ("color", self.color_net)):
            for i in range(len(net.layers)):
                names += [f"{tag}_w{i}", f"{tag}_b{i}"]
        names.append("log_s")
        for i, p in enumerate(self.poses):
            if p.trainable:
                names += [f"nu{i}", f"t{i}"]
        return names


def level_dims(lo, hi, voxel_size):
    """gs/feature_grid.py:55-56."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    if np.any(hi <= lo):
        raise ValueError("degenerate world box")
    return np.maximum(np.ceil((hi - lo) / voxel_size).astype(int) + 1, 2)


def allocate_model(lo, hi, voxel_sizes, geom_width, color_voxel, color_width, poses, dtype,
                   device, trainable=None):
    """Create the arena and the container objects (values all zero except the
    pose translations).  ``trainable[f]``: frame f's pose is refined (its nu
    and t join the arena after log_s, gs/optimizer.py:217-226)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    sizes = sorted(voxel_sizes, reverse=True)  # coarse first (gs/feature_grid.py:87)
    cv = sizes[-1] if color_voxel is None else color_voxel
    geoms = [GridGeom(lo, vs, level_dims(lo, hi, vs)) for vs in sizes]
    cgeom = GridGeom(lo, cv, level_dims(lo, hi, cv))
    in_g = geom_width * len(sizes)
    in_c = color_width + 3
    specs = [(f"level{i}", (g.n_vertices, geom_width), "grid") for i, g in enumerate(geoms)]
    specs.append(("colorgrid", (cgeom.n_vertices, color_width), "grid"))
    for tag, iw, ow in (("geom", in_g, 1), ("color", in_c, 3)):
        dims = [iw, HIDDEN_WIDTH, HIDDEN_WIDTH, ow]
        for i, (a, b) in enumerate(zip(dims[:-1], dims[1:])):
            specs.append((f"{tag}_w{i}", (a, b), f"mlp_{tag}"))
            specs.append((f"{tag}_b{i}", (b,), f"mlp_{tag}"))
    specs.append(("log_s", (), "log_s"))
    trainable = [False] * len(poses) if trainable is None else [bool(t) for t in trainable]
    for i, tr in enumerate(trainable):
        if tr:
            specs += [(f"nu{i}", (3,), "pose"), (f"t{i}", (3,), "pose")]
    arena = ParamArena(specs, dtype, device)
    levels = [GridLevel(g, arena[f"level{i}"]) for i, g in enumerate(geoms)]
    color = GridLevel(cgeom, arena["colorgrid"])
    grid = MultiGrid(levels, color, lo, hi)
    geom_net = DecoderNet([(arena[f"geom_w{i}"], arena[f"geom_b{i}"]) for i in range(3)])
    color_net = DecoderNet([(arena[f"color_w{i}"], arena[f"color_b{i}"]) for i in range(3)])
    pose_objs = [PoseParam.from_matrix(p, trainable=tr, dtype=dtype,
                                       nu_param=arena[f"nu{i}"] if tr else None,
                                       t_param=arena[f"t{i}"] if tr else None)
                 for i, (p, tr) in enumerate(zip(poses, trainable))]
    return ModelState(grid, geom_net, color_net, arena["log_s"], pose_objs, arena)


def init_parameters(model, seed, truncation, chunk=1 << 24):
    """The reference's random init, stream for stream (gs/optimizer.py:188-199,
    gs/feature_grid.py:58-59, gs/decoders.py:40-49).  Grid draws are
    generated in chunks (the PCG64 stream is position-addressed, so chunking
    yields the same values) and uploaded chunk by chunk."""
    import torch
    dt = model.dtype
    rng = seeds.substream(seed, seeds.GRID_INIT)
    for lev in model.grid.levels + [model.grid.color]:
        p = lev.features
        flat = p.data.view(-1)
        n = p.size
        for s0 in range(0, n, chunk):
            k = min(chunk, n - s0)
            vals = rng.uniform(-FEATURE_INIT_SCALE, FEATURE_INIT_SCALE, size=k).astype(dt)
            flat[s0:s0 + k].copy_(torch.from_numpy(vals))
    for net, idx in ((model.geom_net, 0), (model.color_net, 1)):
        r = seeds.substream(seed, seeds.NET_INIT, idx)
        for W, b in net.layers:
            a = W.shape[0]
            bound = np.sqrt(6.0 / a)
            W.set(r.uniform(-bound, bound, size=W.shape).astype(dt))
            b.set(np.zeros(b.shape, dtype=dt))
    model.log_s.set(np.asarray(np.log(1.0 / truncation), dtype=dt))


def world_box_from_frusta(poses, intrinsics, far_per_frame, padding=0.5):
    """gs/feature_grid.py:186-218."""
    poses = np.asarray(poses, dtype=np.float64)
    far = np.broadcast_to(np.asarray(far_per_frame, dtype=np.float64), (poses.shape[0],))
    corners_px = np.array([[0.0, 0.0], [intrinsics.width, 0.0], [0.0, intrinsics.height],
                           [intrinsics.width, intrinsics.height]])
    dirs = np.stack([(corners_px[:, 0] - intrinsics.cx) / intrinsics.fx,
                     (corners_px[:, 1] - intrinsics.cy) / intrinsics.fy, np.ones(4)], axis=1)
    pts = [poses[:, :3, 3]]
    for f in range(poses.shape[0]):
        world_dirs = dirs @ poses[f, :3, :3].T
        pts.append(poses[f, :3, 3] + far[f] * world_dirs)
    allpts = np.concatenate(pts, axis=0)
    return allpts.min(axis=0) - padding, allpts.max(axis=0) + padding


def derive_bounds(dataset, cfg):
    """gs/optimizer.py:146-178 (every 4th pixel; camera centres; padding)."""
    from . import camera
    if cfg.bounds is not None:
        return (np.asarray(cfg.bounds[0], dtype=np.float64),
                np.asarray(cfg.bounds[1], dtype=np.float64))
    intr = dataset.intrinsics
    lo = np.full(3, np.inf)
    hi = np.full(3, -np.inf)
    any_depth = False
    step = 4
    for f in range(len(dataset)):
        d = dataset.depths_mm[f][::step, ::step].astype(np.float64) / 1000.0
        v, u = np.nonzero(d > 0)
        if not v.size:
            continue
        any_depth = True
        pix = np.stack([u * step, v * step], axis=1).astype(np.float64)
        dirs_c = camera.pixel_rays(intr, pix)
        scale = camera.ray_to_z_scale(intr, pix)
        R, t = dataset.poses[f, :3, :3], dataset.poses[f, :3, 3]
        pts = t + (dirs_c * (d[v, u] * scale)[:, None]) @ R.T
        lo = np.minimum(lo, pts.min(axis=0))
        hi = np.maximum(hi, pts.max(axis=0))
    if not any_depth:
        far = np.full(len(dataset), cfg.max_depth)
        return world_box_from_frusta(dataset.poses, intr, far, padding=cfg.bounds_padding)
    centers = dataset.poses[:, :3, 3]
    lo = np.minimum(lo, centers.min(axis=0)) - cfg.bounds_padding
    hi = np.maximum(hi, centers.max(axis=0)) + cfg.bounds_padding
    return lo, hi
