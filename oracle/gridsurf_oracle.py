"""CPU oracle for one GO-Surf training step -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
it.  The GPU path in ``paper_2206_14735_b200`` never calls into it.

It restates, in plain numpy, the reference's per-iteration optimisation
step (``gs/`` = ``/root/reference/pkg/src/gridsurf/``):

    draw_ray_batch            gs/sampler.py:58-88
    train_objective (forward) gs/renderer.py:279-468
    dc.grad(total, params)    gs/diffcore.py:1035-1104  (hand-derived adjoints,
                              SURVEY.md Appendix A; no generic autodiff)
    Adam.step                 gs/optimizer.py:38-91

Forward values are computed with the *same numpy operations in the same
order* as the reference, so in both precisions every forward quantity
(ray batch, stratified and importance depths, phi, grad-phi, colours,
weights, loss parts) is bit-identical to the reference run on the same
machine (pinned by ``tests/golden``).  The backward uses closed-form
adjoints instead of the tape; it agrees with the reference to ~1e-15
relative in double precision and to ~1e-5 (max-norm relative) in single.

Parity pinning: ``tests/golden/make_golden.py`` runs the reference package
itself and stores its outputs; ``tests/test_oracle_golden.py`` checks this
module against them.
"""

from __future__ import annotations

import numpy as np

SIGMA_FLOOR = 1e-12  # gs/renderer.py:42
TRANS_FLOOR = 1e-15  # gs/renderer.py:43
MIN_SEPARATION = 1e-9  # gs/sampler.py:32

# stream tags, gs/seeds.py:14-25
RAYS, STRATIFY, IMPORTANCE, SMOOTH = 1, 2, 3, 4
SPHERE_INIT, NET_INIT, GRID_INIT = 7, 9, 10


def substream(seed, tag, *indices):
    """gs/seeds.py:28-30."""
    return np.random.default_rng(
        np.random.SeedSequence((int(seed), int(tag)) + tuple(int(i) for i in indices)))


# ---------------------------------------------------------------------------
# camera (gs/camera.py:142-171)


def pixel_rays(intr, pixels):
    """gs/camera.py:142-157 (float64)."""
    px = np.atleast_2d(np.asarray(pixels, dtype=np.float64))
    d = np.stack([(px[:, 0] - intr.cx) / intr.fx, (px[:, 1] - intr.cy) / intr.fy,
                  np.ones(px.shape[0])], axis=1)
    return d / np.linalg.norm(d, axis=1, keepdims=True)


def ray_to_z_scale(intr, pixels):
    """gs/camera.py:160-171."""
    px = np.atleast_2d(np.asarray(pixels, dtype=np.float64))
    d = np.stack([(px[:, 0] - intr.cx) / intr.fx, (px[:, 1] - intr.cy) / intr.fy,
                  np.ones(px.shape[0])], axis=1)
    return np.linalg.norm(d, axis=1)


# ---------------------------------------------------------------------------
# sampler (gs/sampler.py)


class Batch:
    """gs/sampler.py:35-55 (RayBatch)."""

    def __init__(self, frame_ids, pixels, color, depth_ray, valid, dir_cam, near, far):
        self.frame_ids, self.pixels, self.color = frame_ids, pixels, color
        self.depth_ray, self.valid, self.dir_cam = depth_ray, valid, dir_cam
        self.near, self.far = near, far

    def __len__(self):
        return self.frame_ids.shape[0]


def draw_ray_batch(dataset, rng, m, near=0.01, far=8.0):
    """gs/sampler.py:58-88."""
    intr = dataset.intrinsics
    f = dataset.colors.shape[0]
    h, w = intr.height, intr.width
    flat = rng.integers(0, f * h * w, size=m)
    return batch_from_flat(dataset, flat, near, far)


def batch_from_flat(dataset, flat, near=0.01, far=8.0):
    """Deterministic part of gs/sampler.py:70-88 given the drawn flat ids."""
    intr = dataset.intrinsics
    h, w = intr.height, intr.width
    m = flat.shape[0]
    frame = flat // (h * w)
    rem = flat % (h * w)
    v, u = rem // w, rem % w
    pixels = np.stack([u, v], axis=1).astype(np.float64)
    color = dataset.colors[frame, v, u].astype(np.float64)
    depth_z = dataset.depths[frame, v, u].astype(np.float64)
    valid = depth_z > 0
    scale = ray_to_z_scale(intr, pixels)
    return Batch(frame.astype(np.int64), pixels, color, depth_z * scale, valid,
                 pixel_rays(intr, pixels), np.full(m, near), np.full(m, far))


def stratified_coarse(near, far, n, uniforms):
    """gs/sampler.py:91-107."""
    near = np.asarray(near)
    far = np.asarray(far)
    if np.any(far <= near):
        raise ValueError("degenerate ray bounds")
    steps = (np.arange(n) + uniforms) / n
    return near[:, None] + (far - near)[:, None] * steps


def enforce_separation(depths, min_sep=MIN_SEPARATION):
    """gs/sampler.py:172-197."""
    d = np.asarray(depths)
    gaps = np.diff(d, axis=1)
    bad_rows = np.where((gaps < min_sep).any(axis=1))[0]
    if bad_rows.size == 0:
        return d
    d = d.copy()
    k = d.shape[1]
    for r in bad_rows:
        row = list(d[r])
        kept = [row[0]]
        for x in row[1:]:
            if x - kept[-1] >= min_sep:
                kept.append(x)
        while len(kept) < k:
            diffs = np.diff(kept)
            j = int(np.argmax(diffs))
            kept.insert(j + 1, kept[j] + diffs[j] / 2.0)
        d[r] = kept
    return d


def importance_refine_with_sources(depths, weights, near, far, uniforms):
    """gs/sampler.py:128-169."""
    depths = np.asarray(depths)
    w = np.asarray(weights)[:, :-1].copy()
    if np.any(w < 0):
        raise ValueError("weights must be non-negative")
    m, a = uniforms.shape
    k = depths.shape[1]
    total = w.sum(axis=1, keepdims=True)
    dead = total[:, 0] <= 0.0
    w[dead] = 1.0
    cdf = np.cumsum(w, axis=1)
    cdf /= cdf[:, -1:]
    idx = np.sum(cdf[:, None, :] <= uniforms[:, :, None], axis=2)
    idx = np.minimum(idx, w.shape[1] - 1)
    cdf_pad = np.concatenate([np.zeros((m, 1)), cdf], axis=1)
    lo = np.take_along_axis(cdf_pad, idx, axis=1)
    hi = np.take_along_axis(cdf_pad, idx + 1, axis=1)
    frac = np.where(hi > lo, (uniforms - lo) / np.maximum(hi - lo, 1e-300), 0.5)
    d_lo = np.take_along_axis(depths, idx, axis=1)
    d_hi = np.take_along_axis(depths, idx + 1, axis=1)
    new = d_lo + frac * (d_hi - d_lo)
    if np.any(dead):
        new[dead] = near[dead, None] + uniforms[dead] * (far - near)[dead, None]
    cat = np.concatenate([depths, new], axis=1)
    src = np.concatenate(
        [np.tile(np.arange(k), (m, 1)), np.full((m, a), -1, dtype=np.int64)], axis=1)
    order = np.argsort(cat, axis=1, kind="stable")
    merged = np.take_along_axis(cat, order, axis=1)
    src = np.take_along_axis(src, order, axis=1)
    out = enforce_separation(merged)
    src = np.where(out == merged, src, -1)
    return out, src


# ---------------------------------------------------------------------------
# trilinear grid (gs/diffcore.py:704-920)


class GridBoundsError(ValueError):
    pass


class Level:
    """GridGeom + features (gs/diffcore.py:704-728, gs/feature_grid.py:39-64)."""

    def __init__(self, origin, voxel_size, dims, feat):
        self.origin = np.asarray(origin, dtype=np.float64)
        self.voxel_size = float(voxel_size)
        self.dims = tuple(int(d) for d in dims)
        self.feat = feat

    @property
    def n_vertices(self):
        return self.dims[0] * self.dims[1] * self.dims[2]


_CORNER_OFFSETS = np.array(
    [[dx, dy, dz] for dx in (0, 1) for dy in (0, 1) for dz in (0, 1)], dtype=np.int64)


def locate(points, lev):
    """gs/diffcore.py:738-751."""
    local = (points - lev.origin) / lev.voxel_size
    dims = np.array(lev.dims)
    eps = 1e-9 * max(lev.dims)
    if np.any(local < -eps) or np.any(local > (dims - 1) + eps):
        raise GridBoundsError("sample point(s) outside grid box")
    cell = np.minimum(np.floor(local).astype(np.int64), dims - 2)
    cell = np.maximum(cell, 0)
    return cell, local - cell


def corner_index(cell, lev):
    """gs/diffcore.py:754-758 (x-major, z fastest; k = 4dx + 2dy + dz)."""
    nx, ny, nz = lev.dims
    flat = (cell[:, 0] * ny + cell[:, 1]) * nz + cell[:, 2]
    offs = (_CORNER_OFFSETS[:, 0] * ny + _CORNER_OFFSETS[:, 1]) * nz + _CORNER_OFFSETS[:, 2]
    return flat[:, None] + offs[None, :]


def corner_weights(frac):
    """gs/diffcore.py:761-767."""
    fx, fy, fz = frac[:, 0], frac[:, 1], frac[:, 2]
    wx = np.stack([1.0 - fx, fx], axis=1)
    wy = np.stack([1.0 - fy, fy], axis=1)
    wz = np.stack([1.0 - fz, fz], axis=1)
    w = wx[:, :, None, None] * wy[:, None, :, None] * wz[:, None, None, :]
    return w.reshape(frac.shape[0], 8)


def corner_jacobian(frac):
    """d w_k / d frac_a, (N, 8, 3): gs/diffcore.py:770-780."""
    fx, fy, fz = frac[:, 0], frac[:, 1], frac[:, 2]
    wx = np.stack([1.0 - fx, fx], axis=1)
    wy = np.stack([1.0 - fy, fy], axis=1)
    wz = np.stack([1.0 - fz, fz], axis=1)
    sx = np.stack([-np.ones_like(fx), np.ones_like(fx)], axis=1)
    jx = (sx[:, :, None, None] * wy[:, None, :, None] * wz[:, None, None, :]).reshape(-1, 8)
    jy = (wx[:, :, None, None] * sx[:, None, :, None] * wz[:, None, None, :]).reshape(-1, 8)
    jz = (wx[:, :, None, None] * wy[:, None, :, None] * sx[:, None, None, :]).reshape(-1, 8)
    return np.stack([jx, jy, jz], axis=2)


def gather_weighted(feat, idx8, w8):
    """gs/diffcore.py:816-827 with numba's arithmetic: the f64 product is
    added to the storage-dtype accumulator and rounded back per corner."""
    dt = feat.dtype
    out = np.zeros((idx8.shape[0], feat.shape[1]), dtype=dt)
    for k in range(8):
        out = (out + w8[:, k:k + 1] * feat[idx8[:, k]]).astype(dt)
    return out


def scatter_weighted(idx8, w8, g, n_vertices):
    """gs/diffcore.py:830-841 (accumulated in float64, returned in g's dtype)."""
    out = np.zeros((n_vertices, g.shape[1]), dtype=np.float64)
    for k in range(8):
        np.add.at(out, idx8[:, k], w8[:, k:k + 1] * g.astype(np.float64))
    return out.astype(g.dtype)


class LevelSample:
    """Per-point lattice location for one level (everything grid_sample keeps)."""

    def __init__(self, lev, pts):
        cell, self.frac = locate(pts, lev)
        self.idx8 = corner_index(cell, lev)
        self.w8 = corner_weights(self.frac)
        self.lev = lev

    def value(self):
        return gather_weighted(self.lev.feat, self.idx8, self.w8)

    def ju(self, u):
        """gs/diffcore.py:874-890: ju[n,k] = sum_a dw_k/dx_a u_a (world units)."""
        J = corner_jacobian(self.frac)  # (N, 8, 3) cell units
        return np.einsum("nka,na->nk", J, u.astype(np.float64)) / self.lev.voxel_size

    def dx(self, g):
        """gs/diffcore.py:844-871: grad_x <interp(feat, x), g>, (N, 3) in g.dtype,
        with numba's arithmetic (storage-dtype channel products summed into a
        float64 accumulator, per-corner rounding of the output)."""
        dt = g.dtype
        feat = self.lev.feat
        fx, fy, fz = self.frac[:, 0], self.frac[:, 1], self.frac[:, 2]
        out = np.zeros((g.shape[0], 3), dtype=dt)
        for k in range(8):
            rows = feat[self.idx8[:, k]]
            acc = np.zeros(g.shape[0], dtype=np.float64)
            for j in range(g.shape[1]):
                acc = acc + (rows[:, j] * g[:, j]).astype(np.float64)
            wx = fx if k & 4 else 1.0 - fx
            wy = fy if k & 2 else 1.0 - fy
            wz = fz if k & 1 else 1.0 - fz
            sx = 1.0 if k & 4 else -1.0
            sy = 1.0 if k & 2 else -1.0
            sz = 1.0 if k & 1 else -1.0
            out[:, 0] = (out[:, 0] + acc * sx * wy * wz).astype(dt)
            out[:, 1] = (out[:, 1] + acc * wx * sy * wz).astype(dt)
            out[:, 2] = (out[:, 2] + acc * wx * wy * sz).astype(dt)
        inv_vs = 1.0 / self.lev.voxel_size
        return (out * inv_vs).astype(dt)


def sigmoid_raw(x):
    """gs/diffcore.py:445-451."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


# ---------------------------------------------------------------------------
# model container


# ---------------------------------------------------------------------------
# poses: Rodrigues map (gs/camera.py:93-139) and its adjoint

SMALL_ANGLE = 1e-4  # gs/camera.py:93


def exp_so3_data(nu):
    """gs/camera.py:125-139 (plain f64)."""
    nu = np.asarray(nu, dtype=np.float64)
    th2 = float(nu @ nu)
    K = np.array([[0.0, -nu[2], nu[1]], [nu[2], 0.0, -nu[0]], [-nu[1], nu[0], 0.0]])
    if np.sqrt(th2) < SMALL_ANGLE:
        a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0
        b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0
    else:
        th = np.sqrt(th2)
        a = np.sin(th) / th
        b = (1.0 - np.cos(th)) / th2
    return np.eye(3) + a * K + b * (K @ K)


def exp_so3_graph(nu):
    """gs/camera.py:96-122 evaluated as the graph does, in nu's dtype.
    Returns E and what the adjoint needs."""
    dt = nu.dtype
    z = np.zeros(1, dtype=dt)
    n0, n1, n2 = nu[0:1], nu[1:2], nu[2:3]
    K = np.concatenate([z, -n2, n1, n2, z, -n0, -n1, n0, z]).reshape(3, 3)
    K2 = np.matmul(K, K)
    th2 = (nu * nu).sum()
    small = float(np.sqrt(th2.item())) < SMALL_ANGLE
    if small:
        a = 1.0 + th2 * (-1.0 / 6.0) + th2 * th2 * (1.0 / 120.0)
        b = 0.5 + th2 * (-1.0 / 24.0) + th2 * th2 * (1.0 / 720.0)
        th = None
    else:
        th = np.sqrt(th2)
        a = np.sin(th) / th
        b = (dt.type(1.0) - np.cos(th)) / th2
    a, b = np.asarray(a, dtype=dt), np.asarray(b, dtype=dt)
    E = np.eye(3, dtype=dt) + a.reshape(1, 1) * K + b.reshape(1, 1) * K2
    return E, dict(K=K, K2=K2, th2=th2, th=th, a=a, b=b, small=small)


def exp_so3_adjoint(nu, aux, Ebar):
    """d/dnu of <E(nu), Ebar> through the graph of gs/camera.py:96-122."""
    dt = nu.dtype
    K, K2, th2, th, a, b = (aux[k] for k in ("K", "K2", "th2", "th", "a", "b"))
    abar = (Ebar * K).sum()
    bbar = (Ebar * K2).sum()
    K2bar = b * Ebar
    Kbar = a * Ebar + np.matmul(K2bar, K.T) + np.matmul(K.T, K2bar)
    if aux["small"]:
        th2bar = abar * (dt.type(-1.0 / 6.0) + dt.type(2.0 / 120.0) * th2) \
            + bbar * (dt.type(-1.0 / 24.0) + dt.type(2.0 / 720.0) * th2)
    else:
        s, c = np.sin(th), np.cos(th)
        thbar = abar * (c / th - s / (th * th)) + bbar * (s / th2)
        th2bar = thbar / (dt.type(2.0) * th) - bbar * (dt.type(1.0) - c) / (th2 * th2)
    nubar = dt.type(2.0) * nu * th2bar
    nubar = nubar + np.array([Kbar[2, 1] - Kbar[1, 2], Kbar[0, 2] - Kbar[2, 0],
                              Kbar[1, 0] - Kbar[0, 1]], dtype=dt)
    return nubar.astype(dt)


def pair_hessian(v, frac):
    """gs/diffcore.py:783-804: off-diagonal trilinear Hessian (cell units)."""
    fx, fy, fz = frac[:, 0], frac[:, 1], frac[:, 2]
    h12 = (1.0 - fz) * (v[:, 0] + v[:, 6] - v[:, 2] - v[:, 4]) + fz * (v[:, 1] + v[:, 7] - v[:, 3] - v[:, 5])
    h13 = (1.0 - fy) * (v[:, 0] + v[:, 5] - v[:, 1] - v[:, 4]) + fy * (v[:, 2] + v[:, 7] - v[:, 3] - v[:, 6])
    h23 = (1.0 - fx) * (v[:, 0] + v[:, 3] - v[:, 1] - v[:, 2]) + fx * (v[:, 4] + v[:, 7] - v[:, 5] - v[:, 6])
    return h12, h13, h23


class Params:
    """ModelState restated (gs/renderer.py:69-105): grids coarse->fine,
    colour grid, two DecoderNets [(W (in,out), b)], log_s, frozen poses."""

    def __init__(self, levels, color, geom, color_net, log_s, lo, hi, poses, trainable=None):
        self.levels, self.color = levels, color
        self.geom, self.color_net = geom, color_net
        self.log_s = log_s
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        self.poses = np.asarray(poses, dtype=np.float64)  # (F, 4, 4)
        # PoseParam (gs/camera.py:53-90): R0 f64, nu / t in the model dtype
        F = self.poses.shape[0]
        dt = self.dtype
        self.trainable = np.zeros(F, dtype=bool) if trainable is None else np.asarray(trainable, bool)
        self.R0 = self.poses[:, :3, :3].copy()
        self.nu = [np.zeros(3, dtype=dt) for _ in range(F)]
        self.t = [self.poses[i, :3, 3].astype(dt) for i in range(F)]

    @property
    def dtype(self):
        return self.levels[0].feat.dtype

    @property
    def finest_voxel(self):
        return min(l.voxel_size for l in self.levels)

    def pose_matrices(self):
        """gs/renderer.py:104-105 / gs/camera.py:75-80: R0 @ exp_so3_data(nu)
        (f64) and the translation as stored (PoseParam.t is in the model dtype)."""
        m = np.zeros((len(self.nu), 4, 4))
        m[:, 3, 3] = 1.0
        for i in range(len(self.nu)):
            m[i, :3, :3] = self.R0[i] @ exp_so3_data(self.nu[i])
            m[i, :3, 3] = np.asarray(self.t[i], dtype=np.float64)
        return m

    def names(self):
        """gs/optimizer.py:217-226."""
        n = [f"level{i}" for i in range(len(self.levels))] + ["colorgrid"]
        for tag, net in (("geom", self.geom), ("color", self.color_net)):
            for i in range(len(net)):
                n += [f"{tag}_w{i}", f"{tag}_b{i}"]
        n.append("log_s")
        for i in np.nonzero(self.trainable)[0]:
            n += [f"nu{i}", f"t{i}"]
        return n

    def arrays(self):
        out = [l.feat for l in self.levels] + [self.color.feat]
        for net in (self.geom, self.color_net):
            for W, b in net:
                out += [W, b]
        out.append(self.log_s)
        for i in np.nonzero(self.trainable)[0]:
            out += [self.nu[i], self.t[i]]
        return out

    def lrs(self, lr_grids=1e-2, lr_decoders=1e-3, lr_poses=5e-4):
        """gs/optimizer.py:229-236."""
        ng = len(self.levels) + 1
        npose = 2 * int(self.trainable.sum())
        return [lr_grids] * ng + [lr_decoders] * (len(self.arrays()) - ng - npose) + [lr_poses] * npose

    def refresh_poses(self):
        """PoseParam.refresh, gs/camera.py:82-87: fold exp(nu) into R0, zero nu."""
        for i in np.nonzero(self.trainable)[0]:
            self.R0[i] = self.R0[i] @ exp_so3_data(self.nu[i])
            self.nu[i][...] = 0.0

    def copy(self):
        cp = lambda l: Level(l.origin, l.voxel_size, l.dims, l.feat.copy())
        P = Params([cp(l) for l in self.levels], cp(self.color),
                   [(W.copy(), b.copy()) for W, b in self.geom],
                   [(W.copy(), b.copy()) for W, b in self.color_net],
                   self.log_s.copy(), self.lo, self.hi, self.poses, self.trainable)
        P.R0 = self.R0.copy()
        P.nu = [a.copy() for a in self.nu]
        P.t = [a.copy() for a in self.t]
        return P


def create_params(lo, hi, poses, seed=0, voxel_sizes=(0.96, 0.24, 0.06, 0.03),
                  geom_width=4, color_voxel=None, color_width=6, dtype=np.float64,
                  truncation=0.16, refine_poses=False, freeze_first_pose=True):
    """build_model(skip_init=True) restated: gs/optimizer.py:181-205,
    MultiGrid.create gs/feature_grid.py:48-91, DecoderNet.create
    gs/decoders.py:40-49 (same RNG streams and draw order)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    rng = substream(seed, GRID_INIT)

    def level(vs, width):
        dims = np.maximum(np.ceil((hi - lo) / vs).astype(int) + 1, 2)
        n = int(np.prod(dims))
        feats = rng.uniform(-1e-4, 1e-4, size=(n, width)).astype(dtype)
        return Level(lo, vs, dims, feats)

    sizes = sorted(voxel_sizes, reverse=True)
    levels = [level(vs, geom_width) for vs in sizes]
    color = level(sizes[-1] if color_voxel is None else color_voxel, color_width)

    def net(in_w, out_w, r):
        sz = [in_w, 32, 32, out_w]
        layers = []
        for a, b in zip(sz[:-1], sz[1:]):
            bound = np.sqrt(6.0 / a)
            W = r.uniform(-bound, bound, size=(a, b)).astype(dtype)
            layers.append((W, np.zeros(b, dtype=dtype)))
        return layers

    geom = net(geom_width * len(levels), 1, substream(seed, NET_INIT, 0))
    cnet = net(color_width + 3, 3, substream(seed, NET_INIT, 1))
    log_s = np.asarray(np.log(1.0 / truncation), dtype=dtype)
    F = np.asarray(poses).shape[0]
    trainable = [refine_poses and not (freeze_first_pose and i == 0) for i in range(F)]
    return Params(levels, color, geom, cnet, log_s, lo, hi, poses, trainable)


def mlp_forward(layers, x):
    """gs/decoders.py:55-63: returns (pre-activations, activations, out)."""
    h = x
    pre, acts = [], []
    last = len(layers) - 1
    for i, (W, b) in enumerate(layers):
        a = np.matmul(h, W) + b.reshape(1, -1)
        pre.append(a)
        if i < last:
            h = np.maximum(a, 0.0)
            acts.append(h)
        else:
            h = a
    return pre, acts, h


def sample_multi(P, pts):
    """gs/feature_grid.py:135-139."""
    ls = [LevelSample(l, pts) for l in P.levels]
    return ls, np.concatenate([s.value() for s in ls], axis=1)


def phi_data(P, pts):
    """gs/renderer.py:236-240."""
    _, z = sample_multi(P, pts)
    return mlp_forward(P.geom, z)[2][:, 0]


def render_weights_data(phi, s):
    """gs/renderer.py:162-173."""
    sig = sigmoid_raw(s * phi)
    ratio = sig[:, 1:] / np.maximum(sig[:, :-1], SIGMA_FLOOR)
    om = np.concatenate(
        [np.minimum(ratio, 1.0), np.ones((phi.shape[0], 1), dtype=phi.dtype)], axis=1)
    trans = np.cumprod(
        np.concatenate([np.ones((phi.shape[0], 1), dtype=phi.dtype), om[:, :-1]], axis=1),
        axis=1)
    return trans * (1.0 - om)


def box_exit(origins, dirs, lo, hi):
    """gs/renderer.py:228-233."""
    r = np.where(np.abs(dirs) < 1e-12, 1e-12, dirs)
    t1 = (lo - origins) / r
    t2 = (hi - origins) / r
    return np.min(np.maximum(t1, t2), axis=1)


def draw_smooth_points(P, dataset, count, truncation, delta, rng):
    """gs/renderer.py:243-276."""
    frames, vs, us = dataset.valid_pixels
    if frames.size == 0:
        return None
    pick = rng.integers(0, frames.size, size=count)
    f, v, u = frames[pick], vs[pick], us[pick]
    pixels = np.stack([u, v], axis=1).astype(np.float64)
    intr = dataset.intrinsics
    d_cam = pixel_rays(intr, pixels)
    scale = ray_to_z_scale(intr, pixels)
    depth_ray = dataset.depths[f, v, u] * scale + rng.uniform(-truncation, truncation, size=count)
    mats = P.pose_matrices()[f]
    dirs = np.einsum("nij,nj->ni", mats[:, :3, :3], d_cam)
    x = mats[:, :3, 3] + depth_ray[:, None] * dirs
    margin = 0.5 * P.finest_voxel
    x = np.clip(x, P.lo + margin, P.hi - margin)
    lo, hi = P.lo + margin, P.hi - margin
    eps_dir = rng.normal(size=(count, 8, 3))
    eps_dir /= np.linalg.norm(eps_dir, axis=2, keepdims=True)
    cand = x[:, None, :] + delta * eps_dir
    ok = ((cand >= lo) & (cand <= hi)).all(axis=2)
    first = np.argmax(ok, axis=1)
    xe = cand[np.arange(count), first]
    xe = np.clip(xe, lo, hi)
    return x, xe


# ---------------------------------------------------------------------------
# geometry sample pass: phi, grad phi, and its adjoint


class GeomPass:
    """phi and grad-phi at points, with what the backward needs.

    grad phi follows gs/renderer.py:358: the MLP vjp gives g = dphi/dz
    (ReLU masks a > 0, gs/diffcore.py:483-492) and each level adds
    J_l^T g_l (gs/diffcore.py:946-991)."""

    def __init__(self, P, pts, flips=()):
        """``flips``: (layer, row, unit) whose ReLU derivative mask is taken on
        the other side of the kink (test-only: a pre-activation within
        rounding of zero, where a float32 run may have gone the other way)."""
        dt = P.dtype
        self.P = P
        self.ls, self.z = sample_multi(P, pts)
        (a0, a1, a2), (h0, h1), out = mlp_forward(P.geom, self.z)
        self.phi = out[:, 0]
        self.h0, self.h1 = h0, h1
        self.pre = (a0, a1)  # ReLU pre-activations (conditioned-parity kink margins)
        self.m0 = (a0 > 0).astype(dt)
        self.m1 = (a1 > 0).astype(dt)
        for layer, row, unit in flips:
            m = self.m0 if layer == 0 else self.m1
            m[row, unit] = 1 - m[row, unit]
        W0, W1, W2 = (P.geom[i][0] for i in range(3))
        ones = np.ones((self.z.shape[0], 1), dtype=dt)
        self.d1 = np.matmul(ones, W2.T) * self.m1
        self.d0 = np.matmul(self.d1, W1.T) * self.m0
        self.g = np.matmul(self.d0, W0.T)
        c = P.levels[0].feat.shape[1]
        gphi = None
        for l, s in enumerate(self.ls):
            part = s.dx(self.g[:, l * c:(l + 1) * c])
            gphi = part if gphi is None else gphi + part
        self.gphi = gphi

    def backward(self, p, u, grads):
        """Accumulate d/dtheta of sum_n p_n phi_n + u_n . gradphi_n
        (SURVEY.md Appendix A)."""
        P = self.P
        dt = P.dtype
        c = P.levels[0].feat.shape[1]
        W0, W1 = P.geom[0][0], P.geom[1][0]
        pc = p.astype(dt)[:, None]
        v = np.zeros_like(self.z)
        for l, s in enumerate(self.ls):
            ju = s.ju(u)  # (N,8) f64
            gl = self.g[:, l * c:(l + 1) * c]
            coef = s.w8 * p.astype(np.float64)[:, None] + ju
            grads[f"level{l}"] += scatter_weighted(s.idx8, coef, gl, s.lev.n_vertices)
            v[:, l * c:(l + 1) * c] = gather_weighted(s.lev.feat, s.idx8, ju)
        q0 = np.matmul(v, W0) * self.m0
        dd1 = np.matmul(q0, W1) * self.m1
        grads["geom_w0"] += np.matmul((pc * self.z + v).T, self.d0)
        grads["geom_w1"] += np.matmul((pc * self.h0 + q0).T, self.d1)
        grads["geom_w2"] += (pc * self.h1 + dd1).sum(axis=0)[:, None]
        grads["geom_b0"] += (pc * self.d0).sum(axis=0)
        grads["geom_b1"] += (pc * self.d1).sum(axis=0)
        grads["geom_b2"] += pc.sum(axis=0)


# ---------------------------------------------------------------------------
# the objective (gs/renderer.py:279-468) and its gradient


def train_objective(P, dataset, batch, iteration, cfg, smooth_override=None,
                    want_grads=True, inject_depths=None, shard=None, inject_rays=None,
                    point_dtype=None, relu_flips=None):
    """One evaluation of the training objective and (optionally) all
    parameter gradients.  Returns a dict of every intermediate.

    ``inject_depths`` replaces the sampled depths (M, N) for component
    parity (the taped pass of another implementation given our samples).
    ``inject_rays`` = (o, r) (M, 3) replaces the realised ray origins and
    directions, and ``point_dtype`` forms the taped points x = o + d r (and
    their clip to the box) in that dtype before the cast to the model dtype
    (gs/renderer.py:348-351 forms them in the model dtype).  Together they
    give the float64 evaluation of the taped pass at exactly the float32
    points a float32 implementation used (conditioned kernel parity).
    ``relu_flips`` = {"geom" | "smooth" | "color": [(layer, row, unit)]}
    takes those ReLU derivative masks on the other side of their kink
    (GeomPass); ``relu_flips["ratio"]`` = [(ray, j)] does the same for the
    derivative of min(ratio, 1) in the alphas (gs/renderer.py:112-134) at
    sigma_{j+1} / sigma_j = 1; test-only.

    ``shard`` (data-parallel restatement; not in the
    reference): dict with ``row_base`` and ``m_global`` (this batch is rows
    [row_base, row_base + m) of a global batch: the stratify / importance
    uniforms are those rows of the global draws), optional global
    normalisers ``n_valid`` / ``n_eik`` / ``n_smooth``, and ``smooth``
    (False: this shard owns no smoothness points).  The shard's parts and
    gradients then sum over shards to the unsharded step."""
    lw = cfg.weights
    dt = P.dtype
    m = len(batch)
    sh = shard or {}
    row0 = int(sh.get("row_base", 0))
    m_glob = int(sh.get("m_global", m))
    margin = 0.5 * P.finest_voxel
    lo_c, hi_c = P.lo + margin, P.hi - margin
    R = {}

    # ray setup: gs/renderer.py:302-317; R = R0 @ exp_so3(nu) in the model
    # dtype (gs/camera.py:68-70, exactly R0 for nu = 0)
    uniq, inv, pose_aux, o, r = realised_rays(P, batch)
    if inject_rays is not None:
        o, r = (np.asarray(a).astype(dt).reshape(m, 3) for a in inject_rays)
    o_data, r_data = o.astype(np.float64), r.astype(np.float64)
    if cfg.fixed_far is not None:
        far = np.full(m, float(cfg.fixed_far))
    else:
        far = np.minimum(box_exit(o_data, r_data, lo_c, hi_c), batch.far)
    near = batch.near
    far = np.maximum(far, near + 0.05)
    R.update(o=o, r=r, far=far)

    # sampling: gs/renderer.py:319-346
    s_val = float(np.exp(P.log_s))
    u0 = substream(cfg.seed, STRATIFY, iteration).random((m_glob, cfg.coarse_samples))[row0:row0 + m]
    depths = stratified_coarse(near, far, cfg.coarse_samples, u0)
    R["depths0"] = depths

    def phi_at(dep_rows, rows):
        pts = o_data[rows] + dep_rows[:, None] * r_data[rows]
        pts = np.clip(pts, lo_c, hi_c).astype(dt)
        return phi_data(P, pts).reshape(-1).astype(np.float64)

    phi_cache = None
    R["rounds"] = []
    for rnd in range(cfg.importance_rounds):
        if phi_cache is None:
            rows = np.repeat(np.arange(m), depths.shape[1])
            phi_cache = phi_at(depths.reshape(-1), rows).reshape(m, -1)
        w = render_weights_data(phi_cache, s_val)
        ui = substream(cfg.seed, IMPORTANCE, iteration, rnd).random(
            (m_glob, cfg.importance_add))[row0:row0 + m]
        prev_phi = phi_cache
        depths, src = importance_refine_with_sources(depths, w, near, far, ui)
        nxt = np.take_along_axis(phi_cache, np.maximum(src, 0), axis=1)
        need_r, need_c = np.nonzero(src < 0)
        if need_r.size:
            nxt[need_r, need_c] = phi_at(depths[need_r, need_c], need_r)
        phi_cache = nxt
        R["rounds"].append(dict(phi_in=prev_phi, weights=w, depths=depths, src=src))
    if inject_depths is not None:
        depths = np.asarray(inject_depths, dtype=np.float64)
    n = depths.shape[1]
    R["depths"] = depths

    # taped pass: gs/renderer.py:348-370
    pdt = dt if point_dtype is None else np.dtype(point_dtype)
    x = o.astype(pdt).reshape(m, 1, 3) + depths[:, :, None].astype(pdt) * r.astype(pdt).reshape(m, 1, 3)
    xu = x.reshape(m * n, 3)
    xf = np.minimum(np.maximum(xu, lo_c.astype(pdt)), hi_c.astype(pdt)).astype(dt)
    xu = xu.astype(dt)
    flips = relu_flips or {}
    G = GeomPass(P, xf, flips.get("geom", ()))
    cs = LevelSample(P.color, xf)
    fc = cs.value()
    vdir = np.broadcast_to(r.reshape(m, 1, 3), (m, n, 3)).reshape(m * n, 3)
    norms = np.linalg.norm(vdir, axis=-1)
    if np.any(np.abs(norms - 1.0) > 1e-6):
        raise ValueError("view directions must be unit length")
    cin = np.concatenate([fc, vdir], axis=1)
    (ca0, ca1, ca2), (ch0, ch1), cy = mlp_forward(P.color_net, cin)
    c_flat = sigmoid_raw(cy)

    phis = G.phi.reshape(m, n)
    colors = c_flat.reshape(m, n, 3)
    s_t = np.exp(P.log_s)  # dt 0-d
    # alphas: gs/renderer.py:112-134
    sig = sigmoid_raw(phis * s_t)
    Dden = np.maximum(sig[:, :-1], dt.type(SIGMA_FLOOR))
    ratio = sig[:, 1:] / Dden
    R["ratio"] = ratio
    head = 1.0 - np.minimum(ratio, 1.0)
    al = np.concatenate([head, np.zeros((m, 1), dtype=dt)], axis=1)
    # composite: gs/renderer.py:137-159
    om = 1.0 - al
    omc = np.maximum(om, dt.type(TRANS_FLOOR))
    logt = np.cumsum(np.log(omc), axis=1)
    trans = np.exp(np.concatenate([np.zeros((m, 1), dtype=dt), logt[:, :n - 1]], axis=1))
    w = trans * al
    dconst = depths.astype(dt)
    chat = (w.reshape(m, n, 1) * colors).sum(axis=1)
    dhat = (w * dconst).sum(axis=1)

    # losses: gs/renderer.py:372-414
    err = chat - batch.color.astype(dt)
    lr_m = np.sqrt((err * err).sum(axis=1) + dt.type(1e-24))
    l_rgb = lr_m.sum() / dt.type(m_glob)
    vmask = batch.valid.astype(dt)
    n_valid = int(batch.valid.sum())
    nv_norm = int(sh.get("n_valid", n_valid))
    d_err = np.abs(dhat - batch.depth_ray.astype(dt))
    l_d = (d_err * vmask).sum() / dt.type(max(nv_norm, 1))
    b = batch.depth_ray[:, None] - depths
    tr_mask = (batch.valid[:, None] & (np.abs(b) <= lw.truncation)).astype(dt)
    fs_mask = (batch.valid[:, None] & (b > lw.truncation)).astype(dt)
    behind_mask = (batch.valid[:, None] & (b < -lw.truncation)).astype(dt)
    b_c = b.astype(dt)
    tr_cnt = tr_mask.sum(axis=1)
    sdf_val = np.abs(phis - b_c) * tr_mask
    per_ray_sdf = sdf_val.sum(axis=1) / np.maximum(tr_cnt, 1.0).astype(dt)
    l_sdf = per_ray_sdf.sum() / dt.type(m_glob)
    fs_cnt = fs_mask.sum(axis=1)
    e5 = np.exp(phis * dt.type(-lw.freespace_alpha))
    inner = np.maximum(dt.type(0.0), e5 - dt.type(1.0))
    fs_raw = np.maximum(inner, phis - b_c)
    per_ray_fs = (fs_raw * fs_mask).sum(axis=1) / np.maximum(fs_cnt, 1.0).astype(dt)
    l_fs = per_ray_fs.sum() / dt.type(m_glob)
    eik_mask = (fs_mask + behind_mask + (~batch.valid[:, None]).astype(dt)).clip(0, 1)
    eik_flat = eik_mask.reshape(-1)
    n_eik = float(max(sh.get("n_eik", eik_flat.sum()), 1.0))
    gp = G.gphi
    nrm = np.sqrt((gp * gp).sum(axis=-1) + dt.type(1e-20))
    diff = 1.0 - nrm
    eik_val = diff * diff
    l_eik = (eik_val * eik_flat.astype(dt)).sum() / dt.type(n_eik)

    # smoothness: gs/renderer.py:416-434
    if smooth_override is not None:
        smooth_pts = smooth_override
    else:
        rng = substream(cfg.seed, SMOOTH, iteration)
        smooth_pts = draw_smooth_points(P, dataset, lw.smooth_count, lw.truncation,
                                        lw.smooth_delta, rng)
    S = None
    if smooth_pts is None or lw.smooth == 0.0 or not sh.get("smooth", True):
        l_smooth = dt.type(0.0)
        n_smooth = 0
    else:
        xs, xe = smooth_pts
        n_smooth = xs.shape[0]
        n_sm_norm = int(sh.get("n_smooth", n_smooth))
        S = GeomPass(P, np.concatenate([xs, xe], axis=0).astype(dt), flips.get("smooth", ()))
        dS = S.gphi[:n_smooth] - S.gphi[n_smooth:]
        l_smooth = (dS * dS).sum() / dt.type(n_sm_norm)
    R["smooth_pts"] = smooth_pts

    total = (l_rgb * dt.type(lw.rgb) + l_d * dt.type(lw.depth) + l_sdf * dt.type(lw.sdf)
             + l_fs * dt.type(lw.fs) + l_eik * dt.type(lw.eik) + l_smooth * dt.type(lw.smooth))
    R["parts"] = {"total": float(total), "rgb": float(l_rgb), "depth": float(l_d),
                  "sdf": float(l_sdf), "fs": float(l_fs), "eik": float(l_eik),
                  "smooth": float(l_smooth), "s": s_val}
    R["extras"] = {"samples_per_ray": n, "n_valid_rays": n_valid,
                   "n_tr": int(tr_cnt.sum()), "n_fs": int(fs_cnt.sum()),
                   "n_eik": int(eik_flat.sum()), "n_smooth": n_smooth,
                   "empty_tr": bool(tr_cnt.sum() == 0), "empty_fs": bool(fs_cnt.sum() == 0)}
    R.update(phi=phis, gphi=gp.reshape(m, n, 3), colors=colors, alpha=al, weights=w,
             chat=chat, dhat=dhat, xf=xf)
    R["pre"] = {"geom": G.pre, "color": (ca0, ca1), "smooth": None if S is None else S.pre}
    R["smooth_gphi"] = None if S is None else S.gphi
    if not want_grads:
        return R

    # ---------------- backward ----------------
    grads = {name: np.zeros_like(a) for name, a in zip(P.names(), P.arrays())}
    M = dt.type(m_glob)
    # photometric + depth seeds
    chat_bar = (dt.type(lw.rgb) / M) * err / lr_m[:, None]
    dhat_bar = dt.type(lw.depth) * vmask * np.sign(dhat - batch.depth_ray.astype(dt)) \
        / dt.type(max(nv_norm, 1))
    w_bar = (chat_bar[:, None, :] * colors).sum(axis=2) + dhat_bar[:, None] * dconst
    c_bar = w[:, :, None] * chat_bar[:, None, :]
    T_bar = w_bar * al
    al_bar = w_bar * trans
    tt = T_bar * trans  # d/d logt_{i-1}
    L_bar = np.zeros_like(al)
    # L_bar_j = sum_{i=j+1}^{n-1} T_bar_i T_i (reverse exclusive scan)
    L_bar[:, :n - 1] = np.flip(np.cumsum(np.flip(tt[:, 1:], axis=1), axis=1), axis=1)
    om_bar = np.where(om >= dt.type(TRANS_FLOOR), L_bar / omc, 0.0).astype(dt)
    al_bar = al_bar - om_bar
    r_take = ratio <= 1.0
    for row, j in flips.get("ratio", ()):
        r_take[row, j] = not r_take[row, j]
    r_bar = np.where(r_take, -al_bar[:, :n - 1], 0.0).astype(dt)
    # size of the phi_bar jump at sample j + 1 if the ratio branch flips (test-only diagnostics)
    R["ratio_jump"] = np.abs(al_bar[:, :n - 1] / Dden * (sig[:, 1:] * (1.0 - sig[:, 1:]))) * s_t
    sig_bar = np.zeros_like(sig)
    sig_bar[:, 1:] += r_bar / Dden
    D_bar = -(r_bar * sig[:, 1:]) / (Dden * Dden)
    sig_bar[:, :-1] += np.where(sig[:, :-1] >= dt.type(SIGMA_FLOOR), D_bar, 0.0).astype(dt)
    z_bar = sig_bar * (sig * (1.0 - sig))
    phi_bar = z_bar * s_t
    grads["log_s"] += np.asarray((z_bar * phis).sum() * s_t, dtype=dt)
    # direct phi terms
    phi_bar += (dt.type(lw.sdf) / M) * tr_mask * np.sign(phis - b_c) \
        / np.maximum(tr_cnt, 1.0).astype(dt)[:, None]
    dfs = np.where(inner >= phis - b_c,
                   np.where(e5 - dt.type(1.0) > 0, e5 * dt.type(-lw.freespace_alpha), 0.0),
                   1.0).astype(dt)
    phi_bar += (dt.type(lw.fs) / M) * fs_mask * dfs / np.maximum(fs_cnt, 1.0).astype(dt)[:, None]
    # eikonal
    u = (dt.type(-2.0 * lw.eik) / dt.type(n_eik)) * (eik_flat * diff / nrm)[:, None] * gp
    G.backward(phi_bar.reshape(-1), u.astype(dt), grads)
    if S is not None:
        us = np.concatenate([dS, -dS], axis=0) * (dt.type(2.0 * lw.smooth) / dt.type(n_sm_norm))
        S.backward(np.zeros(2 * n_smooth, dtype=dt), us.astype(dt), grads)
    # colour: sigma(MLP_c([fc, r])) backprop
    cb = c_bar.reshape(m * n, 3)
    y_bar = cb * (c_flat * (1.0 - c_flat))
    cW = [P.color_net[i][0] for i in range(3)]
    grads["color_w2"] += np.matmul(ch1.T, y_bar)
    grads["color_b2"] += y_bar.sum(axis=0)
    cm0, cm1 = (ca0 > 0).astype(dt), (ca1 > 0).astype(dt)
    for layer, row, unit in flips.get("color", ()):
        cm = cm0 if layer == 0 else cm1
        cm[row, unit] = 1 - cm[row, unit]
    a1b = np.matmul(y_bar, cW[2].T) * cm1
    grads["color_w1"] += np.matmul(ch0.T, a1b)
    grads["color_b1"] += a1b.sum(axis=0)
    a0b = np.matmul(a1b, cW[1].T) * cm0
    grads["color_w0"] += np.matmul(cin.T, a0b)
    grads["color_b0"] += a0b.sum(axis=0)
    in_bar = np.matmul(a0b, cW[0].T)
    fc_bar = in_bar[:, :fc.shape[1]]
    grads["colorgrid"] += scatter_weighted(cs.idx8, cs.w8, fc_bar.astype(dt), P.color.n_vertices)
    if P.trainable[uniq].any():
        R["pose"] = pose_backward(P, G, cs, phi_bar.reshape(-1), u.astype(dt), fc_bar.astype(dt),
                      in_bar[:, fc.shape[1]:].astype(dt), xu, lo_c, hi_c, depths, batch, uniq, inv,
                      pose_aux, m, n, grads)
    R["grads"] = grads
    R["adjoints"] = dict(phi_bar=phi_bar, u=u.reshape(m, n, 3), c_bar=c_bar)
    return R


def realised_rays(P, batch):
    """gs/renderer.py:302-309: per unique frame R = R0 @ exp_so3(nu) in the
    model dtype (gs/camera.py:68-70, exactly R0 for nu = 0), o = t, r = R dir_cam."""
    dt = P.dtype
    m = len(batch)
    uniq, inv = np.unique(batch.frame_ids, return_inverse=True)
    pose_aux = []
    R9 = np.empty((len(uniq), 9), dtype=dt)
    for j, f in enumerate(uniq):
        E, aux = exp_so3_graph(P.nu[f])
        R0c = P.R0[f].astype(dt)
        R9[j] = np.matmul(R0c, E).reshape(9)
        pose_aux.append((R0c, aux))
    T3 = np.stack([P.t[f] for f in uniq]).astype(dt)
    r_sel = np.take(R9, inv, axis=0).reshape(m, 3, 3)
    o = np.take(T3, inv, axis=0)
    r = np.matmul(r_sel, batch.dir_cam[:, :, None].astype(dt)).reshape(m, 3)
    return uniq, inv, pose_aux, o, r


def pose_grads_given(P, batch, depths, phi_bar, u, c_bar, lo_c, hi_c):
    """Component restatement: the pose gradients of a step whose sampled
    depths and loss adjoints (phi_bar (M, N), u (M, N, 3), c_bar (M, N, 3))
    are given -- the taped point / colour recomputation plus pose_backward."""
    dt = P.dtype
    m, n = depths.shape
    uniq, inv, pose_aux, o, r = realised_rays(P, batch)
    x = o.reshape(m, 1, 3) + depths[:, :, None].astype(dt) * r.reshape(m, 1, 3)
    xu = x.reshape(m * n, 3)
    xf = np.minimum(np.maximum(xu, lo_c.astype(dt)), hi_c.astype(dt))
    G = GeomPass(P, xf)
    cs = LevelSample(P.color, xf)
    fc = cs.value()
    vdir = np.broadcast_to(r.reshape(m, 1, 3), (m, n, 3)).reshape(m * n, 3)
    cin = np.concatenate([fc, vdir], axis=1)
    (ca0, ca1, ca2), _, cy = mlp_forward(P.color_net, cin)
    c_flat = sigmoid_raw(cy)
    cW = [P.color_net[i][0] for i in range(3)]
    y_bar = c_bar.reshape(m * n, 3).astype(dt) * (c_flat * (1.0 - c_flat))
    a1b = np.matmul(y_bar, cW[2].T) * (ca1 > 0)
    a0b = np.matmul(a1b, cW[1].T) * (ca0 > 0)
    in_bar = np.matmul(a0b, cW[0].T)
    grads = {nm: np.zeros_like(a) for nm, a in zip(P.names(), P.arrays())
             if nm.startswith("nu") or (nm[0] == "t" and nm[1:].isdigit())}
    inter = pose_backward(P, G, cs, np.asarray(phi_bar, dt).reshape(-1), np.asarray(u, dt).reshape(-1, 3),
                          in_bar[:, :fc.shape[1]].astype(dt), in_bar[:, fc.shape[1]:].astype(dt), xu, lo_c,
                          hi_c, depths, batch, uniq, inv, pose_aux, m, n, grads)
    return grads, inter


def pose_backward(P, G, cs, p, u, fc_bar, vdir_bar, xu, lo_c, hi_c, depths, batch, uniq, inv,
                  pose_aux, m, n, grads):
    """Gradients of the trainable poses.

    Per taped sample the cotangent of the tracked point xf collects
    (gs/renderer.py:352-365, gs/diffcore.py:893-991):
      * phi:        J_l^T zbar_l with zbar = phi_bar * g (grid_sample vjp);
      * grad phi:   the in-cell Hessian block, u against (h12, h13, h23) of
                    the per-corner contraction theta_k . g_l (_grid_dx_op vjp,
                    gs/diffcore.py:971-978; g is piecewise constant in z);
      * colour:     J_c^T fc_bar.
    The clip passes it where lo <= x <= hi (maximum/minimum ties,
    gs/diffcore.py:506-529); x = o + d r gives o_bar = sum_n x_bar and
    r_bar = sum_n d x_bar + view-direction cotangents; r = R dir_cam,
    index_select per frame, R = R0 exp_so3(nu) (gs/camera.py:68-70)."""
    dt = P.dtype
    c = P.levels[0].feat.shape[1]
    zbar = p.astype(dt)[:, None] * G.g
    xb = None
    for l, s in enumerate(G.ls):
        gl = G.g[:, l * c:(l + 1) * c]
        part = s.dx(zbar[:, l * c:(l + 1) * c])
        # per-corner contraction, as _nb_dx_forward's gc (f64 accumulator)
        gc = np.zeros((gl.shape[0], 8))
        for k in range(8):
            rows = s.lev.feat[s.idx8[:, k]]
            for j in range(c):
                gc[:, k] = gc[:, k] + (rows[:, j] * gl[:, j]).astype(np.float64)
        h12, h13, h23 = pair_hessian(gc, s.frac)
        vs2 = s.lev.voxel_size * s.lev.voxel_size
        ua = u.astype(np.float64)
        hx = np.empty_like(u)
        hx[:, 0] = (h12 * ua[:, 1] + h13 * ua[:, 2]) / vs2
        hx[:, 1] = (h12 * ua[:, 0] + h23 * ua[:, 2]) / vs2
        hx[:, 2] = (h13 * ua[:, 0] + h23 * ua[:, 1]) / vs2
        part = part + hx
        xb = part if xb is None else xb + part
    xb = xb + cs.dx(fc_bar)
    inside = (xu >= lo_c.astype(dt)) & (xu <= hi_c.astype(dt))
    xb = np.where(inside, xb, dt.type(0.0)).astype(dt).reshape(m, n, 3)
    o_bar = xb.sum(axis=1)
    r_bar = (xb * depths[:, :, None].astype(dt)).sum(axis=1) + vdir_bar.reshape(m, n, 3).sum(axis=1)
    Rsel_bar = r_bar[:, :, None] * batch.dir_cam.astype(dt)[:, None, :]
    R9_bar = np.zeros((len(uniq), 3, 3), dtype=dt)
    T3_bar = np.zeros((len(uniq), 3), dtype=dt)
    np.add.at(R9_bar, inv, Rsel_bar)
    np.add.at(T3_bar, inv, o_bar)
    for j, f in enumerate(uniq):
        if not P.trainable[f]:
            continue
        R0c, aux = pose_aux[j]
        Ebar = np.matmul(R0c.T, R9_bar[j])
        grads[f"nu{f}"] += exp_so3_adjoint(P.nu[f], aux, Ebar)
        grads[f"t{f}"] += T3_bar[j]
    return dict(xbar=xb, vdir_bar=vdir_bar.reshape(m, n, 3), o_bar=o_bar, r_bar=r_bar)


# ---------------------------------------------------------------------------
# Adam (gs/optimizer.py:38-91)


class Adam:
    """gs/optimizer.py:58-91: per-tensor step counts, f64 math, dt storage,
    non-finite gradient entries zeroed and counted."""

    def __init__(self, arrays, lrs, beta1=0.9, beta2=0.999, eps=1e-8):
        self.lrs = list(lrs)
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.m = [np.zeros_like(a) for a in arrays]
        self.v = [np.zeros_like(a) for a in arrays]
        self.t = [0] * len(arrays)
        self.skipped = 0

    def step(self, arrays, grads):
        b1, b2, eps = self.beta1, self.beta2, self.eps
        for i, (p, g) in enumerate(zip(arrays, grads)):
            self.t[i] += 1
            t = float(self.t[i])
            c1 = 1.0 - b1 ** t
            c2 = 1.0 - b2 ** t
            g64 = np.asarray(g, dtype=p.dtype).astype(np.float64).reshape(p.shape)
            bad = ~np.isfinite(g64)
            if bad.any():
                self.skipped += int(bad.sum())
                g64 = np.where(bad, 0.0, g64)
            mi = b1 * self.m[i].astype(np.float64) + (1.0 - b1) * g64
            vi = b2 * self.v[i].astype(np.float64) + (1.0 - b2) * g64 * g64
            self.m[i][...] = mi
            self.v[i][...] = vi
            p[...] = p.astype(np.float64) - self.lrs[i] * (mi / c1) / (np.sqrt(vi / c2) + eps)


class InitError(RuntimeError):
    """gs/decoders.py InitError."""


def geometric_init(P, center, radius, seed=0, max_steps=2000, tol=0.01, batch=4096,
                   lr_grid=1e-2, lr_net=1e-3, info=None):
    """gs/decoders.py:102-177: fit the geometry levels + decoder to a sphere SDF
    with Adam on uniform in-box batches plus 13 anchors; early exit on the
    held-out RMSE checks (step >= 100, every 50 steps); final 10k check."""
    dt = P.dtype
    center = np.asarray(center, dtype=np.float64)
    lo = P.lo + 0.5 * P.finest_voxel
    hi = P.hi - 0.5 * P.finest_voxel
    if np.any(center - radius < P.lo) or np.any(center + radius > P.hi):
        raise ValueError("sphere must fit inside the grid box")
    L = len(P.levels)
    names = [f"level{i}" for i in range(L)] + [f"geom_{k}{i}" for i in range(3) for k in ("w", "b")]
    arrays = [P.levels[i].feat for i in range(L)] + [P.geom[i][j] for i in range(3) for j in (0, 1)]
    opt = Adam(arrays, [lr_grid] * L + [lr_net] * 6)

    def sdf(x):
        return np.linalg.norm(x - center, axis=1, keepdims=True) - radius

    axes = np.concatenate([np.eye(3), -np.eye(3)], axis=0)
    anchors = np.clip(np.concatenate([center[None, :], center + radius * axes,
                                      center + 2.0 * radius * axes]), lo, hi)
    anchor_target = sdf(anchors).astype(dt)

    def rmse(n_pts, idx):
        pts = substream(seed, SPHERE_INIT, 10_000 + idx).uniform(lo, hi, size=(n_pts, 3))
        phi = phi_data(P, pts.astype(dt))[:, None]
        return float(np.sqrt(np.mean((phi - sdf(pts)) ** 2)))

    def anchor_err():
        phi = phi_data(P, anchors.astype(dt))[:, None]
        return float(np.max(np.abs(phi - sdf(anchors))))

    steps = 0
    for step in range(max_steps):
        pts = substream(seed, SPHERE_INIT, step).uniform(lo, hi, size=(batch, 3))
        target = sdf(pts).astype(dt)
        grads = {n: np.zeros_like(a) for n, a in zip(names, arrays)}
        for x, t, n in ((pts.astype(dt), target, batch), (anchors.astype(dt), anchor_target, len(anchors))):
            G = GeomPass(P, x)
            g = dt.type(1.0) / dt.type(n)  # mean vjp, then mul vjp: g*err + g*err
            pe = g * (G.phi - t[:, 0])
            G.backward(pe + pe, np.zeros((x.shape[0], 3), dtype=dt), grads)
        opt.step(arrays, [grads[n] for n in names])
        steps += 1
        if step >= 100 and step % 50 == 0 and rmse(2048, step) < 0.8 * tol and anchor_err() < 0.8 * tol:
            break
    final = rmse(10_000, -1)
    if info is not None:
        info["steps"] = steps
    if final >= tol:
        raise InitError(f"sphere pre-fit RMSE {final:.4f} m did not reach {tol} m within {max_steps} steps")
    return final


def train_step(P, opt, dataset, cfg, iteration):
    """gs/optimizer.py:363-373: one full iteration (draw, objective, grad, Adam)."""
    batch = draw_ray_batch(dataset, substream(cfg.seed, RAYS, iteration), cfg.batch_rays,
                           near=cfg.near, far=cfg.max_depth)
    R = train_objective(P, dataset, batch, iteration, cfg)
    names = P.names()
    opt.step(P.arrays(), [R["grads"][n] for n in names])
    if P.trainable.any() and (iteration + 1) % cfg.pose_refresh_every == 0:
        P.refresh_poses()
    return R


# ---------------------------------------------------------------------------
# marching cubes (test infrastructure): numpy restatement of the device
# kernel over the generated 256-case table (paper_2206_14735_b200/mc_table.py),
# standing in for skimage.measure.marching_cubes, which is not installed here.
# Cells in C order, triangles in table order; vertices welded per lattice
# edge in order of first use; vertex = origin-free grid coordinates scaled by
# spacing (as skimage).


def marching_cubes(vol, level=0.0, spacing=(1.0, 1.0, 1.0), table=None):
    if table is None:
        import importlib.util
        import os
        here = os.path.dirname(os.path.abspath(__file__))
        spec = importlib.util.spec_from_file_location(
            "mc_table", os.path.join(here, "..", "paper_2206_14735_b200", "mc_table.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        table = (mod.TABLE, mod.NTRI, mod.EDGE_CORNERS)
    tab, ntri, edges = table
    vol = np.asarray(vol, dtype=np.float32)
    nx, ny, nz = vol.shape
    corners = np.array([[(k >> 2) & 1, (k >> 1) & 1, k & 1] for k in range(8)])
    idx = np.zeros((nx - 1, ny - 1, nz - 1), dtype=np.int64)
    vals = []
    for k, (dx, dy, dz) in enumerate(corners):
        v = vol[dx:nx - 1 + dx, dy:ny - 1 + dy, dz:nz - 1 + dz]
        vals.append(v)
        idx |= (v < np.float32(level)).astype(np.int64) << k
    cells = np.flatnonzero(ntri[idx.reshape(-1)] > 0)
    verts, keys = [], []
    for c in cells:
        i, r = divmod(int(c), (ny - 1) * (nz - 1))
        j, k = divmod(r, nz - 1)
        m = idx[i, j, k]
        for q in range(3 * int(ntri[m])):
            e = tab[m, q]
            a, b = edges[e]
            va = float(vals[a][i, j, k])
            vb = float(vals[b][i, j, k])
            t = (float(np.float32(level)) - va) / (vb - va)
            pa = np.array([i, j, k]) + corners[a]
            pb = np.array([i, j, k]) + corners[b]
            verts.append([(pa[d] + t * (pb[d] - pa[d])) * spacing[d] for d in range(3)])
            ax = int(np.flatnonzero(pb - pa)[0])
            keys.append(((int(pa[0]) * ny + int(pa[1])) * nz + int(pa[2])) * 3 + ax)
    verts = np.asarray(verts, dtype=np.float64).reshape(-1, 3)
    # welded: one vertex per lattice edge, in order of first use (what the
    # device path returns; scikit-image's meshes are welded too)
    keys = np.asarray(keys, dtype=np.int64)
    if len(keys) == 0:
        return verts, np.zeros((0, 3), dtype=np.int64)
    _, first, inv = np.unique(keys, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    return verts[first[order]], rank[inv.reshape(-1)].reshape(-1, 3).astype(np.int64)
