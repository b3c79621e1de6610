"""Device step engine: owns the workspace and launches ``gsb_train_step``.

One engine per (model, dataset).  A step is one C-ABI call that enqueues the
whole objective + backward on the caller's CUDA stream (ray setup and
stratification, three importance rounds, taped forward, rendering/losses,
fused backward with grid scatter and MLP gradient reduction); nothing in it
synchronises with the host.  The per-iteration host inputs are only what
the reference draws with numpy's integer/normal samplers: the ray ids
(gs/sampler.py:70), the smoothness point set (gs/renderer.py:243-276) and
the PCG64 states of the uniform streams, which the device regenerates.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import seeds
from .camera import pixel_rays, ray_to_z_scale


@dataclass
class HostDraws:
    """Everything one iteration needs from the host RNG."""

    iteration: int
    ray_ids: np.ndarray          # (M,) int64 flat ids into F*H*W
    smooth: np.ndarray | None    # (2S, 3) model dtype: x then x+eps (explicit points)
    rng_stratify: object
    rng_importance: list
    # raw smoothness draws (pick, jitter, normals) turned into points on the
    # device by gsb_smooth_points; exclusive with `smooth`
    smooth_raw: tuple | None = None
    smooth_delta: float = 0.004

    @property
    def n_smooth(self):
        if self.smooth is not None:
            return self.smooth.shape[0] // 2
        return 0 if self.smooth_raw is None else len(self.smooth_raw[0])

    @property
    def h2d_bytes(self):
        b = self.ray_ids.nbytes
        if self.smooth is not None:
            b += self.smooth.nbytes
        if self.smooth_raw is not None:
            b += sum(a.nbytes for a in self.smooth_raw)
        return b


def draw_smooth_points(model, dataset, count, truncation, delta, rng):
    """gs/renderer.py:243-276, same RNG calls in the same order.

    The k-th valid pixel comes from the dataset's per-row prefix count
    instead of the full np.nonzero list (same pixel, same order)."""
    n_valid = dataset.n_valid
    if n_valid == 0:
        return None
    pick = rng.integers(0, n_valid, size=count)
    f, v, u = dataset.valid_pixel(pick)
    pixels = np.stack([u, v], axis=1).astype(np.float64)
    intr = dataset.intrinsics
    d_cam = pixel_rays(intr, pixels)
    scale = ray_to_z_scale(intr, pixels)
    depth_ray = dataset.depth_at(f, v, u) * scale + rng.uniform(-truncation, truncation, size=count)
    mats = model.pose_matrices()[f]
    dirs = np.einsum("nij,nj->ni", mats[:, :3, :3], d_cam)
    x = mats[:, :3, 3] + depth_ray[:, None] * dirs
    x = model.grid.clamp_points(x)
    lo, hi = model.grid.clamp_box()
    eps_dir = rng.normal(size=(count, 8, 3))
    eps_dir /= np.linalg.norm(eps_dir, axis=2, keepdims=True)
    cand = x[:, None, :] + delta * eps_dir
    ok = ((cand >= lo) & (cand <= hi)).all(axis=2)
    first = np.argmax(ok, axis=1)
    xe = cand[np.arange(count), first]
    xe = np.clip(xe, lo, hi)
    return x, xe


def smooth_raw_draws(dataset, count, truncation, rng):
    """The RNG calls of draw_smooth_points (gs/renderer.py:253-268), in order:
    integers (valid pixel), uniform (range jitter), normal (8 directions)."""
    n_valid = dataset.n_valid
    if n_valid == 0:
        return None
    pick = rng.integers(0, n_valid, size=count)
    jitter = rng.uniform(-truncation, truncation, size=count)
    normals = rng.normal(size=(count, 8, 3))
    return (np.ascontiguousarray(pick, dtype=np.int64), np.ascontiguousarray(jitter),
            np.ascontiguousarray(normals))


def host_draws(model, dataset, cfg, iteration, ray_ids=None, smooth_override=None,
               device_smooth=True):
    """Host-side randomness of iteration `iteration` (gs/optimizer.py:363-366,
    gs/renderer.py:320-336, 416-423).  With ``device_smooth`` the smoothness
    points are left as raw draws for gsb_smooth_points."""
    lw = cfg.weights
    if ray_ids is None:
        intr = dataset.intrinsics
        n = len(dataset) * intr.height * intr.width
        ray_ids = seeds.substream(cfg.seed, seeds.RAYS, iteration).integers(
            0, n, size=cfg.batch_rays)
    smooth = raw = None
    if lw.smooth != 0.0:
        rng = seeds.substream(cfg.seed, seeds.SMOOTH, iteration)
        if smooth_override is not None:
            pts = smooth_override
        elif device_smooth:
            pts = None
            raw = smooth_raw_draws(dataset, lw.smooth_count, lw.truncation, rng)
        else:
            pts = draw_smooth_points(model, dataset, lw.smooth_count, lw.truncation,
                                     lw.smooth_delta, rng)
        if pts is not None:
            smooth = np.concatenate([pts[0], pts[1]], axis=0).astype(model.dtype)
    rs = _lib.Pcg64.from_generator(seeds.substream(cfg.seed, seeds.STRATIFY, iteration))
    ri = [_lib.Pcg64.from_generator(seeds.substream(cfg.seed, seeds.IMPORTANCE, iteration, r))
          for r in range(cfg.importance_rounds)]
    return HostDraws(iteration, np.asarray(ray_ids, dtype=np.int64), smooth, rs, ri, raw,
                     float(lw.smooth_delta))


def model_struct(m):
    """gsb_model_t of a ModelState (arena pointers, level descriptors)."""
    a = m.arena
    ms = _lib.Model()
    ms.precision = 0 if a.dtype == np.float32 else 1
    if len(m.grid.levels) > _lib.MAX_LEVELS:
        raise ValueError("too many grid levels")
    ms.n_levels = len(m.grid.levels)

    def lev(gl):
        L = _lib.Level()
        L.nx, L.ny, L.nz = gl.geom.dims
        L.channels = gl.width
        L.ox, L.oy, L.oz = (float(x) for x in gl.geom.origin)
        L.voxel = gl.geom.voxel_size
        L.offset = gl.features.offset
        return L

    for i, gl in enumerate(m.grid.levels):
        ms.levels[i] = lev(gl)
    ms.color = lev(m.grid.color)
    ms.mlp_offset = a["geom_w0"].offset
    ms.log_s_offset = m.log_s.offset
    ms.n_params = a.n
    lo, hi = m.grid.clamp_box()
    for i in range(3):
        ms.lo_c[i] = float(lo[i])
        ms.hi_c[i] = float(hi[i])
    ms.params = a.params.data_ptr()
    ms.grads = a.grads.data_ptr()
    return ms


class StepEngine:
    """Launches training steps for one model on one device dataset."""

    def __init__(self, model, dataset):
        import torch
        self.torch = torch
        self.model = model
        self.dataset = dataset
        self.device = model.arena.params.device
        self.lib = _lib.lib()
        self._ws = {}
        self.col, self.dep, _ = dataset.device_tensors(self.device, model.dtype)
        self.mstruct = self._model_struct()
        # deterministic scatter mode (validation): bit-reproducible grid gradients
        self.deterministic = False
        self._init_poses()
        self.dstruct = self._dataset_struct()

    # ---- poses
    def _init_poses(self):
        """Ray pose table (F, 12) from the MODEL's poses: R0c exp_so3(nu) and t in
        the model dtype (gs/renderer.py:218-225), and the f64 PoseParam.matrix
        table for the smoothness points.  Frozen poses: computed once here.
        Trainable poses (pose refinement): gsb_pose_table refreshes both from
        the arena every step (``pose_tables``)."""
        torch = self.torch
        model = self.model
        dt = model.dtype
        F = len(model.poses)
        R0 = np.stack([p.R0 for p in model.poses]).reshape(F, 9)
        tab = np.zeros((F, 12))
        tab[:, :9] = R0.astype(dt).astype(np.float64)
        tab[:, 9:] = np.stack([np.asarray(p.t_data(), dtype=dt) for p in model.poses]).astype(np.float64)
        mats = model.pose_matrices()
        tab64 = np.concatenate([mats[:, :3, :3].reshape(-1, 9), mats[:, :3, 3]], axis=1)
        self.pose_tab = torch.from_numpy(np.ascontiguousarray(tab)).to(self.device)
        self.pose_tab64 = torch.from_numpy(np.ascontiguousarray(tab64)).to(self.device)
        self.refine = model.refine_poses
        if not self.refine:
            return
        off = lambda p, q: (q.offset if p.trainable else -1)
        self._pose_dev = dict(
            R0=torch.from_numpy(np.ascontiguousarray(R0)).to(self.device),
            nu_off=torch.tensor([off(p, p.nu) for p in model.poses], dtype=torch.int64, device=self.device),
            t_off=torch.tensor([off(p, p.t) for p in model.poses], dtype=torch.int64, device=self.device),
            t_fixed=self.pose_tab[:, 9:].contiguous())
        self._pose_ver = tuple(p.version for p in model.poses)
        d = self._pose_dev
        self.pstruct = _lib.Pose(F, d["R0"].data_ptr(), d["nu_off"].data_ptr(), d["t_off"].data_ptr(),
                                 d["t_fixed"].data_ptr())

    def pose_tables(self, stream=None):
        """Refresh the pose tables from the current R0 / nu / t (pose refinement)."""
        if self.refine:
            ver = tuple(p.version for p in self.model.poses)
            if ver != self._pose_ver:  # a PoseParam.refresh folded nu into R0 on the host
                R0 = np.stack([p.R0 for p in self.model.poses]).reshape(-1, 9)
                self._pose_dev["R0"].copy_(self.torch.from_numpy(np.ascontiguousarray(R0)))
                self._pose_ver = ver
            _lib.check(self.lib.gsb_pose_table(C.byref(self.mstruct), C.byref(self.pstruct),
                                               self.pose_tab.data_ptr(), self.pose_tab64.data_ptr(),
                                               _lib.stream_handle(stream)), "gsb_pose_table")


    # ---- ABI structs
    def _model_struct(self):
        return model_struct(self.model)

    def _dataset_struct(self):
        ds = self.dataset
        intr = ds.intrinsics
        d = _lib.Dataset()
        d.colors = self.col.data_ptr()
        d.depth_mm = self.dep.data_ptr()
        d.n_frames = len(ds)
        d.height, d.width = intr.height, intr.width
        d.fx, d.fy, d.cx, d.cy = (float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy))
        d.poses = self.pose_tab.data_ptr()
        return d

    # ---- workspace
    def workspace(self, M, Nc, R, A, S):
        key = (M, Nc, R, A, S)
        if key not in self._ws:
            torch = self.torch
            nbytes = C.c_size_t(0)
            _lib.check(self.lib.gsb_step_workspace_size(C.byref(self.mstruct), M, Nc, R, A, S,
                                                        C.byref(nbytes)), "workspace size")
            offs = [C.c_int64(0) for _ in range(5)]
            ld = C.c_int32(0)
            _lib.check(self.lib.gsb_step_workspace_layout(
                C.byref(self.mstruct), M, Nc, R, A, S, *[C.byref(o) for o in offs],
                C.byref(ld)), "workspace layout")
            buf = torch.zeros(int(nbytes.value), dtype=torch.uint8, device=self.device)
            N = Nc + R * A
            tdt = torch.float32 if self.model.dtype == np.float32 else torch.float64
            esz = 4 if tdt == torch.float32 else 8
            po, co, so, do, wo = (o.value for o in offs)
            views = dict(
                buf=buf, ld=ld.value, N=N,
                parts=buf[po:po + 8 * _lib.N_PARTS].view(torch.float64),
                counts=buf[co:co + 8 * 4].view(torch.int64),
                status=buf[so:so + 4 * _lib.N_STATUS].view(torch.int32),
                depths=buf[do:do + 8 * M * ld.value].view(torch.float64).view(M, ld.value),
                weights=buf[wo:wo + esz * M * N].view(tdt).view(M, N),
            )
            reg = (C.c_int64 * len(_lib.REGIONS))()
            _lib.check(self.lib.gsb_step_workspace_regions(C.byref(self.mstruct), M, Nc, R, A, S,
                                                           reg), "workspace regions")
            views["regions"] = dict(zip(_lib.REGIONS, list(reg)))
            NS = M * N + 2 * S
            sizes = dict(phi=(NS,), gphi=(NS, 3), color=(M * N, 3), pbar=(NS,), ubar=(NS, 3),
                         cbar=(M * N, 3), ray_o=(M, 3), ray_r=(M, 3))
            for k, shp in sizes.items():
                o = views["regions"][k]
                n = int(np.prod(shp))
                views[k] = buf[o:o + esz * n].view(tdt).view(*shp)
            o = views["regions"]["ray_far"]
            views["ray_far"] = buf[o:o + 8 * M].view(torch.float64)
            self._ws[key] = views
        return self._ws[key]

    # ---- one step
    def step_struct(self, cfg, draws, ray_ids_dev, smooth_dev, ws, ray_base=0, m_global=None,
                    smooth_global=None, phases=3, exact=False):
        st = _lib.Step()
        st.ray_ids = ray_ids_dev.data_ptr()
        st.n_rays = int(ray_ids_dev.numel())
        st.ray_base = int(ray_base)
        st.m_global = float(m_global if m_global is not None else st.n_rays)
        st.n_coarse = cfg.coarse_samples
        st.n_rounds = cfg.importance_rounds
        st.n_add = cfg.importance_add
        st.has_fixed_far = 1 if cfg.fixed_far is not None else 0
        st.near = float(cfg.near)
        st.max_depth = float(cfg.max_depth)
        st.fixed_far = float(cfg.fixed_far) if cfg.fixed_far is not None else 0.0
        st.rng_stratify = draws.rng_stratify
        for r, g in enumerate(draws.rng_importance):
            st.rng_importance[r] = g
        lw = cfg.weights
        st.w_rgb, st.w_depth, st.w_sdf = float(lw.rgb), float(lw.depth), float(lw.sdf)
        st.w_fs, st.w_eik, st.w_smooth = float(lw.fs), float(lw.eik), float(lw.smooth)
        st.truncation = float(lw.truncation)
        st.fs_alpha = float(lw.freespace_alpha)
        if smooth_dev is not None:
            st.smooth_pts = smooth_dev.data_ptr()
            st.n_smooth = int(smooth_dev.shape[0] // 2)
        else:
            st.smooth_pts = None
            st.n_smooth = 0
        st.smooth_global = float(smooth_global if smooth_global is not None else max(st.n_smooth, 1))
        st.exact_gather = 1 if exact else 0
        st.phases = phases
        st.workspace = ws["buf"].data_ptr()
        st.workspace_bytes = ws["buf"].numel()
        return st

    def _smooth_tables(self):
        """(F, 12) f64 pose_matrices() rows and the (F*H) valid-pixel row
        prefix counts, device-resident (the pose table is the engine's, kept
        current by ``pose_tables`` under pose refinement)."""
        if not hasattr(self, "_smooth_tab"):
            torch = self.torch
            ds = self.dataset
            mask = (ds.depths_mm > 0).reshape(-1, ds.depths_mm.shape[-1])
            # per-row compaction: row r's valid columns, in order, come first
            if mask.shape[1] >= 1 << 15:
                raise ValueError("image width exceeds the int16 valid-column index")
            valid_u = np.argsort(~mask, axis=1, kind="stable").astype(np.int16)
            self._smooth_tab = (
                self.pose_tab64,
                torch.from_numpy(np.ascontiguousarray(ds._rows(), dtype=np.int64)).to(self.device),
                torch.from_numpy(np.ascontiguousarray(valid_u)).to(self.device))
        return self._smooth_tab

    def upload_smooth_raw(self, raw):
        """Raw smoothness draws -> one device buffer [pick | jitter | normals]."""
        pick, jitter, normals = raw
        packed = np.concatenate([pick.view(np.float64), jitter, normals.reshape(-1)])
        return self.torch.from_numpy(packed).pin_memory().to(self.device, non_blocking=True)

    def smooth_points_dev(self, raw_dev, count, delta, stream=None):
        """gsb_smooth_points on device-resident raw draws -> (2S, 3) points."""
        poses, row_cum, valid_u = self._smooth_tables()
        out = self.torch.empty((2 * count, 3), dtype=self.model.arena.params.dtype,
                               device=self.device)
        base = raw_dev.data_ptr()
        _lib.check(self.lib.gsb_smooth_points(
            C.byref(self.mstruct), C.byref(self.dstruct), poses.data_ptr(), row_cum.data_ptr(),
            valid_u.data_ptr(), base, base + 8 * count, base + 16 * count, count, float(delta),
            out.data_ptr(), _lib.stream_handle(stream)), "gsb_smooth_points")
        return out

    def smooth_points(self, raw, delta, stream=None):
        """gsb_smooth_points: raw host draws -> (2S, 3) device points."""
        return self.smooth_points_dev(self.upload_smooth_raw(raw), len(raw[0]), delta, stream)

    def upload(self, draws, stream=None):
        """Host draws -> device inputs.  On the default path the host-to-device
        copies go on a copy stream the step's stream then waits for, so the
        copies of step k+1 overlap step k's kernels (the caller runs ahead)."""
        torch = self.torch
        self.pose_tables(stream)
        # (large batches only: at 1024 rays the step is host-bound and the
        # extra stream bookkeeping costs more than the copy it hides)
        side = (stream is None and self.device.type == "cuda" and len(draws.ray_ids) >= 4096
                and os.environ.get("GSB_COPY_STREAM", "1") != "0")
        cur = torch.cuda.current_stream(self.device) if side else None
        if side:
            if getattr(self, "_copy_stream", None) is None:
                self._copy_stream = torch.cuda.Stream(device=self.device)
            ctx = torch.cuda.stream(self._copy_stream)
        else:
            ctx = contextlib.nullcontext()
        raw_dev = sm = None
        with ctx:
            ids = torch.from_numpy(draws.ray_ids).pin_memory().to(self.device, non_blocking=True)
            if draws.smooth is not None:
                sm = torch.from_numpy(np.ascontiguousarray(draws.smooth)).pin_memory().to(
                    self.device, non_blocking=True)
            elif draws.smooth_raw is not None:
                raw_dev = self.upload_smooth_raw(draws.smooth_raw)
        if side:
            cur.wait_stream(self._copy_stream)
            for t in (ids, sm, raw_dev):
                if t is not None:
                    t.record_stream(cur)
        if raw_dev is not None:
            sm = self.smooth_points_dev(raw_dev, len(draws.smooth_raw[0]), draws.smooth_delta, stream)
        return ids, sm

    def launch(self, cfg, draws, ray_ids_dev, smooth_dev, stream=None, fresh=True, **kw):
        """Enqueue one objective + backward; returns the workspace views.
        ``fresh=False`` continues a step in the same workspace (phase 2 after
        a phase-1 launch and the count all-reduce): status words are kept."""
        M = int(ray_ids_dev.numel())
        S = 0 if smooth_dev is None else int(smooth_dev.shape[0] // 2)
        ws = self.workspace(M, cfg.coarse_samples, cfg.importance_rounds, cfg.importance_add, S)
        if kw.get("phases", 3) & 12 != 8:  # part B continues part A's gradients
            self.model.arena.zero_grads()
        if fresh:
            ws["status"].zero_()
        st = self.step_struct(cfg, draws, ray_ids_dev, smooth_dev, ws, **kw)
        phases = kw.get("phases", 3)
        if self.refine:
            buf = self._pose_scratch(cfg, M)
            st.pose_work, st.pose_work_bytes = buf.data_ptr(), buf.numel()
        if self.deterministic:
            buf = self._det_scratch(cfg, M, S)
            st.det_work, st.det_work_bytes = buf.data_ptr(), buf.numel()
        if fresh and phases & 1:
            self.pose_tables(stream)
        _lib.check(self.lib.gsb_train_step(C.byref(self.mstruct), C.byref(self.dstruct),
                                           C.byref(st), _lib.stream_handle(stream)),
                   "gsb_train_step")
        if phases & 2:
            self.model.arena.grads_clean = False
            if self.refine and (phases & 12) != 4:  # after the whole backward (or its part B)
                self._pose_grad(cfg, st, M, stream)
        return ws

    def _det_scratch(self, cfg, M, S):
        key = ("det", M, cfg.coarse_samples, cfg.importance_rounds, cfg.importance_add, S)
        if key not in self._ws:
            nbytes = C.c_size_t(0)
            _lib.check(self.lib.gsb_det_scratch_size(C.byref(self.mstruct), M, cfg.coarse_samples,
                                                     cfg.importance_rounds, cfg.importance_add, S,
                                                     C.byref(nbytes)), "det scratch size")
            self._ws[key] = self.torch.empty(max(int(nbytes.value), 1), dtype=self.torch.uint8,
                                             device=self.device)
        return self._ws[key]

    def _pose_scratch(self, cfg, M):
        key = ("pose", M, cfg.coarse_samples, cfg.importance_rounds, cfg.importance_add)
        if key not in self._ws:
            nbytes = C.c_size_t(0)
            _lib.check(self.lib.gsb_pose_scratch_size(C.byref(self.mstruct), M, cfg.coarse_samples,
                                                      cfg.importance_rounds, cfg.importance_add,
                                                      C.byref(nbytes)), "pose scratch size")
            self._ws[key] = self.torch.empty(max(int(nbytes.value), 1), dtype=self.torch.uint8,
                                             device=self.device)
        return self._ws[key]

    def _pose_grad(self, cfg, st, M, stream):
        buf = self._pose_scratch(cfg, M)
        _lib.check(self.lib.gsb_pose_grad(C.byref(self.mstruct), C.byref(self.dstruct), C.byref(st),
                                          C.byref(self.pstruct), buf.data_ptr(), buf.numel(),
                                          _lib.stream_handle(stream)), "gsb_pose_grad")
