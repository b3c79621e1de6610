"""Adam, configuration, model construction, checkpoints and the training
loop (gs/optimizer.py), over the device parameter arena."""

from __future__ import annotations

import ctypes as C
import logging
import os
from dataclasses import asdict, dataclass, field

import numpy as np

from . import _lib
from . import checkpoint as ckpt
from . import model as mdl
from . import sampler, seeds
from .data import Dataset
from .renderer import LossWeights, engine_for, parts_from, check_status
from .engine import host_draws

__all__ = ["Adam", "TrainConfig", "DivergenceError", "train", "build_model", "make_optimizer",
           "save_model", "load_model", "Trainer", "CSV_HEADER"]

log = logging.getLogger("gridsurf_b200")
MAX_ADAM_SEGMENTS = 32  # GSB_ADAM_MAX_SEGS (csrc/gsb_kernels.cuh)


class DivergenceError(RuntimeError):
    pass


class Adam:
    """Bias-corrected Adam with per-parameter learning rates (gs/optimizer.py:58-91).

    One fused launch over the whole arena: float64 register math, storage
    in the model dtype, non-finite gradient entries zeroed and counted, the
    gradient arena cleared on the way out."""

    def __init__(self, params, lrs, beta1=0.9, beta2=0.999, eps=1e-8):
        import torch
        if len(params) != len(lrs):
            raise ValueError("one learning rate per parameter")
        self.params = list(params)
        if not self.params:
            raise ValueError("no parameters")
        self.arena = self.params[0].arena
        if any(p.arena is not self.arena for p in self.params):
            raise ValueError("all parameters must live in one arena")
        self.lrs = [float(l) for l in lrs]
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.m_arena = torch.zeros_like(self.arena.params)
        self.v_arena = torch.zeros_like(self.arena.params)
        self.t = [0] * len(self.params)
        self.status = torch.zeros(_lib.N_STATUS, dtype=torch.int32, device=self.arena.device)
        self._skipped_seen = 0

    @property
    def m(self):
        return [self.m_arena[p.offset:p.offset + p.size].view(p.shape) for p in self.params]

    @property
    def v(self):
        return [self.v_arena[p.offset:p.offset + p.size].view(p.shape) for p in self.params]

    @property
    def skipped(self):
        return int(self.status[_lib.ST_ADAM_BAD].item())

    def _segments(self):
        """(begin, lr) runs over the arena.  Every parameter starts on a
        4-element boundary whenever its learning-rate group can differ from
        its predecessor's, so a 16-byte vector never straddles two rates;
        arena ranges no parameter of this optimizer covers get lr 0."""
        A = mdl.ParamArena.ALIGN
        up = lambda x: (x + A - 1) // A * A
        spans = sorted((p.offset, p.offset + p.size, lr) for p, lr in zip(self.params, self.lrs))
        begins, lrs = [0], [spans[0][2] if spans[0][0] < A else 0.0]
        pos = 0
        for b, e, lr in spans:
            if b - up(pos) >= A and lrs[-1] != 0.0:
                begins.append(up(pos))
                lrs.append(0.0)
            if lrs[-1] != lr:
                if b % A:
                    raise ValueError("learning-rate boundary inside a vector group")
                begins.append(b)
                lrs.append(lr)
            pos = e
        if self.arena.n - up(pos) >= A and lrs[-1] != 0.0:
            begins.append(up(pos))
            lrs.append(0.0)
        return begins, lrs

    def _segments_in(self, lo, hi):
        """The learning-rate runs of arena range [lo, hi), relative to lo."""
        b, l = self._segments()
        begins, lrs = [0], [0.0]
        for x, lr in zip(b, l):
            if x <= lo:
                lrs[0] = lr
            elif x < hi:
                begins.append(x - lo)
                lrs.append(lr)
        return begins, lrs

    def _segments_owned(self, owned):
        """Runs over the whole arena where only the ``owned`` [lo, hi) ranges
        keep their learning rates; the rest is marked not-owned (lr -1: the
        kernel only zeroes those gradients)."""
        b, l = self._segments()
        cuts = sorted({0, self.arena.n} | set(b) | {x for r in owned for x in r})
        begins, lrs = [], []
        for x, y in zip(cuts[:-1], cuts[1:]):
            if x == y:
                continue
            lr = l[max(i for i, s in enumerate(b) if s <= x)]
            if not any(lo <= x and y <= hi for lo, hi in owned):
                lr = -1.0
            if lrs and lrs[-1] == lr:
                continue
            begins.append(x)
            lrs.append(lr)
        return begins, lrs

    def _launch(self, guard=None, guard_threshold=0.0, stream=None, lo=0, hi=None,
                guard_status=None, owned=None):
        """One fused update of arena range [lo, hi) (default: all of it), or
        of the whole arena where only the ``owned`` ranges are updated and the
        other gradients zeroed (a data-parallel rank's shards, parallel.py).
        ``guard`` / ``guard_status`` (the step's parts and status words) skip
        the update where the reference raises before its Adam step."""
        ts = set(self.t)
        if len(ts) != 1:
            raise NotImplementedError("per-tensor step counts must agree for the fused update")
        t = float(self.t[0])
        c1 = 1.0 - self.beta1 ** t  # host pow == numba's libm pow (bit-exact)
        c2 = 1.0 - self.beta2 ** t
        a = self.arena
        hi = a.n if hi is None else int(hi)
        lo = int(lo)
        if lo % mdl.ParamArena.ALIGN or (hi - lo) % mdl.ParamArena.ALIGN or not 0 <= lo <= hi <= a.n:
            raise ValueError("Adam range must be 16-byte aligned inside the arena")
        if owned is not None:
            if (lo, hi) != (0, a.n):
                raise ValueError("owned ranges are given over the whole arena")
            if any(x % mdl.ParamArena.ALIGN for r in owned for x in r):
                raise ValueError("owned ranges must be 16-byte aligned")
            b, l = self._segments_owned(owned)
        else:
            b, l = self._segments_in(lo, hi) if (lo, hi) != (0, a.n) else self._segments()
        if len(b) > MAX_ADAM_SEGMENTS:
            raise ValueError("too many learning-rate segments")
        B = (C.c_int64 * len(b))(*b)
        Lr = (C.c_double * len(l))(*l)
        esz = a.params.element_size()
        _lib.check(_lib.lib().gsb_adam_step(
            0 if a.dtype == np.float32 else 1, a.params.data_ptr() + lo * esz, a.grads.data_ptr() + lo * esz,
            self.m_arena.data_ptr() + lo * esz, self.v_arena.data_ptr() + lo * esz, hi - lo, B, Lr, len(b),
            self.beta1, self.beta2, self.eps, c1, c2,
            None if guard is None else guard.data_ptr(), float(guard_threshold),
            None if guard_status is None else guard_status.data_ptr(),
            self.status.data_ptr(), _lib.stream_handle(stream)), "gsb_adam_step")
        a.grads_clean = True
        a.generation = getattr(a, "generation", 0) + 1

    def step(self, grads, guard=None, guard_threshold=0.0):
        """gs/optimizer.py:77-91.  `grads` are normally the arena views from
        renderer.grad(); any other arrays are copied into the arena first."""
        import torch
        a = self.arena
        fused = len(grads) == len(self.params) and all(
            isinstance(g, torch.Tensor) and g.data_ptr() == p.grad.data_ptr()
            for g, p in zip(grads, self.params))
        if not fused:
            a.grads.zero_()
            for p, g in zip(self.params, grads):
                gt = g if isinstance(g, torch.Tensor) else torch.as_tensor(np.asarray(g))
                p.grad.copy_(gt.reshape(p.shape).to(device=a.device, dtype=a.grads.dtype))
        self.t = [t + 1 for t in self.t]
        self._launch(guard=guard, guard_threshold=guard_threshold)


class AdamOverlap:
    """Step k's colour-grid update on a side stream, under step k+1's
    sampling phase.

    The sampling phase (ray setup, coarse + importance SDF evaluations and
    importance rounds, gs/renderer.py:302-346) reads the geometry grids, the
    geometry MLP and log_s, never the colour grid; the colour grid is next
    read by the taped forward of phase 2.  So each step's Adam is split into
    the colour-grid range [lo, hi) of the arena, launched on `side` once the
    step's gradients are final, and the rest, on the step's own stream; the
    next step's phase 2 waits for the colour range.  Every element is still
    updated exactly once per step, from the same gradients, with the same
    guard (a device snapshot of the step's parts and status words, since the
    next phase 1 resets them): results are bit-identical to the fused launch.
    Single-GPU only (the data-parallel path shards Adam instead).  Opt-in: on
    one B200 at config 2 the concurrent HBM stream slowed the latency-bound
    sampling and taped kernels by more than it hid (1.412 vs 1.384 ms)."""

    def __init__(self, opt, model):
        import torch
        self.torch = torch
        self.opt = opt
        cg = model.arena["colorgrid"]
        A = mdl.ParamArena.ALIGN
        self.lo = cg.offset // A * A
        self.hi = min(-(-(cg.offset + cg.size) // A) * A, opt.arena.n)
        dev = opt.arena.device
        self.side = torch.cuda.Stream(device=dev)
        self.snap_parts = torch.zeros(_lib.N_PARTS, dtype=torch.float64, device=dev)
        self.snap_status = torch.zeros(_lib.N_STATUS, dtype=torch.int32, device=dev)
        self.ev_grads = torch.cuda.Event()
        self.ev_done = torch.cuda.Event()
        self.pending = False

    def wait_colour(self, stream=None):
        """Before a phase 2: the previous step's colour-grid update is done."""
        if self.pending:
            (stream or self.torch.cuda.current_stream()).wait_event(self.ev_done)

    def step(self, ws, guard_threshold, stream=None):
        """Step k's Adam, after its phase 2 (ws: its workspace views)."""
        torch = self.torch
        cur = stream or torch.cuda.current_stream()
        opt = self.opt
        with torch.cuda.stream(cur):
            self.wait_colour(cur)  # the snapshot buffers are reused
            self.snap_parts.copy_(ws["parts"])
            self.snap_status.copy_(ws["status"])
        opt.t = [t + 1 for t in opt.t]
        kw = dict(guard=self.snap_parts, guard_threshold=guard_threshold, guard_status=self.snap_status)
        if self.lo > 0:
            opt._launch(lo=0, hi=self.lo, stream=cur, **kw)
        if self.hi < opt.arena.n:
            opt._launch(lo=self.hi, hi=opt.arena.n, stream=cur, **kw)
        self.ev_grads.record(cur)
        self.side.wait_event(self.ev_grads)
        opt._launch(lo=self.lo, hi=self.hi, stream=self.side, **kw)
        self.ev_done.record(self.side)
        self.pending = True

    def drain(self, stream=None):
        """Make the current stream wait for the last colour-grid update."""
        self.wait_colour(stream)
        self.pending = False


@dataclass
class TrainConfig:
    """All knobs of a reconstruction run (gs/optimizer.py:94-143)."""

    iterations: int = 10000
    batch_rays: int = 6144
    coarse_samples: int = sampler.N_COARSE
    importance_rounds: int = sampler.N_IMPORTANCE_ROUNDS
    importance_add: int = sampler.N_IMPORTANCE_ADD
    seed: int = 0
    precision: str = "double"
    refine_poses: bool = False
    freeze_first_pose: bool = True
    lr_grids: float = 1e-2
    lr_decoders: float = 1e-3
    lr_poses: float = 5e-4
    pose_refresh_every: int = 100
    checkpoint_every: int = 1000
    near: float = 0.01
    max_depth: float = 8.0
    bounds: tuple | None = None
    bounds_padding: float = 0.5
    voxel_sizes: tuple = mdl.DEFAULT_GEOM_VOXELS
    color_voxel: float | None = None
    geom_feat_dim: int = mdl.GEOM_FEATURE_WIDTH
    color_feat_dim: int = mdl.COLOR_FEATURE_WIDTH
    init_steps: int = 2000
    init_tol: float = 0.01
    sphere_radius_scale: float = 0.5
    divergence_threshold: float = 1e6
    fixed_far: float | None = None
    weights: LossWeights = field(default_factory=LossWeights)

    def __post_init__(self):
        if self.iterations < 0:
            raise ValueError("iterations must be >= 0")
        if self.precision not in ("double", "single"):
            raise ValueError("precision must be 'double' or 'single'")

    @property
    def dtype(self):
        return np.float64 if self.precision == "double" else np.float32

    def echo(self):
        d = asdict(self)
        d["weights"] = asdict(self.weights)
        for k, v in list(d.items()):
            if isinstance(v, tuple):
                d[k] = list(v)
        return d


def _device(device=None):
    import torch
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 path needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def derive_bounds(dataset, cfg):
    """gs/optimizer.py:146-178 (model.derive_bounds)."""
    return mdl.derive_bounds(Dataset.wrap(dataset), cfg)


def build_model(dataset, cfg, initial_poses=None, skip_init=False, device=None):
    """gs/optimizer.py:181-214: grids, decoders, sharpness, poses."""
    dataset = Dataset.wrap(dataset)
    lo, hi = mdl.derive_bounds(dataset, cfg)
    poses = dataset.poses if initial_poses is None else np.asarray(initial_poses)
    trainable = [cfg.refine_poses and not (cfg.freeze_first_pose and i == 0) for i in range(len(poses))]
    model = mdl.allocate_model(lo, hi, cfg.voxel_sizes, cfg.geom_feat_dim, cfg.color_voxel,
                               cfg.color_feat_dim, poses, cfg.dtype, _device(device), trainable=trainable)
    mdl.init_parameters(model, cfg.seed, cfg.weights.truncation)
    if not skip_init:
        from .geometry import geometric_init
        center = 0.5 * (lo + hi)
        radius = cfg.sphere_radius_scale * float(np.min(hi - lo))
        rmse = geometric_init(model, center, radius, seed=cfg.seed, max_steps=cfg.init_steps,
                              tol=cfg.init_tol)
        log.info("sphere pre-fit RMSE %.4f m", rmse)
    return model


def _lr_list(model, cfg):
    """gs/optimizer.py:394-399."""
    return ([cfg.lr_grids] * len(model.grid_params())
            + [cfg.lr_decoders] * len(model.decoder_params())
            + [cfg.lr_poses] * len(model.pose_params()))


def make_optimizer(model, cfg):
    """gs/optimizer.py:229-236."""
    return Adam(model.parameters(), _lr_list(model, cfg))


# ---------------------------------------------------------------------------
# checkpoints (GSURFCKPT1, gs/optimizer.py:243-325)


def save_model(path, model, cfg, iteration, opt=None):
    if model.arena.params.is_cuda:  # all streams, the side-stream Adam included
        import torch
        torch.cuda.synchronize(model.arena.params.device)
    names = model.param_names()
    arrays = {n: p.numpy() for n, p in zip(names, model.parameters())}
    # the reference stores log_s as a 0-d array
    order = list(names)
    arrays["R0"] = np.stack([p.R0 for p in model.poses], axis=0)
    arrays["pose_nu"] = np.stack([np.asarray(p.nu_data(), dtype=np.float64) for p in model.poses], axis=0)
    arrays["pose_t"] = np.stack([np.asarray(p.t_data(), dtype=np.float64) for p in model.poses], axis=0)
    order += ["R0", "pose_nu", "pose_t"]
    if opt is not None:
        for name, m, v, t in zip(names, opt.m, opt.v, opt.t):
            arrays[f"adam_m_{name}"] = m.cpu().numpy()
            arrays[f"adam_v_{name}"] = v.cpu().numpy()
            arrays[f"adam_t_{name}"] = np.array([t], dtype=np.int64)
            order += [f"adam_m_{name}", f"adam_v_{name}", f"adam_t_{name}"]
    header = {
        "kind": "gridsurf-model",
        "iteration": int(iteration),
        "config": cfg.echo(),
        "grid": {
            "lo": list(map(float, model.grid.lo)),
            "hi": list(map(float, model.grid.hi)),
            "levels": [{"origin": list(map(float, l.geom.origin)),
                        "voxel_size": l.geom.voxel_size, "dims": list(l.geom.dims),
                        "width": int(l.width)} for l in model.grid.levels + [model.grid.color]],
        },
        "pose_trainable": [bool(p.trainable) for p in model.poses],
        "has_adam": opt is not None,
        "array_order": order,
    }
    ckpt.write_container(path, header, arrays)


def load_model(path, device=None):
    """Rebuild (model, cfg, iteration, opt-or-None) from a GSURFCKPT1 file."""
    import torch
    header, arrays = ckpt.read_container(path)
    cfg_d = dict(header["config"])
    w = cfg_d.pop("weights")
    cfg = TrainConfig(**{**cfg_d,
                         "bounds": tuple(map(tuple, cfg_d["bounds"])) if cfg_d.get("bounds") else None,
                         "voxel_sizes": tuple(cfg_d["voxel_sizes"]),
                         "weights": LossWeights(**w)})
    g = header["grid"]
    lv = g["levels"]
    dt = arrays["level0"].dtype
    poses = np.zeros((len(header["pose_trainable"]), 4, 4))
    poses[:, 3, 3] = 1.0
    poses[:, :3, :3] = arrays["R0"]
    poses[:, :3, 3] = arrays["pose_t"]
    model = mdl.allocate_model(g["lo"], g["hi"], [m["voxel_size"] for m in lv[:-1]],
                               lv[0]["width"], lv[-1]["voxel_size"], lv[-1]["width"], poses, dt,
                               _device(device), trainable=header["pose_trainable"])
    for lev, meta in zip(model.grid.levels + [model.grid.color], lv):
        if list(lev.geom.dims) != list(meta["dims"]) or not np.allclose(lev.geom.origin,
                                                                        meta["origin"]):
            raise ckpt.CheckpointError("grid geometry does not match the checkpoint")
    names = model.param_names()
    for n, p in zip(names, model.parameters()):
        p.set(arrays[n])
    opt = None
    if header.get("has_adam"):
        opt = Adam(model.parameters(), [0.0] * len(model.parameters()))
        for n, p, m, v in zip(names, model.parameters(), opt.m, opt.v):
            m.copy_(torch.from_numpy(np.ascontiguousarray(arrays[f"adam_m_{n}"])).reshape(p.shape))
            v.copy_(torch.from_numpy(np.ascontiguousarray(arrays[f"adam_v_{n}"])).reshape(p.shape))
        opt.t = [int(arrays[f"adam_t_{n}"][0]) for n in names]
    return model, cfg, int(header["iteration"]), opt


# ---------------------------------------------------------------------------
# training loop (gs/optimizer.py:331-391)

CSV_HEADER = "iter,total,rgb,depth,sdf,fs,eik,smooth,s\n"


class DrawPrefetcher:
    """Host draws (numpy RNG, gs/optimizer.py:363-366 + gs/renderer.py:320-336,
    416-423) of the next iterations on a background thread.  The main thread
    spends each step waiting on CUDA events, which releases the GIL, so the
    draws of iteration k+1 overlap the device work of iteration k."""

    def __init__(self, fn, start, depth=2):
        import queue
        import threading
        self._queue_mod = queue
        self.fn = fn
        self.q = queue.Queue(maxsize=depth)
        self.stop_ev = threading.Event()
        self.t = threading.Thread(target=self._run, args=(int(start),), daemon=True)
        self.t.start()

    def _run(self, it):
        while not self.stop_ev.is_set():
            try:
                item = self.fn(it)
            except BaseException as e:  # surfaced by get()
                item = e
            while not self.stop_ev.is_set():
                try:
                    self.q.put((it, item), timeout=0.1)
                    break
                except self._queue_mod.Full:
                    continue
            if isinstance(item, BaseException):
                return
            it += 1

    def get(self, it):
        got, item = self.q.get()
        if isinstance(item, BaseException):
            raise item
        if got != it:
            raise RuntimeError(f"draw prefetch out of order: wanted {it}, got {got}")
        return item

    def close(self):
        self.stop_ev.set()
        self.t.join(timeout=5)


class Trainer:
    """The device-resident inner loop: draw -> objective+backward -> Adam.

    Loss parts for iteration k are copied to pinned host memory and read
    one iteration later, so the host never waits on the GPU inside the
    loop; divergence is enforced on the device (the Adam launch is skipped
    when the total is non-finite or above the threshold, and stays skipped)
    so the model state matches the reference's when the error surfaces.

    With ``dist`` (torch.distributed, one process per GPU) each rank takes
    its row shard of the global batch and the step runs as
    parallel.DataParallelStep."""

    def __init__(self, model, dataset, cfg, opt, dist=None, rank=0, world=1, overlap_adam=False):
        import torch
        from .parallel import DataParallelStep
        self.torch = torch
        self.model, self.cfg, self.opt = model, cfg, opt
        self.dataset = Dataset.wrap(dataset)
        self.engine = engine_for(model, self.dataset)
        self.host_parts = torch.zeros((2, _lib.N_PARTS), dtype=torch.float64).pin_memory()
        # the step's status words (grid bounds, importance overflow, view
        # directions), read with the parts: the workspace copy is zeroed by
        # the next launch
        self.host_status = torch.zeros((2, _lib.N_STATUS), dtype=torch.int32).pin_memory()
        self.events = [torch.cuda.Event(), torch.cuda.Event()]
        self.rank, self.world = int(rank), int(world)
        self.dp = DataParallelStep(self.engine, dist) if dist is not None and world > 1 else None
        # opt-in, single GPU: the colour-grid Adam of step k under step k+1's
        # sampling (AdamOverlap; bit-identical, measured slower at config 2)
        self.overlap = AdamOverlap(opt, model) if (overlap_adam and self.dp is None) else None
        self.prefetcher = None
        self.last_h2d = 0

    def draws(self, it):
        """(this rank's HostDraws, step kwargs) of iteration ``it``."""
        from .parallel import shard_draws
        d = host_draws(self.model, self.dataset, self.cfg, it)
        if self.world == 1:
            return d, {}
        return shard_draws(d, self.rank, self.world)

    def start_prefetch(self, start_it):
        self.stop_prefetch()
        self.prefetcher = DrawPrefetcher(self.draws, start_it)

    def stop_prefetch(self):
        if self.prefetcher is not None:
            self.prefetcher.close()
            self.prefetcher = None

    def launch(self, it, draws=None, slot=0):
        if draws is not None:
            d, kw = draws if isinstance(draws, tuple) else (draws, {})
        elif self.prefetcher is not None:
            d, kw = self.prefetcher.get(it)
        else:
            d, kw = self.draws(it)
        self.last_h2d = d.h2d_bytes
        ids, sm = self.engine.upload(d)
        if self.overlap is not None:
            self.engine.launch(self.cfg, d, ids, sm, phases=1, **kw)
            self.overlap.wait_colour()
            ws = self.engine.launch(self.cfg, d, ids, sm, phases=2, fresh=False, **kw)
        elif self.dp is None:
            ws = self.engine.launch(self.cfg, d, ids, sm, **kw)
        else:
            ws = self.dp(self.cfg, d, ids, sm, **kw)
        self.host_parts[slot].copy_(ws["parts"], non_blocking=True)
        self.host_status[slot].copy_(ws["status"], non_blocking=True)
        self.events[slot].record()
        if self.overlap is not None:
            self.overlap.step(ws, self.cfg.divergence_threshold)
        elif self.dp is None:
            self.opt.t = [t + 1 for t in self.opt.t]
            self.opt._launch(guard=ws["parts"], guard_threshold=self.cfg.divergence_threshold,
                             guard_status=ws["status"])
        else:
            self.opt.t = [t + 1 for t in self.opt.t]
            self.dp.adam(self.opt, guard=ws["parts"], guard_threshold=self.cfg.divergence_threshold,
                         guard_status=ws["status"])
        if self.engine.refine and (it + 1) % self.cfg.pose_refresh_every == 0:
            for p in self.model.poses:  # gs/optimizer.py:374-376
                p.refresh()
        return ws

    def drain(self):
        """Order every later read of the parameters (host copies, checkpoints)
        after the side-stream colour-grid update of the last step."""
        if self.overlap is not None:
            self.overlap.drain()

    def parts(self, slot):
        self.events[slot].synchronize()
        p = self.host_parts[slot].numpy()
        return {k: float(p[i]) for i, k in enumerate(_lib.PART_NAMES)}

    def status(self, slot):
        """Host copy of the step's status words (valid after parts(slot))."""
        self.events[slot].synchronize()
        return self.host_status[slot].numpy().copy()


def train(dataset, cfg, out_dir, initial_poses=None, resume=None):
    """Optimise a model on a dataset; returns (model, final checkpoint path)
    (gs/optimizer.py:334-391).  Writes loss_log.csv and checkpoints."""
    os.makedirs(out_dir, exist_ok=True)
    dataset = Dataset.wrap(dataset)
    if resume is not None:
        model, cfg_loaded, start_it, opt = load_model(resume)
        cfg = cfg_loaded if cfg is None else cfg
        if opt is None:
            opt = make_optimizer(model, cfg)
        opt.lrs = _lr_list(model, cfg)
        csv_mode = "a"
    else:
        model = build_model(dataset, cfg, initial_poses=initial_poses)
        opt = make_optimizer(model, cfg)
        start_it = 0
        csv_mode = "w"
    csv_path = os.path.join(out_dir, "loss_log.csv")
    final_path = os.path.join(out_dir, "ckpt_final.gsck")
    T = Trainer(model, dataset, cfg, opt)
    every = max(cfg.checkpoint_every, 1)

    launched = []  # iterations whose Adam launch is enqueued but not yet checked

    def finish(it, slot, csv):
        parts = T.parts(slot)
        # the reference raises inside train_objective (GridBoundsError, ...)
        # or right after it (DivergenceError), before its Adam step: the
        # device skipped this and every later Adam launch (guard), so only
        # the host step counters run ahead and are rolled back
        try:
            check_status(T.status(slot), cfg.precision)
            if not np.isfinite(parts["total"]) or parts["total"] > cfg.divergence_threshold:
                raise DivergenceError(f"loss diverged at iteration {it}: {parts}")
        except Exception:
            k = len(launched) - launched.index(it)
            opt.t = [t - k for t in opt.t]
            raise
        launched.remove(it)
        csv.write(f"{it},{parts['total']:.10g},{parts['rgb']:.10g},{parts['depth']:.10g},"
                  f"{parts['sdf']:.10g},{parts['fs']:.10g},{parts['eik']:.10g},"
                  f"{parts['smooth']:.10g},{parts['s']:.10g}\n")
        if it % 50 == 0:
            log.info("iter %d total %.5f", it, parts["total"])

    with open(csv_path, csv_mode) as csv:
        if csv_mode == "w":
            csv.write(CSV_HEADER)
        pending = None  # (iteration, slot)
        T.start_prefetch(start_it)
        try:
            for it in range(start_it, cfg.iterations):
                slot = it % 2
                T.launch(it, slot=slot)
                launched.append(it)
                if pending is not None:
                    finish(pending[0], pending[1], csv)
                pending = (it, slot)
                if (it + 1) % every == 0:
                    finish(it, slot, csv)
                    pending = None
                    T.drain()
                    save_model(os.path.join(out_dir, f"ckpt_{it + 1:06d}.gsck"), model, cfg,
                               it + 1, opt)
            if pending is not None:
                finish(pending[0], pending[1], csv)
        finally:
            T.stop_prefetch()
            T.drain()
            csv.flush()
    save_model(final_path, model, cfg, cfg.iterations, opt)
    return model, final_path
