"""Benchmark: GO-Surf training iterations (forward + backward + Adam) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}]

Workload (BASELINE.json configs[1]): ScanNet-shaped synthetic RGB-D sequence
(640x480, ScanNet intrinsics), the paper's 4-level grid (0.96/0.24/0.06/0.03 m,
colour 0.03 m) over the pinned 7 x 7 x 3.25 m box (P = 63.9 M parameters),
M = 6144 rays per GPU, 96 + 3x12 = 132 samples per ray, smoothness on,
float32.  A step = one full training iteration: device ray draw +
stratified + 3 importance rounds, taped forward, rendering, six losses,
fused backward with grid scatter, dense Adam over all parameters.

value: rays/s with the step inputs already resident in HBM (device-timed).
e2e:   rays/s through the public API (host numpy draws each step, pinned
       H2D of ray ids + smoothness points, D2H of the loss parts).
Multi-GPU (torchrun): weak scaling, 6144 rays per rank from one global batch,
NCCL all-reduce of the partition counts and of the gradient arena.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training rays/sec (fwd+bwd+Adam) at 1/2/4/8 B200; % HBM roofline; vs CPU ref"
M_PER_GPU = 6144
FRAMES = 8


def peaks():
    """(HBM GB/s, bf16 dense TFLOP/s burst, kind) from MEASURED_PEAKS.json
    (driver-written), else the B200_PROFILING.md fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), float(d.get("bf16_tflops", 1590.0)), "measured"
    return 6650.0, 1590.0, "fallback"


def make_cfg(precision="single", batch=M_PER_GPU, seed=0, config=2, coarse=96, smooth=True):
    """config 2 (BASELINE configs[1]) or 4 (configs[3]); c5's axes: the ray
    batch, the coarse samples (N = coarse + 3 x 12) and smoothness on/off."""
    from paper_2206_14735_b200 import optimizer, scenes
    kw = dict(precision=precision, batch_rays=batch, seed=seed, iterations=10 ** 6,
              coarse_samples=coarse)
    if config == 4:
        kw.update(bounds=scenes.CONFIG4_BOUNDS, voxel_sizes=scenes.CONFIG4_VOXELS,
                  color_voxel=scenes.CONFIG4_COLOR_VOXEL)
    elif config == 1:
        pass  # the reference's defaults: 4-level grid, bounds derived from the frames
    else:
        kw.update(bounds=scenes.CONFIG2_BOUNDS)
    cfg = optimizer.TrainConfig(**kw)
    if not smooth:
        cfg.weights.smooth = 0.0
    return cfg


class Clocks:
    """SM clock + throttle-reason sampling during the timed region
    (B200_PROFILING.md clocks line): NVML in-process every 20 ms (nvidia-smi
    spawns are too slow for a sub-second region), nvidia-smi as fallback."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self):
        self.samples = []  # (sm_mhz, max_mhz, set of reasons)
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        import pynvml as N
        N.nvmlInit()
        idx = int(os.environ.get("LOCAL_RANK", "0"))
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            idx = int(vis.split(",")[idx])
        h = N.nvmlDeviceGetHandleByIndex(idx)
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)

        def read():
            sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            return sm, mx, {k for k, b in bits.items() if r & b}
        return read

    def _smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

        def read():
            out = subprocess.run(["nvidia-smi", "-i", os.environ.get("LOCAL_RANK", "0"),
                                  f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                 capture_output=True, text=True, timeout=5).stdout
            f = [x.strip() for x in out.strip().split(",")]
            return (float(f[0]), float(f[1]),
                    {self.NAMES[i] for i in range(4) if f[2 + i].lower().startswith("active")})
        return read

    def start(self):
        try:
            read = self._nvml()
            read()
            period = 0.02
        except Exception:
            read, period = self._smi(), 0.2

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(read())
                except Exception:
                    pass
                self._stop.wait(period)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples]
        reasons = sorted(set().union(*[s[2] for s in self.samples])) if self.samples else []
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def b_alg_bytes(model, M, N, S):
    """Algorithmic HBM bytes of one step."""
    P = sum(p.size for p in model.parameters())
    G_s = sum(8 * l.width * 4 for l in model.grid.levels
              if l.features.size * 4 > 32 * 2 ** 20)
    Cc_s = 8 * 6 * 4 if model.grid.color.features.size * 4 > 32 * 2 ** 20 else 0
    n_imp = N - 12  # coarse + 2 x 12 evaluated (the last round's 12 are not)
    return 32 * P + M * (n_imp * G_s + N * 2 * (G_s + Cc_s)) + 2 * S * 2 * G_s, P


HID, IN_G, IN_C = 32, 16, 9
MAC_GEO_FWD = IN_G * HID + HID * HID + HID                       # 1568
MAC_DELTA = HID * HID + HID * IN_G                                # dphi/dz chain
MAC_COL_FWD = IN_C * HID + HID * HID + HID * 3
MAC_GEO_BWD = MAC_GEO_FWD + MAC_DELTA + IN_G * HID + HID * HID + IN_G * HID + HID * HID + HID
MAC_COL_BWD = MAC_COL_FWD + 3 * HID + HID * HID + HID * 6 + (IN_C + 1) * HID + HID * HID + HID * 3


def workload_name(args, N):
    sm = "off" if args.no_smooth else "on"
    if args.config == 1:
        return (f"config1: sphere-in-box room, 20 RGB-D frames 160x120, default 4-level grid "
                f"(0.96/0.24/0.06/0.03 m), derived bounds, {args.rays} rays, "
                f"{args.coarse}+3x12 samples/ray, smoothness {sm}")
    if args.config == 4:
        return (f"config4: 10 m synthetic room, 640x480 RGB-D, 4-level grid "
                f"(0.96/0.24/0.06/0.02 m + 0.02 m colour), 11 m box, "
                f"{args.coarse}+3x12 samples/ray, smoothness {sm}")
    if args.refine_poses:
        sm += ", pose refinement on"
    return (f"config2: ScanNet-shaped 640x480 RGB-D, paper 4-level grid "
            f"(0.96/0.24/0.06/0.03 m + 0.03 m colour), pinned 7x7x3.25 m box, "
            f"{args.coarse}+3x12 samples/ray, smoothness {sm}")


def traffic_of(kernel, workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full summary (profiles/traffic.json) of the same
    workload (its "workload" key), else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    if d.get("workload") != workload:
        return None
    for k, v in d.get("kernels", {}).items():
        if k.startswith(kernel):
            return v
    return None


def kernel_table(model, kt, K, M, N, S, P, peak_hbm, peak_bf16, workload=None):
    """Per-kernel algorithmic work over live CUDA-event times,
    against both roofs: measured HBM bandwidth, and the 3xTF32 tensor rate
    the float32 MLPs run at (tf32 is half the measured bf16 dense rate, and
    3xTF32 spends three tf32 MMAs per fp32-accurate product).  `bound` is
    the roof with the larger ideal time.  Kernels launched once per step
    also carry `dram_frac`: the measured DRAM bytes of one launch
    (profiles/traffic.json, ncu) over its live time, against the copy peak."""
    G_s = sum(8 * l.width * 4 for l in model.grid.levels if l.features.size * 4 > 32 * 2 ** 20)
    Cc_s = 8 * 6 * 4 if model.grid.color.features.size * 4 > 32 * 2 ** 20 else 0
    n_imp = N - 12  # coarse + 2 x 12 evaluated (the last round's 12 are not)
    NS = M * N + 2 * S
    work = {  # kernel: (bytes, MACs) per step
        "k_adam": (32 * P, 0),
        "k_sdf_eval": (M * n_imp * G_s, M * n_imp * MAC_GEO_FWD),
        "k_fwd": (NS * G_s + M * N * Cc_s, NS * (MAC_GEO_FWD + MAC_DELTA) + M * N * MAC_COL_FWD),
        "k_bwd_geom": (NS * G_s, NS * MAC_GEO_BWD),
        "k_bwd_color": (M * N * Cc_s, M * N * MAC_COL_BWD),
    }
    tensor_peak = peak_bf16 / 2.0 / 3.0  # TFLOP/s of fp32-accurate 3xTF32 products
    rows = []
    for name, (ms, n) in sorted(kt.items(), key=lambda x: -x[1][0]):
        t = ms / K / 1e3
        b, mac = work.get(name, (0, 0))
        hbm = b / t / 1e9 if t > 0 else 0.0
        fl = 2 * mac / t / 1e12 if t > 0 else 0.0
        t_hbm, t_ten = b / (peak_hbm * 1e9), 2 * mac / (tensor_peak * 1e12)
        r = {"kernel": name, "ms_per_step": ms / K, "launches_per_step": n / K,
             "alg_bytes": b, "alg_flops": 2 * mac, "hbm_gbs": hbm, "tflops": fl,
             "hbm_frac": hbm / peak_hbm, "tensor_frac": fl / tensor_peak}
        tr = traffic_of(name, workload) if workload else None
        if tr is not None and t > 0 and n == K:  # one launch per step: ncu DRAM bytes over its time
            r["traffic_bytes"] = tr
            r["dram_frac"] = tr / t / 1e9 / peak_hbm
        if t_ten > t_hbm:
            r.update(bound="tensor", achieved=fl, peak=tensor_peak, unit="TFLOP/s", frac=fl / tensor_peak,
                     peak_kind="3xTF32 rate derived from the measured bf16 dense peak "
                               "(MEASURED_PEAKS.json bf16_tflops / 2 (tf32) / 3 (passes))")
        else:
            r.update(bound="hbm", achieved=hbm, peak=peak_hbm, unit="GB/s",
                     frac=hbm / peak_hbm, peak_kind="measured (MEASURED_PEAKS.json hbm_gbs)")
        rows.append(r)
    return rows


# ----------------------------------------------------------------------------
# reference arm: the unmodified reference package (baseline/ref_step.py)

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available():
    return os.path.isdir(os.path.join(REF_DIR, "gridsurf"))


def reference_step(steps, warmup, rays, frames, config, precision="single", timeout=1500):
    """Time the reference's own training step (gs/optimizer.py:362-373) on
    the host cores in a separate process (baseline/ref_step.py): the
    reference's scenegen renders the dataset, nothing of this repository
    (no _gsb.so) is loaded there.  Returns its JSON dict."""
    threads = str(os.cpu_count() or 1)
    env = dict(os.environ, OPENBLAS_NUM_THREADS=threads, OMP_NUM_THREADS=threads,
               MKL_NUM_THREADS=threads, NUMBA_CACHE_DIR=os.path.join(
                   os.environ.get("TMPDIR", "/tmp"), "gsb_ref_numba"),
               PYTHONDONTWRITEBYTECODE="1")
    env.pop("CUDA_VISIBLE_DEVICES", None)
    cmd = [sys.executable, os.path.join(ROOT, "baseline", "ref_step.py"), "--steps", str(steps),
           "--warmup", str(warmup), "--rays", str(rays), "--frames", str(frames),
           "--config", str(config), "--precision", precision]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
    if out.returncode != 0:
        raise RuntimeError(f"reference step failed: {out.stderr[-2000:]}")
    return json.loads(out.stdout.strip().splitlines()[-1])


def port_step(steps, warmup, rays, frames, config, threads):
    """Fallback when baseline/_ref is absent: the oracle port of the same step
    (oracle/gridsurf_oracle.py, ~3x slower than gridsurf on the same cores),
    on a dataset rendered by the oracle's host renderer (no repo .so)."""
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle import gridsurf_oracle as O
    from oracle import scene_host as SH
    from _golden import cfg_ns
    ds = SH.config_dataset(config, frames, threads)
    bounds = SH.CONFIG2_BOUNDS if config == 2 else None
    cfg = cfg_ns(precision="single", batch_rays=rays, bounds=bounds)
    lo, hi = O.derive_bounds(ds, cfg)
    P = O.create_params(lo, hi, ds.poses, seed=0, dtype=np.float32)
    opt = O.Adam(P.arrays(), P.lrs())
    times = []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        O.train_step(P, opt, ds, cfg, it)
        if it >= warmup:
            times.append(time.perf_counter() - t0)
    tot = float(sum(times))
    return {"value": rays * steps / tot, "ms_per_step": 1e3 * tot / steps, "steps": steps,
            "warmup": warmup, "threads": threads, "rays": rays, "frames": frames,
            "params": int(sum(a.size for a in P.arrays()))}


def cpu_reference(steps, warmup, rays, frames, config):
    """(result dict, kind): the reference itself when installed, else the port."""
    threads = os.cpu_count() or 1
    if reference_available():
        return reference_step(steps, warmup, rays, frames, config), "reference"
    return port_step(steps, warmup, rays, frames, config, threads), "port"


def ref_sample_text(r, kind, config):
    who = ("the unmodified reference package (gridsurf 0.1.0 from baseline/_ref): "
           "draw_ray_batch + train_objective + dc.grad + Adam.step"
           if kind == "reference" else "the oracle port of the reference step")
    return (f"{who}, config{config}, {r['rays']} rays x 132 samples per step, {r['frames']} "
            f"frames rendered by its own scenegen, dense Adam over {r['params']} parameters; "
            f"{r['steps']} timed steps after {r['warmup']} warm-up (numba JIT), "
            f"{r['threads']} host threads")


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    rays = args.rays if args.config != 1 else 1024
    frames = args.frames if args.config == 2 else 20
    # full-size steps (the whole 6144-ray batch, same frames and bounds as the
    # B200 arm); ~9 s per c2 step on 8 cores, so at most 20 are timed
    steps = max(1, min(args.steps, 20))
    r, kind = cpu_reference(steps, 1, rays, frames, args.config)
    v = r["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "rays/s",
            "n_gpus": args.gpus, "steps": r["steps"], "warmup": r["warmup"],
            "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(args, 132), "rays_per_gpu": rays,
                       "samples_per_ray": 132, "params": r["params"], "frames": frames},
            "cpu_baseline": {"value": v, "unit": "rays/s", "cores": r["threads"], "kind": kind,
                             "sample": ref_sample_text(r, kind, args.config)},
            "e2e": {"value": v, "unit": "rays/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
# B200 arm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="single")
    ap.add_argument("--frames", type=int, default=FRAMES)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rays", type=int, default=M_PER_GPU)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 4],
                    help="2: ScanNet-shaped room (headline); 1: sphere-in-box 20 x 160x120, M = 1024 "
                         "(the reference's CPU-runnable case); 4: 10 m scene, 0.02 m grid (P = 1.7 B)")
    ap.add_argument("--coarse", type=int, default=96, help="coarse samples per ray (c5 sweep)")
    ap.add_argument("--no-smooth", action="store_true", help="lambda_smooth = 0 (c5 sweep)")
    ap.add_argument("--refine-poses", action="store_true",
                    help="pose refinement on (refine_poses=True, frame 0 frozen; not the headline)")
    ap.add_argument("--no-prefetch", action="store_true",
                    help="host draws on the main thread in the e2e leg (default: a background "
                         "thread, as train() does)")
    ap.add_argument("--overlap-adam", action="store_true",
                    help="step k's colour-grid Adam on a side stream under step k+1's sampling "
                         "(optimizer.AdamOverlap; measured slower on one B200: 1.412 vs 1.384 ms)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling (SURVEY 8d c3(i)): the global batch is --rays, split by rows "
                         "across the ranks (default: weak, --rays per rank)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    from paper_2206_14735_b200 import _lib, engine, optimizer, parallel, scenes
    from paper_2206_14735_b200.renderer import engine_for

    ws_, rank, local = dist_env()
    local = local % max(torch.cuda.device_count(), 1)  # (functional smoke runs may share a GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if ws_ > 1:
        import torch.distributed as dist
        # GSB_DIST_BACKEND=gloo only for functional smoke runs of the N > 1 path
        # on fewer GPUs than ranks (host collectives; not a measurement)
        backend = os.environ.get("GSB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        pg = dist
    W = max(args.warmup, 3)
    K = args.steps
    # weak: --rays per rank (global batch rays x ranks); strong: --rays in total,
    # rank g takes rows parallel.shard_rows(rays, g, N) of the one global batch
    M_glob = args.rays if args.strong else args.rays * ws_
    lo_r, hi_r = parallel.shard_rows(M_glob, rank, ws_)
    M = hi_r - lo_r  # this rank's rays
    cfg = make_cfg(args.precision, batch=M_glob, config=args.config, coarse=args.coarse,
                   smooth=not args.no_smooth)
    cfg.refine_poses = bool(args.refine_poses)
    if args.config == 4:
        ds = scenes.config4(frames=args.frames, threads=min(8, os.cpu_count() or 1))
    elif args.config == 1:
        ds = scenes.config1(frames=20)
    else:
        ds = scenes.config2(frames=args.frames, threads=min(8, os.cpu_count() or 1))
    model = optimizer.build_model(ds, cfg, skip_init=True, device=dev)
    opt = optimizer.make_optimizer(model, cfg)
    eng = engine_for(model, ds)
    N = cfg.coarse_samples + cfg.importance_rounds * cfg.importance_add

    dp = parallel.DataParallelStep(eng, pg) if pg is not None else None

    def draws_for(it):
        """Host draws of the global batch; this rank's shard (rank 0: smoothness)."""
        return parallel.shard_draws(engine.host_draws(model, ds, cfg, it), rank, ws_)

    S = cfg.weights.smooth_count if cfg.weights.smooth != 0.0 else 0

    def objective(d, kw, ids, sm):
        if isinstance(sm, tuple):  # device-resident raw smoothness draws: part of the step
            sm = eng.smooth_points_dev(*sm)
        if dp is None:
            return eng.launch(cfg, d, ids, sm, **kw)
        return dp(cfg, d, ids, sm, **kw)

    def adam_step():
        opt.t = [t + 1 for t in opt.t]
        if dp is None:
            opt._launch()
        else:
            dp.adam(opt)  # sharded Adam + all-gather (parallel.py)

    # opt-in (--overlap-adam), single GPU: step k's colour-grid Adam on a side
    # stream under step k+1's sampling phase (optimizer.AdamOverlap;
    # bit-identical).  Measured slower: the HBM stream slows the latency-bound
    # sampling and forward kernels more than it hides (1.412 vs 1.384 ms)
    ov = optimizer.AdamOverlap(opt, model) if (dp is None and args.overlap_adam) else None

    def one_step(d, kw, ids, sm):
        if ov is None:
            w = objective(d, kw, ids, sm)
            adam_step()
            return w
        if isinstance(sm, tuple):
            sm = eng.smooth_points_dev(*sm)
        eng.launch(cfg, d, ids, sm, phases=1, **kw)
        ov.wait_colour()
        w = eng.launch(cfg, d, ids, sm, phases=2, fresh=False, **kw)
        ov.step(w, cfg.divergence_threshold)
        return w

    # ---- device-resident inputs for warmup + timed steps
    pre = []
    for it in range(W + K):
        d, kw = draws_for(it)
        ids = torch.from_numpy(d.ray_ids).to(dev)
        sm = None
        if d.smooth_raw is not None:
            sm = (eng.upload_smooth_raw(d.smooth_raw), d.n_smooth, d.smooth_delta)
        pre.append((d, kw, ids, sm))
    torch.cuda.synchronize()
    for it in range(W):
        one_step(*pre[it])
    torch.cuda.synchronize()

    # timed region: objective and Adam event pairs on the step stream
    clocks = Clocks()
    clocks.start()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    t_step, t_adam = [], []
    launches0 = eng.lib.gsb_launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for k in range(K):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        c = torch.cuda.Event(enable_timing=True)
        a.record()
        if ov is None:
            objective(*pre[W + k])
            b.record()
            adam_step()
        else:  # b: after phase 2; c: after the main-stream part of Adam
            d_, kw_, ids_, sm_ = pre[W + k]
            if isinstance(sm_, tuple):
                sm_ = eng.smooth_points_dev(*sm_)
            eng.launch(cfg, d_, ids_, sm_, phases=1, **kw_)
            ov.wait_colour()
            w_ = eng.launch(cfg, d_, ids_, sm_, phases=2, fresh=False, **kw_)
            b.record()
            ov.step(w_, cfg.divergence_threshold)
        c.record()
        t_step.append((a, b))
        t_adam.append((b, c))
    if ov is not None:
        ov.drain()  # the timed region ends after the last colour-grid update
    ev1.record()
    torch.cuda.synchronize()
    launches = int(eng.lib.gsb_launch_count() - launches0)
    if pg:
        pg.barrier()
    clk = clocks.stop()
    total_ms = ev0.elapsed_time(ev1)
    if pg:
        tt = torch.tensor([total_ms], device=dev)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / K
    adam_ms = float(np.mean([x.elapsed_time(y) for x, y in t_adam]))
    obj_ms = float(np.mean([x.elapsed_time(y) for x, y in t_step]))
    value = M_glob * K / (total_ms / 1e3)

    # ---- per-kernel live timing (CUDA events between launches on the step
    # stream, gsb_timing_enable); a separate pass so `value` carries no markers
    eng.lib.gsb_timing_enable(1)
    for k in range(K):  # fused Adam here: the per-kernel events live on one stream
        objective(*pre[W + k])
        adam_step()
    torch.cuda.synchronize()
    eng.lib.gsb_timing_enable(0)
    kt = _lib.kernel_times()

    # ---- e2e through the public API (host draws + H2D + D2H of parts);
    # the Trainer prefetches host draws on a background thread
    T = optimizer.Trainer(model, ds, cfg, opt, dist=pg, rank=rank, world=ws_,
                          overlap_adam=args.overlap_adam)
    base_it = W + K
    if not args.no_prefetch:  # as train() runs (optimizer.py: T.start_prefetch)
        T.start_prefetch(base_it)
    # untimed e2e warm-up: prefetch thread start, pinned staging, first draws
    pending = None
    for k in range(W):
        T.launch(base_it + k, slot=k % 2)
        if pending is not None:
            T.parts(pending)
        pending = k % 2
    if pending is not None:
        T.parts(pending)
    base_it += W
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    gc.collect()
    gc.disable()  # no collector pause inside the timed host loop
    t0 = time.perf_counter()
    pending = None
    for k in range(K):
        T.launch(base_it + k, slot=k % 2)
        if pending is not None:
            T.parts(pending)
        pending = k % 2
    if pending is not None:
        T.parts(pending)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    gc.enable()
    T.stop_prefetch()
    if pg:
        tt = torch.tensor([e2e_s], device=dev)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e = M_glob * K / e2e_s

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel + per-kernel table
    peak, peak_bf16, peak_kind = peaks()
    B, P = b_alg_bytes(model, M, N, S)
    table = kernel_table(model, kt, K, M, N, S, P, peak, peak_bf16,
                         f"config{args.config}" + ("-pose" if args.refine_poses else ""))
    dom = max(table, key=lambda r: r["ms_per_step"])
    roofline = {"bound": dom["bound"], "kernel": dom["kernel"], "achieved": dom["achieved"],
                "peak": dom["peak"], "unit": dom["unit"], "frac": dom["frac"],
                "traffic": None, "peak_kind": dom["peak_kind"],
                "share_of_step": dom["ms_per_step"] / ms_step,
                "step_b_alg_gb": B / 1e9,
                "step_hbm_frac": B / (ms_step / 1e3) / 1e9 / peak,
                "objective_ms": obj_ms, "adam_ms": adam_ms,
                "kernels": table}
    roofline["note"] = ("k_adam's algorithmic bytes are 32 B/param (p, g, m, v read and written); it "
                        "reads all 16 B/param but skips the gradient-zeroing store where g is already "
                        "+0 and every store where g, m and v are all +0 (never-touched parameters: the "
                        "update would rewrite the same bits), so its algorithmic-byte rate can exceed "
                        "the copy peak; `traffic` / the table's dram_frac use the measured DRAM bytes "
                        "per launch (profiles/traffic.json, ncu)")
    tr = traffic_of(dom["kernel"], f"config{args.config}" + ("-pose" if args.refine_poses else ""))
    if tr is not None:
        roofline["traffic"] = tr
    cpu = None
    if not args.no_cpu_baseline and ws_ == 1:
        # one full-size reference step after one warm-up step (~10-30 s of CPU work)
        r, kind = cpu_reference(1, 1, M if args.config != 1 else 1024,
                                args.frames if args.config == 2 else 20, args.config)
        cpu = {"value": r["value"], "unit": "rays/s", "cores": r["threads"], "kind": kind,
               "sample": ref_sample_text(r, kind, args.config)}
    line = {"metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": ws_, "steps": K,
            "warmup": W, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None, "dtype": "f32" if args.precision == "single" else "f64",
            "data": "synthetic",
            "config": {"workload": workload_name(args, N),
                       "rays_per_gpu": M, "global_rays": M_glob, "samples_per_ray": N, "params": P,
                       "frames": 20 if args.config == 1 else args.frames,
                       "frames_note": "SURVEY 8(d) defines c2 at F = 300 frames; the step "
                                      "cost does not depend on F (it only sets the ray-id range)",
                       "l2": f"working set (params/grad/m/v arenas = {4 * P * model.arena.params.element_size() / 1e9:.2f} GB) "
                             "> L2 (126 MB); no explicit flush"},
            "samples_per_s": value * N,
            "e2e": {"value": e2e, "unit": "rays/s", "h2d_bytes_per_step": int(T.last_h2d),
                    "d2h_bytes_per_step": 8 * 8},
            "gpu_launches": launches,
            "roofline": roofline, "cpu_baseline": cpu, "clocks": clk}
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
