"""Conditioned float32 parity of the production (tcgen05) step kernels.

The float32 step samples its own depths; a float32 run of the reference
samples slightly different ones, and at random init the objective is
ill-conditioned (alpha = 1 - sigma_{i+1}/sigma_i cancels), so comparing the
two end to end only bounds the kernels loosely.  Here the float32 device
step's OWN inputs are handed to the float64 oracle:

* its sampled depths (``ws["depths"]``) through ``inject_depths``;
* its float32 ray origins / directions (``ws["ray_o"]``, ``ws["ray_r"]``)
  through ``inject_rays``, with the taped points formed in float32 exactly as
  the step forms them (``point_dtype``), so both sides evaluate the same
  points;
* its float32 parameters, widened to float64;
* the same smoothness points (float32-representable, ``smooth_override``).

What remains is the kernels' own float32 / 3xTF32 arithmetic against float64
(gs/renderer.py:348-468 forward, gs/diffcore.py:1035-1104 backward), held to
the north-star tolerances: per-sample phi / grad-phi / colour
<= 1e-5 of the max-norm, loss parts <= 1e-5 relative, per-tensor gradients
<= 1e-4 of the tensor's max-norm.

The model is in the state training starts from: the sphere pre-fit
(``build_model(skip_init=False)``, gs/optimizer.py:206-213), as the survey's
f32-vs-f64 measurement was.  Cases: the small golden scene,
BASELINE configs[0] (c1: 20 x 160x120, 1024 rays) and a 512-ray slice of the
benchmarked config 2 (640x480, pinned 7 x 7 x 3.25 m box, P = 63.9 M).
"""

import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from _golden import OracleDataset, cfg_ns, load, rel_maxnorm  # noqa: E402
from oracle import gridsurf_oracle as O  # noqa: E402

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SAMPLE_TOL = 1e-5
PART_TOL = 1e-5
GRAD_TOL = 1e-4
PART_KEYS = ("total", "rgb", "depth", "sdf", "fs", "eik", "smooth")


def _dataset(case):
    from paper_2206_14735_b200 import camera, data, scenes
    if case == "c2":
        ds = scenes.config2(frames=2)
        return ds, dict(bounds=scenes.CONFIG2_BOUNDS, batch_rays=512)
    if case == "c1":
        z = np.load(os.path.join(HERE, "golden", "c1_double.npz"))
        import json
        meta = json.loads(z["meta_json"].tobytes().decode())
        fx, fy, cx, cy, w, h = meta["intr"]
        ds = data.Dataset(z["colors_u8"], z["depths_u16"], z["poses"],
                          camera.Intrinsics(fx, fy, cx, cy, int(w), int(h)))
        return ds, dict(batch_rays=1024)
    G = load("small", "double")
    i = G.ds.intrinsics
    ds = data.Dataset(G.a["colors_u8"], G.a["depths_u16"], G.a["poses"],
                      camera.Intrinsics(i.fx, i.fy, i.cx, i.cy, i.width, i.height))
    kw = {k: v for k, v in G.meta["cfg"].items() if k not in ("precision", "bounds", "voxel_sizes")}
    kw["voxel_sizes"], kw["bounds"] = G.cfg.voxel_sizes, G.cfg.bounds
    # its pinned box is a flat slab: a sphere of half the smallest extent
    # would touch the box faces
    return ds, dict(kw, smooth_count=G.meta["smooth_count"], sphere_radius_scale=0.4)


def oracle_from_model(model, poses, dtype):
    """Oracle parameters holding the device model's values (widened)."""
    P = O.create_params(model.grid.lo, model.grid.hi, poses, dtype=dtype,
                        voxel_sizes=tuple(l.geom.voxel_size for l in model.grid.levels),
                        geom_width=model.grid.levels[0].width,
                        color_voxel=model.grid.color.geom.voxel_size,
                        color_width=model.grid.color.width)
    for dst, src in zip(P.arrays(), model.parameters()):
        dst[...] = np.asarray(src.numpy(), dtype=dtype).reshape(dst.shape)
    return P


# ReLU kinks: where a pre-activation is within float32 rounding of zero the
# float32 step and the float64 oracle may take different sides, and the
# derivative (dphi/dz, so grad-phi and every gradient behind it) jumps while
# the values stay continuous.  That is the measure-zero set on which the
# derivative is not defined, not a kernel error.  So a sample whose grad-phi
# disagrees is re-evaluated by the oracle with the derivative masks of its
# near-zero units (|a| < KINK_MARGIN x the layer's max |a|) on the other side
# (relu_flips); it counts as a kink only if that reproduces the device's
# value, and the oracle step is then re-run with those flips.  Colour-net
# kinks are invisible in the forward (the colour is continuous), so if a
# colour gradient disagrees, the near-zero colour units are tried the same
# way (at most 2^4 combinations).  The alphas have the same kind of kink:
# alpha = 1 - min(sigma_{j+1} / sigma_j, 1) (gs/renderer.py:112-134) is
# continuous at ratio = 1 but its derivative is not, and where two adjacent
# samples have sigma equal to float32 rounding (a ray grazing a level set,
# where phi is stationary along it) the float32 step and the float64 oracle
# can take different sides.  The gradient then differs at that sample's
# corners while every per-sample value agrees; if a geometry gradient
# disagrees, the intervals with |ratio - 1| < RATIO_MARGIN are tried on the
# other side the same way.  Samples are never dropped and parameters never
# changed.
KINK_MARGIN = 1e-6
RATIO_MARGIN = 1e-5


def _near_zero(pre, margin=KINK_MARGIN):
    """{(layer, row, unit)} with |pre-activation| < margin x layer max."""
    out = []
    for layer, a in enumerate(pre):
        a = np.abs(np.asarray(a, dtype=np.float64))
        for row, unit in zip(*np.nonzero(a < margin * a.max())):
            out.append((layer, int(row), int(unit)))
    return out


def _geom_kink_flips(P64, pts, dev_g, ora_g, pre, scale):
    """Flips that make the oracle's grad-phi reproduce the device's at the
    samples where they disagree (only among near-zero units)."""
    import itertools
    bad = np.nonzero(np.abs(dev_g - ora_g).max(axis=1) > 0.25 * SAMPLE_TOL * scale)[0]
    cand = _near_zero(pre)
    flips = []
    for srow in bad:
        units = [(l, u) for l, r, u in cand if r == srow][:6]
        best = None
        for k in range(1, len(units) + 1):
            for sub in itertools.combinations(units, k):
                g = O.GeomPass(P64, pts[srow:srow + 1], [(l, 0, u) for l, u in sub]).gphi[0]
                e = np.abs(g - dev_g[srow]).max() / scale
                if best is None or e < best[0]:
                    best = (e, sub)
        if best is not None and best[0] <= SAMPLE_TOL:
            flips += [(l, int(srow), u) for l, u in best[1]]
    return flips


def _grad_errs(g, R, names):
    return {n: rel_maxnorm(g[n], R["grads"][n]) for n in names}


def resolve_kinks(oracle, R, dev, g, names, M, N, nsm):
    """Re-run the oracle with the ReLU kink flips the device took (see above)."""
    import itertools
    P64 = oracle.P
    flips = {}
    scale = np.abs(R["gphi"]).max()
    xf = R["xf"]
    fg = _geom_kink_flips(P64, xf, dev["gphi"][:M * N], R["gphi"].reshape(-1, 3), R["pre"]["geom"], scale)
    if fg:
        flips["geom"] = fg
    if nsm and R["smooth_gphi"] is not None:
        xs, xe = oracle.smooth
        pts = np.concatenate([xs, xe], axis=0)
        fs = _geom_kink_flips(P64, pts, dev["gphi"][M * N:M * N + 2 * nsm], R["smooth_gphi"],
                              R["pre"]["smooth"], scale)
        if fs:
            flips["smooth"] = fs
    if flips:
        R = oracle.run(flips)
    geo = [n for n in names if not n.startswith("color")]
    errs = _grad_errs(g, R, geo)
    if max(errs.values()) > 0.25 * GRAD_TOL:
        # candidates: near 1 (not exactly 1: saturated equal sigmas round the
        # same on both sides) and with a jump that matters
        dr = np.abs(R["ratio"] - 1.0)
        jump = R["ratio_jump"]
        near = (dr < RATIO_MARGIN) & (dr > 0) & (jump > 1e-3 * jump.max())
        rows, js = np.nonzero(near)
        cand = sorted(zip(rows.tolist(), js.tolist()), key=lambda t: dr[t])[:4]
        best = (max(errs.values()), R, None)
        for k in range(1, len(cand) + 1):  # the fewest flips that close the gap
            for sub in itertools.combinations(cand, k):
                R2 = oracle.run(dict(flips, ratio=list(sub)))
                e = max(_grad_errs(g, R2, geo).values())
                if e < best[0]:
                    best = (e, R2, sub)
            if best[0] <= 0.1 * GRAD_TOL:
                break
        if best[2] is not None:
            flips["ratio"] = list(best[2])
            R = best[1]
    col = [n for n in names if n.startswith("color")]
    errs = _grad_errs(g, R, col)
    if max(errs.values()) > GRAD_TOL:
        cand = sorted(_near_zero(R["pre"]["color"]),
                      key=lambda t: abs(R["pre"]["color"][t[0]][t[1], t[2]]))[:4]
        best = (max(errs.values()), R, None)
        for k in range(1, len(cand) + 1):
            for sub in itertools.combinations(cand, k):
                R2 = oracle.run(dict(flips, color=list(sub)))
                e = max(_grad_errs(g, R2, col).values())
                if e < best[0]:
                    best = (e, R2, sub)
        if best[2] is not None:
            flips["color"] = list(best[2])
            R = best[1]
    return R, flips


class _Oracle:
    def __init__(self, P, ods, ob, iteration, ocfg, smooth, depths, rays):
        self.P, self.smooth = P, smooth
        self.args = (ods, ob, iteration, ocfg)
        self.kw = dict(smooth_override=smooth, inject_depths=depths, inject_rays=rays,
                       point_dtype=np.float32)

    def run(self, flips=None):
        return O.train_objective(self.P, *self.args, relu_flips=flips, **self.kw)


def run_case(case, iteration=3):
    from paper_2206_14735_b200 import optimizer, renderer, sampler, seeds
    ds, kw = _dataset(case)
    smooth_count = kw.pop("smooth_count", None)
    cfg = optimizer.TrainConfig(precision="single", **kw)
    if smooth_count is not None:
        cfg.weights.smooth_count = smooth_count
    model = optimizer.build_model(ds, cfg, skip_init=False, device=torch.device("cuda", 0))
    ods = OracleDataset(ds.colors_u8, ds.depths_mm, ds.poses, ds.intrinsics)
    ocfg = cfg_ns(precision="double", batch_rays=cfg.batch_rays, seed=cfg.seed,
                  bounds=(tuple(model.grid.lo), tuple(model.grid.hi)),
                  voxel_sizes=tuple(cfg.voxel_sizes), coarse_samples=cfg.coarse_samples,
                  importance_rounds=cfg.importance_rounds, importance_add=cfg.importance_add,
                  near=cfg.near, max_depth=cfg.max_depth)
    ocfg.weights.smooth_count = cfg.weights.smooth_count
    P32 = oracle_from_model(model, ds.poses, np.float32)
    P64 = oracle_from_model(model, ds.poses, np.float64)
    # smoothness points drawn as the step draws them, float32-representable
    rng = O.substream(cfg.seed, O.SMOOTH, iteration)
    xs, xe = O.draw_smooth_points(P32, ods, cfg.weights.smooth_count, cfg.weights.truncation,
                                  cfg.weights.smooth_delta, rng)
    sm = (xs.astype(np.float32).astype(np.float64), xe.astype(np.float32).astype(np.float64))

    batch = sampler.draw_ray_batch(ds, seeds.substream(cfg.seed, seeds.RAYS, iteration),
                                   cfg.batch_rays, near=cfg.near, far=cfg.max_depth)
    total, parts, extras = renderer.train_objective(model, ds, batch, iteration, cfg,
                                                    smooth_override=sm)
    grads = renderer.grad(total, model.parameters())
    g = {n: t.cpu().numpy().copy() for n, t in zip(model.param_names(), grads)}
    eng = renderer.engine_for(model, ds)
    M, N = cfg.batch_rays, extras["samples_per_ray"]
    ws = eng.workspace(M, cfg.coarse_samples, cfg.importance_rounds, cfg.importance_add,
                       cfg.weights.smooth_count)
    dev = {k: ws[k].cpu().numpy().astype(np.float64) for k in ("phi", "gphi", "color", "ray_o",
                                                                 "ray_r")}
    ob = O.draw_ray_batch(ods, O.substream(cfg.seed, O.RAYS, iteration), cfg.batch_rays)
    oracle = _Oracle(P64, ods, ob, iteration, ocfg, sm, extras["depths"], (dev["ray_o"], dev["ray_r"]))
    R, flips = resolve_kinks(oracle, oracle.run(), dev, g, model.param_names(), M, N,
                             cfg.weights.smooth_count)
    return dict(model=model, parts=parts, extras=extras, g=g, dev=dev, R=R, M=M, N=N,
                flips=flips, oracle=oracle)


CASES = ["small", "c1", "c2"]


@pytest.fixture(scope="module", params=CASES)
def conditioned(request):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return request.param, run_case(request.param)


def test_per_sample_outputs(conditioned):
    case, r = conditioned
    R, dev, M, N = r["R"], r["dev"], r["M"], r["N"]
    errs = {
        "phi": rel_maxnorm(dev["phi"][:M * N], R["phi"].reshape(-1)),
        "gphi": rel_maxnorm(dev["gphi"][:M * N], R["gphi"].reshape(-1, 3)),
        "color": rel_maxnorm(dev["color"], R["colors"].reshape(-1, 3)),
    }
    print(case, "per-sample", errs, "kink flips", r["flips"])
    assert max(errs.values()) <= SAMPLE_TOL, errs


def test_loss_parts(conditioned):
    case, r = conditioned
    parts, ref = r["parts"], r["R"]["parts"]
    errs = {k: abs(parts[k] - ref[k]) / max(abs(ref[k]), 1e-12) for k in PART_KEYS}
    print(case, "parts", errs)
    assert max(errs.values()) <= PART_TOL, errs
    for k in ("n_tr", "n_fs", "n_eik", "n_valid_rays"):
        assert r["extras"][k] == r["R"]["extras"][k], k


def test_gradients(conditioned):
    case, r = conditioned
    errs = {n: rel_maxnorm(r["g"][n], r["R"]["grads"][n]) for n in r["model"].param_names()}
    print(case, "grads", errs)
    assert max(errs.values()) <= GRAD_TOL, errs
