"""Golden vectors for mesh extraction and metrics, by running the REFERENCE's
``gridsurf.mesher`` (gs/mesher.py).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_golden_mesh.py

scikit-image (the reference's marching cubes) is not installed in this image,
so a stub ``skimage.measure.marching_cubes`` backed by the oracle's
marching cubes (the generated table of mc_table.py) is injected before the
reference mesher is imported.  Everything else is the reference's own code:
sdf_volume, mesh_from_sdf (degenerate-face drop), subdivide_to_edge_length,
cull_mesh (z-buffer visibility), sample_surface, nearest_neighbors, evaluate.
Parity for the marching-cubes table itself is therefore unpinned.

Model: case "small" after the reference's full sphere pre-fit (double), so
the zero level set is a sphere-like surface inside the box.
"""

from __future__ import annotations

import json
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

from oracle import gridsurf_oracle as O  # noqa: E402

_sk = types.ModuleType("skimage")
_measure = types.ModuleType("skimage.measure")


def _marching_cubes(vol, level=0.0, spacing=(1.0, 1.0, 1.0), method="lorensen"):
    v, f = O.marching_cubes(vol, level, spacing)
    return v, f, None, None


_measure.marching_cubes = _marching_cubes
_sk.measure = _measure
sys.modules["skimage"] = _sk
sys.modules["skimage.measure"] = _measure

from gridsurf import decoders, mesher, optimizer  # noqa: E402
from make_golden import CASES, render  # noqa: E402

RES = 0.1
DENSITY = 2e3


def main():
    case = CASES["small"]
    ds = render(case)
    z = np.load(os.path.join(HERE, "init_small_double.npz"))
    meta_init = json.loads(z["meta_json"].tobytes().decode())
    out = {}
    for precision in ("double", "single"):
        cfg = optimizer.TrainConfig(precision=precision, **case["cfg"])
        model = optimizer.build_model(ds, cfg, skip_init=True)
        decoders.geometric_init(model.grid, model.geom_net, meta_init["center"], meta_init["radius"],
                                seed=cfg.seed, max_steps=cfg.init_steps, tol=cfg.init_tol)
        pre = "d_" if precision == "double" else "s_"
        for i, l in enumerate(model.grid.levels):
            out[f"{pre}level{i}"] = l.features.data.copy()
        for i, (W, b) in enumerate(model.geom_net.layers):
            out[f"{pre}geom_w{i}"] = W.data.copy()
            out[f"{pre}geom_b{i}"] = b.data.copy()
        vol, lo, res = mesher.sdf_volume(model, RES)
        out[f"{pre}vol"] = vol
        out[f"{pre}vol_lo"] = np.asarray(lo)
        if precision == "double":
            mesh = mesher.mesh_from_sdf(vol, lo, res)
            out["mesh_v"], out["mesh_f"] = mesh.vertices, mesh.faces
            # ground truth: the analytic sphere, through the same extraction
            c, r = np.asarray(meta_init["center"]), meta_init["radius"]
            h = 0.05
            axes = [lo[a] + np.arange(int((2 * r + 0.6) / h) + 1) * h + (c[a] - r - 0.3 - lo[a]) for a in range(3)]
            X, Y, Zz = np.meshgrid(*axes, indexing="ij")
            gvol = (np.sqrt((X - c[0]) ** 2 + (Y - c[1]) ** 2 + (Zz - c[2]) ** 2) - r).astype(np.float32)
            gt = mesher.mesh_from_sdf(gvol, np.array([axes[0][0], axes[1][0], axes[2][0]]), h)
            out["gt_v"], out["gt_f"] = gt.vertices, gt.faces
            sub = mesher.subdivide_to_edge_length(mesh, 0.06)
            out["sub_v"], out["sub_f"] = sub.vertices, sub.faces
            culled = mesher.cull_mesh(mesh, ds, max_edge=0.12)
            out["cull_v"], out["cull_f"] = culled.vertices, culled.faces
            p_pts, p_nrm = mesher.sample_surface(mesh, DENSITY)
            g_pts, g_nrm = mesher.sample_surface(gt, DENSITY)
            d, i = mesher.nearest_neighbors(p_pts, g_pts, 0.05)
            out["nn_q"], out["nn_ref"], out["nn_d"], out["nn_i"] = p_pts, g_pts, d, i
            rep = mesher.evaluate(mesh, gt, threshold=0.05, density=DENSITY)
            out["metrics_json"] = np.frombuffer(rep.to_json().encode(), dtype=np.uint8)
            print(rep.table())
    meta = dict(res=RES, density=DENSITY, case="small", init=meta_init)
    out["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    path = os.path.join(HERE, "mesh_small.npz")
    np.savez_compressed(path, **out)
    print(path, {k: v.shape for k, v in out.items() if hasattr(v, "shape")})


if __name__ == "__main__":
    main()
