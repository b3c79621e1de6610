"""Where a device-trained mesh misses: train SPEC scene #3 (seed S) R times,
and for each run report the final loss, C-l1 / completion at 2000 iterations
(2 cm) and where the ground-truth points farther than 5 cm from the
prediction lie (sphere vs box faces).  Usage (GPU box):
python tools/diag_trained.py [seed] [runs]"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_trained_mesh import gt_mesh, scene_dataset  # noqa: E402
from paper_2206_14735_b200 import mesher, optimizer  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
R = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ds = scene_dataset()
for run in range(R):
    with tempfile.TemporaryDirectory() as d:
        cfg = optimizer.TrainConfig(precision="single", iterations=2000, batch_rays=1024, seed=seed,
                                    checkpoint_every=200)
        model, _ = optimizer.train(ds, cfg, d)
        log = np.loadtxt(os.path.join(d, "loss_log.csv"), delimiter=",", skiprows=1)
        m, _, _, _ = optimizer.load_model(os.path.join(d, "ckpt_002000.gsck"))
        gt = gt_mesh(m, 0.02, ds)
        pred = mesher.cull_mesh(mesher.extract_mesh(m, resolution=0.02), ds)
        rep = mesher.evaluate(pred, gt)
        g_pts, _ = mesher.sample_surface(gt, mesher.EVAL_DENSITY, mesher.EVAL_SEED)
        p_pts, _ = mesher.sample_surface(pred, mesher.EVAL_DENSITY, mesher.EVAL_SEED)
        dg, _ = mesher.nearest_neighbors(g_pts, p_pts, 0.05)
        dp, _ = mesher.nearest_neighbors(p_pts, g_pts, 0.05)
        far_g = g_pts[dg > 0.05]
        far_p = p_pts[dp > 0.05]
        r = np.linalg.norm(far_g - np.array([0.0, 0.0, 0.0]), axis=1) if len(far_g) else np.zeros(0)
        print(f"run {run} seed {seed}: final loss {log[-1, 1]:.4f} (min {log[:, 1].min():.4f}) "
              f"C-l1 {rep.chamfer_l1:.4f} acc {rep.accuracy:.4f} comp {rep.completion:.4f} "
              f"F {rep.f_score:.3f} faces {len(pred.faces)}; gt pts > 5 cm: {len(far_g)} / {len(g_pts)}, "
              f"pred pts > 5 cm: {len(far_p)} / {len(p_pts)}", flush=True)
        if len(far_g):
            lo, hi = far_g.min(axis=0), far_g.max(axis=0)
            print("   missing gt region bbox", np.round(lo, 2).tolist(), np.round(hi, 2).tolist(),
                  "mean", np.round(far_g.mean(axis=0), 2).tolist(), "|x| median", float(np.median(r)), flush=True)
        if len(far_p):
            print("   spurious pred region bbox", np.round(far_p.min(axis=0), 2).tolist(),
                  np.round(far_p.max(axis=0), 2).tolist(), flush=True)
